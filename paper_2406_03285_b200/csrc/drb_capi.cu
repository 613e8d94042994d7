// C ABI of the B200 rehearsal buffer (include/drb_rb.h). Host C++: allocation, IPC
// wiring, launch sequencing, error mapping. Conventions follow the reference C ABI
// (proj/src/capi/drb_capi.cpp:15-59): thread-local last error, status codes, guarded calls.

#include <cuda.h>
#include <cuda_runtime.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <stdexcept>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "drb_internal.cuh"

using namespace drb_b200;

namespace {

thread_local std::string t_last_error;

struct status_error : std::runtime_error {
    drb_status code;
    status_error(drb_status c, const std::string& what) : std::runtime_error(what), code(c) {}
};

[[noreturn]] void fail(drb_status c, const std::string& what) { throw status_error(c, what); }

void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess)
        fail(DRB_ERR_INTERNAL, std::string(what) + ": " + cudaGetErrorString(e));
}

template <typename F>
drb_status guarded(F&& f) {
    try {
        f();
        return DRB_OK;
    } catch (const status_error& e) {
        t_last_error = e.what();
        return e.code;
    } catch (const std::bad_alloc&) {
        t_last_error = "out of memory";
        return DRB_ERR_INTERNAL;
    } catch (const std::exception& e) {
        t_last_error = e.what();
        return DRB_ERR_INTERNAL;
    } catch (...) {
        t_last_error = "unknown error";
        return DRB_ERR_INTERNAL;
    }
}

#define DRB_REQUIRE(cond)                                           \
    do {                                                            \
        if (!(cond)) {                                              \
            t_last_error = "null argument";                         \
            return DRB_ERR_INVALID_ARGUMENT;                        \
        }                                                           \
    } while (0)

// Host restatement of derive_key (rng.cpp:19-27) — used only to key the device streams.
uint64_t host_mix64(uint64_t z) {
    z += kPhi;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

uint64_t derive_key(uint64_t seed, uint64_t worker, uint64_t purpose, uint64_t k1, uint64_t k2) {
    uint64_t key = host_mix64(seed);
    key = host_mix64(key ^ (worker * 0xd1342543de82ef95ULL));
    key = host_mix64(key ^ (purpose * 0xaf251af3b0f025b5ULL));
    key = host_mix64(key ^ k1);
    key = host_mix64(key ^ k2);
    return key;
}

struct device_guard {
    int prev = -1;
    explicit device_guard(int dev) {
        cudaGetDevice(&prev);
        if (prev != dev)
            cuda_check(cudaSetDevice(dev), "cudaSetDevice");
    }
    ~device_guard() {
        int cur = -1;
        cudaGetDevice(&cur);
        if (prev >= 0 && cur != prev)
            cudaSetDevice(prev);
    }
};

struct handle_blob {
    uint32_t magic;
    uint32_t version;
    int32_t pid;
    int32_t device;
    uint32_t rank;
    uint32_t world;
    uint64_t region_bytes;
    uint64_t region_ptr;  // raw device pointer (same-process peers)
    uint64_t slab_bytes;
    uint64_t slab_ptr;
    cudaIpcMemHandle_t ipc;
    cudaIpcMemHandle_t slab_ipc;  // the slab: peers pull representatives from it
};
constexpr uint32_t kBlobMagic = 0x44524233;  // "DRB3"

// Scoped temporary device allocation for the synchronous test-facing calls.
struct dev_tmp {
    void* p = nullptr;
    explicit dev_tmp(size_t bytes) { cuda_check(cudaMalloc(&p, bytes ? bytes : 16), "cudaMalloc"); }
    ~dev_tmp() { cudaFree(p); }
    template <typename T>
    T* as() const { return static_cast<T*>(p); }
};

}  // namespace

namespace drb_b200 {
// Shared with drb_dataset.cu: one thread-local last error for the whole C ABI.
void set_last_error(const char* what) { t_last_error = what; }
}  // namespace drb_b200

struct drb_rb {
    drb_rb_config cfg{};
    RegionLayout layout{};
    uint32_t copy_smem = 0;           // dynamic smem of the copy kernel
    uint32_t solo_smem = 0;           // kSoloSmem unless DRB_SOLO=0
    uint32_t grid = 0;                // copy-kernel CTAs (one wave)
    int sm_count = 0;
    cudaStream_t stream = nullptr;    // default stream of the handle (copy kernel)
    cudaStream_t s_sel = nullptr;     // selection chain sel(i)
    cudaStream_t s_plan = nullptr;    // planning chain plan(i)
    cudaStream_t h2d = nullptr;       // host-path input copies
    cudaStream_t d2h = nullptr;       // host-path output copies
    cudaStream_t s_wait = nullptr;    // multi-rank: peers_wait(i) -> "m'_i ready", off the copy chain
    uint8_t* slab = nullptr;          // [K][cap][S]
    uint32_t* slab_labels = nullptr;  // [K][cap]
    uint8_t* region = nullptr;        // own peer-shareable region
    uint8_t* peers[kMaxWorld] = {};   // every rank's region, mapped here
    bool peer_opened[kMaxWorld] = {};
    uint8_t* slab_peers[kMaxWorld] = {};  // every rank's slab, mapped here
    bool slab_opened[kMaxWorld] = {};
    bool connected = false;
    SelState* sel = nullptr;          // [2], sel[cur_sel] is current
    PlanState* plan = nullptr;        // [2], plan[cur_plan] is current
    uint32_t cur_sel = 0, cur_plan = 0;
    uint64_t ver = 0;                 // occupancy table version index (slot = ver % 3)
    uint32_t* report = nullptr;       // [2K+2]
    uint32_t* plist = nullptr;        // [kListRing][plist_words]: P_i, plan(i-1) -> copy(i)
    uint32_t* wlist = nullptr;        // [kListRing][wlist_words]: W_i, sel(i) -> copy(i)
    uint32_t* mailbox = nullptr;      // host-mapped, mb_words(R) (drb_internal.cuh)
    uint32_t* mailbox_dev = nullptr;
    static constexpr int kEv = 40;  // > kListRing (and > the multi-rank lag): per-iteration events in flight
    cudaEvent_t ev_user[kEv] = {}, ev_sel[kEv] = {}, ev_plan[kEv] = {}, ev_copy[kEv] = {};
    cudaEvent_t rel[kEv] = {};  // split steps: the consumer's release at each call
    uint32_t aug_ring = kAugRingDefault;  // R: m' ring depth
    std::vector<cudaEvent_t> done;    // [R] completion of the copy that last wrote each m' slot
    std::vector<uint8_t> slot_run;    // [R] 1: the slot was last filled by a run (see run_done)
    cudaEvent_t run_done = nullptr;   // resident run(): one event after the run's last m'
    cudaEvent_t in_free[2] = {};      // host path: staging slot reusable
    cudaEvent_t h2d_done[2] = {};
    uint8_t* stage = nullptr;         // host path: device staging [2][max_batch][S]
    uint32_t* stage_labels = nullptr; // [2][max_batch]
    uint64_t cand_key = 0, evict_key = 0, samp_key[kMaxWorld] = {};
    uint64_t step = 0;
    uint64_t seq = 0;
    uint64_t dep_floor = 0;           // steps below this completed before a graph capture
    cudaStream_t last_copy_stream = nullptr;
    uint64_t ver0 = 0;                // engine: table version / state parities at start()
    uint32_t sel_par0 = 0, plan_par0 = 0;
    uint32_t dbg_bits = 0;            // DRB_DBG experiment bits (0 in production)
    bool use_persist = true;          // resident engine (DRB_PERSIST=0: three kernels per step)
    bool last_run_persistent = false; // (three-kernel path) the latest drb_rb_run was persistent
    RunCtl* runctl = nullptr;         // device counters of the resident engine
    bool rmode = false;               // this engine runs resident (decided at start())
    FeedDesc* feed = nullptr;         // [kFeedRing] descriptor mirror (device)
    FeedDesc* hdesc = nullptr;        // [kFeedRing] descriptors as the host writes them (mapped)
    FeedDesc* hdesc_dev = nullptr;    // its device address
    uint64_t* feed_seq = nullptr;     // [kFeedRing] posted sequence words (device)
    uint64_t posted = 0;              // descriptors posted
    uint64_t gen = 0;                 // generation of the latest launched instance
    bool alive = false;               // an instance of generation `gen` may be running or queued
    cudaStream_t s_run = nullptr;     // where instances run, one behind the other
    uint32_t run_grid = 0;            // CTAs of an instance (2 control + copy CTAs)
    uint64_t idle_ns = 100ull * 1000;  // an idle instance leaves after this long (frees its SMs)
    uint8_t* astage = nullptr;        // staging of unaligned device batches [4][max_batch][S]
    bool feeder_last = true;          // feeder + ready warps on the last copy CTA, not the sel CTA
    // Under ncu / compute-sanitizer (CUDA_INJECTION64_PATH set) or DRB_TOOL_MODE=1 kernels run
    // one at a time: a resident instance would wait forever for a post queued behind it. So every
    // post launches its own instance (after the post's sequence word) and instances leave as
    // soon as they are idle.
    bool tool_mode = false;
    uint32_t a_ahead = 8;             // A's run-ahead over the completed B (DRB_A_AHEAD)
    uint64_t released = 0;            // split steps: the last m' release written (step index)
    uint64_t release_every = 1;       // split steps: release cadence, max(1, (R - 2) / 4)
    uint64_t* timings = nullptr;      // DRB_RB_FLAG_TIMINGS: per-round device stamps [kTimingRing][8]
    uint64_t timings_drained = 0;     // first round not yet returned by drb_rb_drain_timings
    unsigned long long* prof = nullptr;  // DRB_DBG 65536: sel/plan phase cycle accumulators [64]
    cudaEvent_t run_end = nullptr;
    cudaEvent_t last_work = nullptr;  // after the handle's latest enqueued iteration (any path)
    bool last_work_valid = false;
    uint64_t prewaited = 0;           // 1 + the iteration whose sel/plan the copy stream already waited for
    bool use_pdl = true;              // copy(i+1) launched programmatically behind copy(i); DRB_PDL=0 off
    bool started = false, shut_down = false;
    double wait_ms = 0.0;
    unsigned long long* trace = nullptr;  // DRB_TRACE=1: per-step phase timestamps
    unsigned long long* timeline = nullptr;  // DRB_TIMELINE=<steps>: per-kernel start/end
    uint32_t timeline_steps = 0;
    uint64_t timeout_ns = 10ull * 1000 * 1000 * 1000;
};

namespace {

void check_engine_alive(drb_rb* h) {
    // Sticky failure of an earlier round (device-written, host-mapped), observed without
    // blocking. A round whose failure is not yet visible is caught on the device instead
    // (the next launch sees DevState::error and reports it in its own mailbox slot).
    const uint32_t e = reinterpret_cast<volatile uint32_t*>(h->mailbox)[kMbSticky];
    if (e)
        fail(DRB_ERR_TRAINING, "engine: background pipeline dead: round failed with status " +
                                   std::to_string(e) +
                                   (e == DRB_ERR_USAGE ? " (label out of range)" : " (peer rendezvous timeout)"));
}

StepParams base_params(drb_rb* h) {
    StepParams p{};
    const auto& c = h->cfg;
    p.K = c.n_classes;
    p.cap = c.per_class_cap;
    p.N = c.world;
    p.me = c.rank;
    p.c = c.candidate_count;
    p.r = c.rep_count;
    p.nmax = c.max_batch;
    p.S = c.sample_bytes;
    p.cand_key = h->cand_key;
    p.evict_key = h->evict_key;
    for (int q = 0; q < kMaxWorld; ++q)
        p.samp_key[q] = h->samp_key[q];
    p.slab = h->slab;
    p.slab_labels = h->slab_labels;
    for (int q = 0; q < kMaxWorld; ++q) {
        p.region[q] = h->peers[q];
        p.slab_peer[q] = h->slab_peers[q];
    }
    p.region[c.rank] = h->region;
    p.slab_peer[c.rank] = h->slab;
    p.off_table = h->layout.off_table;
    p.off_counts = h->layout.off_counts;
    p.aug_ring = h->aug_ring;
    p.off_aug = h->layout.off_aug;
    p.off_auglab = h->layout.off_auglab;
    p.aug_slot_bytes = h->layout.aug_slot_bytes;
    p.auglab_slot_elems = align_up(h->layout.rows * 4, 256) / 4;
    p.report = h->report;
    p.mailbox = h->mailbox_dev;
    p.timeout_ns = h->timeout_ns;
    p.smem_bytes = h->copy_smem;
    p.solo_smem = h->solo_smem;
    static const uint32_t dbg = std::getenv("DRB_DBG") ? uint32_t(std::strtoul(std::getenv("DRB_DBG"), nullptr, 0)) : 0u;
    p.dbg = dbg;
    p.trace = h->trace;
    p.prof = h->prof;
    p.timeline = h->timeline;
    p.timeline_steps = h->timeline_steps ? h->timeline_steps : 1;
    p.evict_m = ~0ull / h->cfg.per_class_cap;
    p.seq = h->seq++;
    p.tslot_in = uint32_t(h->ver % kTableRing);
    p.tslot_out = uint32_t((h->ver + 1) % kTableRing);
    p.sel_in = h->sel + h->cur_sel;
    p.sel_out = h->sel + (h->cur_sel ^ 1);
    p.plan_in = h->plan + h->cur_plan;
    p.plan_out = h->plan + (h->cur_plan ^ 1);
    return p;
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

// Stream memory operations (driver API, resolved through the runtime: no -lcuda): the
// resident engine's descriptors are posted and its `ready` word is waited for in stream
// order on the caller's stream, with no kernel launch.
struct memops_t {
    CUresult (*batch)(CUstream, unsigned int, CUstreamBatchMemOpParams*, unsigned int) = nullptr;
    CUresult (*wait64)(CUstream, CUdeviceptr, cuuint64_t, unsigned int) = nullptr;
    bool ok = false;
};
const memops_t& memops() {
    static const memops_t m = [] {
        memops_t r{};
        cudaDriverEntryPointQueryResult q{};
        void* f = nullptr;
        if (cudaGetDriverEntryPointByVersion("cuStreamBatchMemOp", &f, 12000, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            r.batch = reinterpret_cast<decltype(r.batch)>(f);
        f = nullptr;
        if (cudaGetDriverEntryPointByVersion("cuStreamWaitValue64", &f, 12000, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            r.wait64 = reinterpret_cast<decltype(r.wait64)>(f);
        cudaGetLastError();
        r.ok = r.batch && r.wait64;
        return r;
    }();
    return m;
}

volatile unsigned long long* mb64(drb_rb* h, uint32_t word) {
    return reinterpret_cast<volatile unsigned long long*>(h->mailbox + word);
}

// Launch the next instance of the resident engine on s_run (behind the previous one).
void rmode_launch(drb_rb* h) {
    RunParams rp{};
    rp.base = base_params(h);
    rp.base.mode = kModeUpdate | kModeAssemble | kModePlan | kModePublish | (h->cfg.world > 1 ? kModePeers : 0u);
    rp.base.vec16 = 1;
    rp.feed = h->feed;
    rp.hdesc = h->hdesc_dev;
    rp.feed_seq = h->feed_seq;
    rp.desc_done_host = reinterpret_cast<volatile unsigned long long*>(h->mailbox_dev + kMbDescDone);
    rp.ready_host = reinterpret_cast<volatile unsigned long long*>(h->mailbox_dev + kMbReady);
    rp.ctl = h->runctl;
    rp.ver0 = h->ver0;
    rp.sel_base = h->sel;
    rp.plan_base = h->plan;
    rp.plist_base = h->plist;
    rp.wlist_base = h->wlist;
    rp.gen = h->gen + 1;
    rp.idle_ns = h->idle_ns;
    rp.host_posted = reinterpret_cast<const volatile unsigned long long*>(h->mailbox_dev + kMbHostPosted);
    rp.exiting = reinterpret_cast<volatile unsigned long long*>(h->mailbox_dev + kMbExiting);
    rp.quiesce = reinterpret_cast<const volatile uint32_t*>(h->mailbox_dev + kMbQuiesce);
    rp.sel_par0 = h->sel_par0;
    rp.plan_par0 = h->plan_par0;
    rp.pw = plist_words(h->cfg.world, h->cfg.rep_count);
    rp.ww = wlist_words(h->cfg.max_batch);
    rp.copy_ctas = h->run_grid - 2;
    rp.feeder_cta = h->feeder_last ? h->run_grid - 1 : 0;
    rp.timings = h->timings;
    rp.tool_mode = h->tool_mode ? 1u : 0u;
    rp.a_ahead = h->a_ahead;
    if (launch_run(rp, h->run_grid, h->s_run))
        fail(DRB_ERR_INTERNAL, std::string("resident engine launch failed: ") + cudaGetErrorString(cudaGetLastError()));
    h->gen = rp.gen;
    h->alive = true;
}

// `s` waits (in stream order) until m'_{end-1} is ready, i.e. every iteration < end is done.
void rmode_wait(drb_rb* h, uint64_t end, cudaStream_t s) {
    const CUresult r = memops().wait64(reinterpret_cast<CUstream>(s), reinterpret_cast<CUdeviceptr>(&h->runctl->ready),
                                       end, CU_STREAM_WAIT_VALUE_GEQ);
    if (r != CUDA_SUCCESS)
        fail(DRB_ERR_INTERNAL, "feed wait: cuStreamWaitValue64 failed (" + std::to_string(int(r)) + ")");
}

// Post one descriptor (steps [i_begin, i_begin + count) over an input ring) in stream order
// on `s`, launching an instance first if none is resident (or the resident one is leaving).
// The descriptor goes into mapped host memory; `s` then stores its sequence word (and, with
// wait_end, waits until m'_{wait_end-1} is ready): one stream memory-operation batch.
void rmode_post(drb_rb* h, const uint8_t* batches, uint64_t batch_stride, const uint32_t* labels,
                uint64_t label_stride, uint32_t ring, uint32_t first, uint32_t n, uint64_t i_begin, uint32_t count,
                cudaStream_t s, uint64_t wait_end = 0, bool split = false, bool early = false) {
    const uint64_t j = h->posted;
    if (j >= kFeedRing) {  // ring slot j % kFeedRing: descriptor j - kFeedRing must be consumed
        const uint64_t need = j - kFeedRing + 1;
        const auto t0 = std::chrono::steady_clock::now();
        while (*mb64(h, kMbDescDone) < need) {
            check_engine_alive(h);
            if (std::chrono::steady_clock::now() - t0 > std::chrono::nanoseconds(h->timeout_ns))
                fail(DRB_ERR_TRAINING, "engine: " + std::to_string(kFeedRing) +
                                           " posted steps are not consumed (is a posting stream blocked?)");
            std::this_thread::yield();
        }
    }
    FeedDesc& d = h->hdesc[j % kFeedRing];
    d.batches = reinterpret_cast<uint64_t>(batches);
    d.labels = reinterpret_cast<uint64_t>(labels);
    d.batch_stride = batch_stride;
    d.label_stride = label_stride;
    d.i_begin = i_begin;
    d.count_n = uint64_t(count) | (uint64_t(n) << 32) | (split ? kDescSplit : 0ull) | (early ? kDescEarly : 0ull);
    d.ring_first = uint64_t(ring) | (uint64_t(first) << 32);
    d.seq = j + 1;
    *reinterpret_cast<volatile uint32_t*>(h->mailbox + kMbQuiesce) = 0;
    *mb64(h, kMbHostPosted) = j + 1;
    std::atomic_thread_fence(std::memory_order_seq_cst);  // (Dekker with the leaving feeder)
    const uint64_t ex = *mb64(h, kMbExiting);
    const bool launch = h->tool_mode || !h->alive || (ex >> 32) == (h->gen & 0xffffffffull);
    uint64_t* seq = h->feed_seq + (j % kFeedRing);
    if (launch) {
        // with a launch: the sequence word first, then the instance, then the wait — an
        // instance launched behind work that waits for it would never start under a tool that
        // serialises the device (ncu, compute-sanitizer)
        {
            CUstreamBatchMemOpParams op;
            std::memset(&op, 0, sizeof op);
            op.writeValue.operation = CU_STREAM_MEM_OP_WRITE_VALUE_64;
            op.writeValue.address = reinterpret_cast<CUdeviceptr>(seq);
            op.writeValue.value64 = j + 1;
            op.writeValue.flags = CU_STREAM_WRITE_VALUE_DEFAULT;
            const CUresult r = memops().batch(reinterpret_cast<CUstream>(s), 1, &op, 0);
            if (r != CUDA_SUCCESS)
                fail(DRB_ERR_INTERNAL, "feed post: cuStreamBatchMemOp failed (" + std::to_string(int(r)) + ")");
        }
        rmode_launch(h);
        if (wait_end)
            rmode_wait(h, wait_end, s);
    } else {
        CUstreamBatchMemOpParams ops[2];
        std::memset(ops, 0, sizeof ops);
        ops[0].writeValue.operation = CU_STREAM_MEM_OP_WRITE_VALUE_64;
        ops[0].writeValue.address = reinterpret_cast<CUdeviceptr>(seq);
        ops[0].writeValue.value64 = j + 1;
        ops[0].writeValue.flags = CU_STREAM_WRITE_VALUE_DEFAULT;  // after the stream's prior work
        uint32_t c = 1;
        if (wait_end) {
            ops[1].waitValue.operation = CU_STREAM_MEM_OP_WAIT_VALUE_64;
            ops[1].waitValue.address = reinterpret_cast<CUdeviceptr>(&h->runctl->ready);
            ops[1].waitValue.value64 = wait_end;
            ops[1].waitValue.flags = CU_STREAM_WAIT_VALUE_GEQ;
            c = 2;
        }
        const CUresult r = memops().batch(reinterpret_cast<CUstream>(s), c, ops, 0);
        if (r != CUDA_SUCCESS)
            fail(DRB_ERR_INTERNAL, "feed post: cuStreamBatchMemOp failed (" + std::to_string(int(r)) + ")");
    }
    h->posted = j + 1;
}

// Ask a resident instance to leave as soon as it is idle (before a device-wide sync).
void rmode_quiesce(drb_rb* h) {
    if (h->rmode)
        *reinterpret_cast<volatile uint32_t*>(h->mailbox + kMbQuiesce) = 1;
}

}  // namespace

extern "C" {

const char* drb_rb_version(void) { return "drb-b200 0.1.0 (sm_100a)"; }

const char* drb_rb_last_error(void) { return t_last_error.c_str(); }

drb_status drb_rng_init(drb_rng* s, uint64_t seed, uint32_t worker, uint32_t purpose) {
    DRB_REQUIRE(s);
    s->key = derive_key(seed, worker, purpose, 0, 0);
    s->ctr = 0;
    return DRB_OK;
}

drb_status drb_rng_keyed(drb_rng* s, uint64_t seed, uint32_t worker, uint32_t purpose,
                         uint64_t k1, uint64_t k2) {
    DRB_REQUIRE(s);
    s->key = derive_key(seed, worker, purpose, k1 + 1, k2 + 1);
    s->ctr = 0;
    return DRB_OK;
}

drb_status drb_rng_draw(drb_rng* s, uint64_t bound, uint64_t n, uint64_t* out, int32_t device) {
    DRB_REQUIRE(s && (out || n == 0));
    return guarded([&] {
        device_guard g(device);
        dev_tmp d_out(n * 8), d_ctr(8);
        if (launch_rng_draw(s->key, s->ctr, bound, n, d_out.as<uint64_t>(), d_ctr.as<uint64_t>(), nullptr))
            fail(DRB_ERR_INTERNAL, "rng_draw launch failed");
        cuda_check(cudaMemcpy(out, d_out.p, n * 8, cudaMemcpyDeviceToHost), "rng_draw copy");
        cuda_check(cudaMemcpy(&s->ctr, d_ctr.p, 8, cudaMemcpyDeviceToHost), "rng_draw ctr");
    });
}

drb_status drb_sample_without_replacement(uint32_t n, uint32_t k, drb_rng* s, uint32_t* out,
                                          uint32_t* out_k, int32_t device) {
    DRB_REQUIRE(s && out_k && (out || k == 0 || n == 0));
    return guarded([&] {
        device_guard g(device);
        const uint32_t kk = k < n ? k : n;
        dev_tmp d_out(size_t(kk) * 4), d_ctr(8);
        if (launch_swor(s->key, s->ctr, n, kk, d_out.as<uint32_t>(), d_ctr.as<uint64_t>(), nullptr))
            fail(DRB_ERR_INTERNAL, "swor launch failed");
        cuda_check(cudaMemcpy(out, d_out.p, size_t(kk) * 4, cudaMemcpyDeviceToHost), "swor copy");
        cuda_check(cudaMemcpy(&s->ctr, d_ctr.p, 8, cudaMemcpyDeviceToHost), "swor ctr");
        *out_k = kk;
    });
}

drb_status drb_plan(uint32_t want, uint32_t n_workers, uint32_t n_classes, const uint32_t* occ,
                    drb_rng* s, drb_slot_ref* out, uint32_t* out_count, int32_t device) {
    DRB_REQUIRE(occ && s && out_count);
    return guarded([&] {
        device_guard g(device);
        const size_t nk = size_t(n_workers) * n_classes;
        if (nk == 0)
            fail(DRB_ERR_USAGE, "plan: empty view");
        uint64_t total = 0;
        for (size_t i = 0; i < nk; ++i)
            total += occ[i];
        if (total >= (1ull << 31))
            fail(DRB_ERR_CONFIG, "plan: view larger than 2^31 slots");
        const uint32_t entries = uint32_t(want < total ? want : total);
        dev_tmp d_occ(nk * 4), d_out(size_t(entries) * 12), d_cnt(4), d_ctr(8);
        cuda_check(cudaMemcpy(d_occ.p, occ, nk * 4, cudaMemcpyHostToDevice), "plan occ");
        if (launch_plan(s->key, s->ctr, want, entries, n_workers, n_classes, d_occ.as<uint32_t>(),
                        d_out.as<uint32_t>(), d_cnt.as<uint32_t>(), d_ctr.as<uint64_t>(), nullptr))
            fail(DRB_ERR_INTERNAL, "plan launch failed");
        uint32_t c = 0;
        cuda_check(cudaMemcpy(&c, d_cnt.p, 4, cudaMemcpyDeviceToHost), "plan count");
        if (c && !out)
            fail(DRB_ERR_INVALID_ARGUMENT, "plan: null output");
        cuda_check(cudaMemcpy(out, d_out.p, size_t(c) * 12, cudaMemcpyDeviceToHost), "plan out");
        cuda_check(cudaMemcpy(&s->ctr, d_ctr.p, 8, cudaMemcpyDeviceToHost), "plan ctr");
        *out_count = c;
    });
}

}  // extern "C"

namespace {

// Regularized upper incomplete gamma Q(a, x): the power series of P for x < a + 1, else the
// modified-Lentz continued fraction of Q (the same split as proj/src/metrics/stats.cpp).
double gamma_q(double a, double x) {
    if (x <= 0.0)
        return 1.0;
    const double front = std::exp(-x + a * std::log(x) - std::lgamma(a));
    if (x < a + 1.0) {
        double term = 1.0 / a, sum = term;
        for (int n = 1; n < 100000; ++n) {
            term *= x / (a + n);
            sum += term;
            if (std::fabs(term) < std::fabs(sum) * 1e-17)
                break;
        }
        return 1.0 - sum * front;
    }
    const double tiny = 1e-300;
    double b = x + 1.0 - a, c = 1.0 / tiny, d = 1.0 / b, h = d;
    for (int i = 1; i < 100000; ++i) {
        const double an = -i * (i - a);
        b += 2.0;
        d = an * d + b;
        if (std::fabs(d) < tiny)
            d = tiny;
        c = b + an / c;
        if (std::fabs(c) < tiny)
            c = tiny;
        d = 1.0 / d;
        const double del = d * c;
        h *= del;
        if (std::fabs(del - 1.0) < 1e-16)
            break;
    }
    return front * h;
}

}  // namespace

extern "C" {

drb_status drb_rb_bias_test(uint32_t n_workers, uint32_t n_classes, uint32_t rep_count, uint64_t seed,
                            uint64_t draws, uint64_t fill, int biased_control, uint64_t* counts,
                            double* statistic, double* p_value, int32_t device) {
    DRB_REQUIRE(statistic && p_value);
    return guarded([&] {
        if (n_workers == 0 || n_workers > kMaxWorld || n_classes == 0)
            fail(DRB_ERR_CONFIG, "bias test: need 1 <= n_workers <= 8 and n_classes >= 1");
        if (fill < n_workers)  // bias.cpp:37-38
            fail(DRB_ERR_CONFIG, "bias test: fill must provide at least one sample per worker");
        if (fill >= (1ull << 31))
            fail(DRB_ERR_CONFIG, "bias test: fill larger than 2^31 slots");
        if (draws == 0 || rep_count == 0)  // make_bias_report: zero expected count per slot
            fail(DRB_ERR_USAGE, "bias test: zero expected count per slot");
        // frozen view after the fill phase (bias.cpp:42-45,84-89): all inserted
        uint64_t total0 = 0;
        for (uint32_t c = 0; c < n_classes; ++c) {
            const uint64_t here = fill / n_workers + (0 < fill % n_workers ? 1 : 0);
            total0 += here / n_classes + (c < here % n_classes ? 1 : 0);
        }
        const uint64_t total = fill;  // sum over ranks of fill_here
        device_guard g(device);
        dev_tmp d_counts(total * 8), d_ctr(8);
        cuda_check(cudaMemset(d_counts.p, 0, total * 8), "bias counts");
        const uint64_t key = derive_key(seed, 0, DRB_PURPOSE_GLOBAL_SAMPLING, 0, 0);
        if (launch_bias_counts(key, rep_count, uint32_t(biased_control ? total0 : total), draws,
                               d_counts.as<unsigned long long>(), d_ctr.as<uint64_t>(), nullptr))
            fail(DRB_ERR_INTERNAL, std::string("bias launch failed: ") + cudaGetErrorString(cudaGetLastError()));
        std::vector<uint64_t> obs(total);
        cuda_check(cudaMemcpy(obs.data(), d_counts.p, total * 8, cudaMemcpyDeviceToHost), "bias counts copy");
        if (counts)
            std::memcpy(counts, obs.data(), total * 8);
        // Pearson chi-square against uniform (metrics.cpp:90-107)
        const double expected = double(rep_count) * double(draws) / double(total);
        double stat = 0.0;
        for (uint64_t x = 0; x < total; ++x) {
            const double diff = double(obs[x]) - expected;
            stat += diff * diff / expected;
        }
        *statistic = stat;
        *p_value = total > 1 ? gamma_q(double(total - 1) / 2.0, stat / 2.0) : 1.0;
    });
}

drb_status drb_rb_create(const drb_rb_config* cfg, drb_rb** out) {
    DRB_REQUIRE(cfg && out);
    *out = nullptr;
    return guarded([&] {
        const auto& c = *cfg;
        if (c.n_classes == 0 || c.per_class_cap == 0)
            fail(DRB_ERR_CONFIG, "rehearsal_buffer: class count and per-class capacity must be >= 1");
        if (c.sample_bytes == 0 || c.sample_bytes % 4)
            fail(DRB_ERR_CONFIG, "rehearsal_buffer: sample_bytes must be a positive multiple of 4");
        if (c.world == 0 || c.world > kMaxWorld || c.rank >= c.world)
            fail(DRB_ERR_CONFIG, "rehearsal_buffer: need 1 <= world <= 8 and rank < world");
        if (c.max_batch == 0 || c.max_batch > 4096)
            fail(DRB_ERR_CONFIG, "rehearsal_buffer: max_batch must be in [1, 4096]");
        if (c.rep_count > 4096 || uint64_t(c.world) * c.rep_count > 4096)
            fail(DRB_ERR_CONFIG, "rehearsal_buffer: world * rep_count must be <= 4096");
        if (c.aug_ring != 0 && (c.aug_ring < kAugRingMin || c.aug_ring > kAugRingMax))
            fail(DRB_ERR_CONFIG, "rehearsal_buffer: aug_ring must be 0 (default 32) or in [6, 65536]");
        if (uint64_t(c.world) * c.n_classes * c.per_class_cap >= (1ull << 31))
            fail(DRB_ERR_CONFIG, "rehearsal_buffer: N*K*cap must be < 2^31 slots");
        const uint32_t plan_bytes = plan_smem_bytes(c.world, c.n_classes, c.rep_count);
        if (plan_bytes > 200 * 1024 || sel_smem_bytes(c.n_classes, c.max_batch) > 200 * 1024)
            fail(DRB_ERR_CONFIG, "rehearsal_buffer: N*K too large for the on-chip view (" +
                                     std::to_string(plan_bytes) + " B shared memory)");
        auto h = new drb_rb();
        std::unique_ptr<drb_rb> guard_h(h);
        h->cfg = c;
        h->aug_ring = c.aug_ring ? c.aug_ring : kAugRingDefault;
        h->release_every = std::max<uint64_t>(1, (h->aug_ring - 2) / 4);
        h->layout = region_layout(c.world, c.n_classes, c.sample_bytes, c.max_batch, c.rep_count, h->aug_ring);
        h->copy_smem = copy_smem(c.world, c.rep_count, c.max_batch).words * 4;
        {
            const char* so = std::getenv("DRB_SOLO");  // DRB_SOLO=0: let the kernels share SMs
            h->solo_smem = (so && so[0] == '0') ? 0u
                                                : solo_smem_for(tma_smem(c.world, c.rep_count, c.max_batch).bytes);
            h->copy_smem = std::max(h->copy_smem, h->solo_smem);
        }
        if (const char* t = std::getenv("DRB_TIMEOUT_MS"))
            h->timeout_ns = std::strtoull(t, nullptr, 10) * 1000000ull;
        device_guard g(c.device);
        cuda_check(cudaDeviceGetAttribute(&h->sm_count, cudaDevAttrMultiProcessorCount, c.device), "sm count");
        int per_sm = 0;
        if (copy_kernel_max_ctas_per_sm(h->copy_smem, &per_sm) || per_sm < 1)
            fail(DRB_ERR_CONFIG, "copy kernel does not fit on an SM");
        // one copy CTA per SM (a single wave), minus the two SMs sel and plan run on
        h->grid = uint32_t(h->sm_count) - ((h->solo_smem && h->sm_count > 4) ? 2u : 0u);
        if (const char* gs = std::getenv("DRB_GRID"))
            h->grid = uint32_t(std::strtoul(gs, nullptr, 10));
        cuda_check(cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking), "stream");
        cuda_check(cudaStreamCreateWithFlags(&h->s_sel, cudaStreamNonBlocking), "stream");
        cuda_check(cudaStreamCreateWithFlags(&h->s_plan, cudaStreamNonBlocking), "stream");
        cuda_check(cudaStreamCreateWithFlags(&h->h2d, cudaStreamNonBlocking), "stream");
        cuda_check(cudaStreamCreateWithFlags(&h->d2h, cudaStreamNonBlocking), "stream");
        cuda_check(cudaStreamCreateWithFlags(&h->s_wait, cudaStreamNonBlocking), "stream");
        cuda_check(cudaStreamCreateWithFlags(&h->s_run, cudaStreamNonBlocking), "stream");
        const uint64_t slab_bytes = uint64_t(c.n_classes) * c.per_class_cap * c.sample_bytes;
        cuda_check(cudaMalloc(&h->slab, slab_bytes), "slab alloc");
        cuda_check(cudaMalloc(&h->slab_labels, uint64_t(c.n_classes) * c.per_class_cap * 4), "labels alloc");
        cuda_check(cudaMemset(h->slab_labels, 0, uint64_t(c.n_classes) * c.per_class_cap * 4), "memset");
        cuda_check(cudaMalloc(&h->region, h->layout.bytes), "region alloc");
        cuda_check(cudaMemset(h->region, 0, h->layout.bytes), "memset");
        cuda_check(cudaMalloc(&h->sel, 2 * sizeof(SelState)), "state alloc");
        cuda_check(cudaMemset(h->sel, 0, 2 * sizeof(SelState)), "memset");
        cuda_check(cudaMalloc(&h->plan, 2 * sizeof(PlanState)), "state alloc");
        cuda_check(cudaMemset(h->plan, 0, 2 * sizeof(PlanState)), "memset");
        cuda_check(cudaMalloc(&h->report, (2ull * c.n_classes + 2) * 4), "report alloc");
        cuda_check(cudaMalloc(&h->plist, uint64_t(kListRing) * plist_words(c.world, c.rep_count) * 4), "plist alloc");
        cuda_check(cudaMemset(h->plist, 0, uint64_t(kListRing) * plist_words(c.world, c.rep_count) * 4), "memset");
        cuda_check(cudaMalloc(&h->wlist, uint64_t(kListRing) * wlist_words(c.max_batch) * 4), "wlist alloc");
        cuda_check(cudaMemset(h->wlist, 0, uint64_t(kListRing) * wlist_words(c.max_batch) * 4), "memset");
        cuda_check(cudaHostAlloc(&h->mailbox, mb_words(h->aug_ring) * 4, cudaHostAllocMapped), "mailbox");
        std::memset(h->mailbox, 0, mb_words(h->aug_ring) * 4);
        cuda_check(cudaHostGetDevicePointer(reinterpret_cast<void**>(&h->mailbox_dev), h->mailbox, 0), "mailbox map");
        h->done.assign(h->aug_ring, nullptr);
        h->slot_run.assign(h->aug_ring, 0);
        cuda_check(cudaEventCreateWithFlags(&h->run_done, cudaEventDisableTiming), "event");
        for (auto& e : h->done)
            cuda_check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
        for (int i = 0; i < drb_rb::kEv; ++i)
            for (cudaEvent_t* e : {&h->ev_user[i], &h->ev_sel[i], &h->ev_plan[i], &h->ev_copy[i], &h->rel[i]})
                cuda_check(cudaEventCreateWithFlags(e, cudaEventDisableTiming), "event");
        for (int i = 0; i < 2; ++i) {
            cuda_check(cudaEventCreateWithFlags(&h->in_free[i], cudaEventDisableTiming), "event");
            cuda_check(cudaEventCreateWithFlags(&h->h2d_done[i], cudaEventDisableTiming), "event");
        }
        h->cand_key = derive_key(c.seed, c.rank, DRB_PURPOSE_CANDIDATE_SELECTION, 0, 0);
        h->evict_key = derive_key(c.seed, c.rank, DRB_PURPOSE_EVICTION, 0, 0);
        for (uint32_t q = 0; q < kMaxWorld; ++q)
            h->samp_key[q] = derive_key(c.seed, q, DRB_PURPOSE_GLOBAL_SAMPLING, 0, 0);
        h->peers[c.rank] = h->region;
        h->slab_peers[c.rank] = h->slab;
        if (const char* tl = std::getenv("DRB_TIMELINE")) {
            h->timeline_steps = uint32_t(std::strtoul(tl, nullptr, 10));
            if (h->timeline_steps) {  // a power of two: stamps index the ring with a mask
                uint32_t p2 = 1;
                while (p2 < h->timeline_steps)
                    p2 <<= 1;
                h->timeline_steps = p2;
            }
            if (h->timeline_steps) {
                cuda_check(cudaMalloc(&h->timeline, h->timeline_steps * uint64_t(kTlStride) * 8), "timeline alloc");
                std::vector<unsigned long long> init(h->timeline_steps * uint64_t(kTlStride), 0ull);
                for (size_t x = 0; x < init.size(); x += kTlStride)
                    for (int k = 0; k < 6; k += 2)
                        init[x + k] = ~0ull;
                cuda_check(cudaMemcpy(h->timeline, init.data(), init.size() * 8, cudaMemcpyHostToDevice), "timeline init");
            }
        }
        if (const char* db = std::getenv("DRB_DBG"))
            h->dbg_bits = uint32_t(std::strtoul(db, nullptr, 0));
        if (const char* pd = std::getenv("DRB_PDL"); pd && pd[0] == '0')
            h->use_pdl = false;
        if (const char* pe = std::getenv("DRB_PERSIST"))
            h->use_persist = pe[0] == '1';
        cuda_check(cudaMalloc(&h->runctl, sizeof(RunCtl)), "run state alloc");
        cuda_check(cudaMemset(h->runctl, 0, sizeof(RunCtl)), "memset");
        cuda_check(cudaMalloc(&h->feed, kFeedRing * sizeof(FeedDesc)), "feed alloc");
        cuda_check(cudaMemset(h->feed, 0, kFeedRing * sizeof(FeedDesc)), "memset");
        cuda_check(cudaMalloc(&h->feed_seq, kFeedRing * 8), "feed alloc");
        cuda_check(cudaMemset(h->feed_seq, 0, kFeedRing * 8), "memset");
        cuda_check(cudaHostAlloc(&h->hdesc, kFeedRing * sizeof(FeedDesc), cudaHostAllocMapped), "feed alloc");
        std::memset(h->hdesc, 0, kFeedRing * sizeof(FeedDesc));
        cuda_check(cudaHostGetDevicePointer(reinterpret_cast<void**>(&h->hdesc_dev), h->hdesc, 0), "feed map");
        // engine CTAs: half the GPU by default, so a training step co-runs on the other half
        h->run_grid = c.engine_ctas ? std::max(3u, std::min(uint32_t(h->sm_count), c.engine_ctas))
                                    : std::max(4u, uint32_t(h->sm_count) / 2);
        if (const char* rg = std::getenv("DRB_RUN_GRID"))
            h->run_grid = std::max(3u, std::min(uint32_t(h->sm_count), uint32_t(std::strtoul(rg, nullptr, 10))));
        if (const char* iu = std::getenv("DRB_IDLE_US"))
            h->idle_ns = std::strtoull(iu, nullptr, 10) * 1000ull;
        if (c.flags & DRB_RB_FLAG_TIMINGS) {
            cuda_check(cudaMalloc(&h->timings, uint64_t(kTimingRing) * kTimingWords * 8), "timings alloc");
            cuda_check(cudaMemset(h->timings, 0, uint64_t(kTimingRing) * kTimingWords * 8), "memset");
        }
        if (std::getenv("CUDA_INJECTION64_PATH") || (std::getenv("DRB_TOOL_MODE") &&
                                                     std::getenv("DRB_TOOL_MODE")[0] == '1'))
            h->tool_mode = true;
        if (const char* aa = std::getenv("DRB_A_AHEAD"))
            h->a_ahead = std::max(2u, uint32_t(std::strtoul(aa, nullptr, 10)));
        if (const char* fl = std::getenv("DRB_FEEDER_LAST"))
            h->feeder_last = fl[0] != '0';
        if (h->dbg_bits & 65536) {
            cuda_check(cudaMalloc(&h->prof, 64 * 8), "prof alloc");
            cuda_check(cudaMemset(h->prof, 0, 64 * 8), "prof alloc");
        }
        cuda_check(cudaEventCreateWithFlags(&h->run_end, cudaEventDisableTiming), "event");
        cuda_check(cudaEventCreateWithFlags(&h->last_work, cudaEventDisableTiming), "event");
        if (const char* tr = std::getenv("DRB_TRACE"); tr && tr[0] == '1')
            cuda_check(cudaMalloc(&h->trace, 32 * 8), "trace alloc");
        if (h->dbg_bits & 64) {
            int occ = 0;
            const uint32_t tb = tma_smem(c.world, c.rep_count, c.max_batch).bytes;
            copy_tma_occupancy(tb, &occ);
            std::fprintf(stderr, "drb: tma copy smem %u B, %d CTA/SM; sel/plan floor %u B; grid %u\n", tb, occ,
                         h->solo_smem, h->grid);
        }
        if (c.world == 1)
            h->connected = true;
        cuda_check(cudaDeviceSynchronize(), "create sync");
        *out = guard_h.release();
    });
}

drb_status drb_rb_destroy(drb_rb* h) {
    if (!h)
        return DRB_OK;
    return guarded([&] {
        device_guard g(h->cfg.device);
        rmode_quiesce(h);
        cudaDeviceSynchronize();
        for (uint32_t w = 0; w < h->cfg.world; ++w) {
            if (h->peer_opened[w])
                cudaIpcCloseMemHandle(h->peers[w]);
            if (h->slab_opened[w])
                cudaIpcCloseMemHandle(h->slab_peers[w]);
        }
        cudaFree(h->slab);
        cudaFree(h->slab_labels);
        cudaFree(h->region);
        cudaFree(h->sel);
        cudaFree(h->plan);
        cudaFree(h->report);
        cudaFree(h->plist);
        cudaFree(h->wlist);
        cudaFree(h->trace);
        cudaFree(h->timeline);
        cudaFree(h->stage);
        cudaFree(h->stage_labels);
        cudaFreeHost(h->mailbox);
        for (auto e : h->done)
            cudaEventDestroy(e);
        if (h->run_done)
            cudaEventDestroy(h->run_done);
        for (int i = 0; i < drb_rb::kEv; ++i)
            for (cudaEvent_t e : {h->ev_user[i], h->ev_sel[i], h->ev_plan[i], h->ev_copy[i], h->rel[i]})
                cudaEventDestroy(e);
        for (int i = 0; i < 2; ++i) {
            cudaEventDestroy(h->in_free[i]);
            cudaEventDestroy(h->h2d_done[i]);
        }
        cudaStreamDestroy(h->stream);
        cudaStreamDestroy(h->s_sel);
        if (h->runctl)
            cudaFree(h->runctl);
        cudaFree(h->feed);
        cudaFree(h->feed_seq);
        cudaFree(h->timings);
        if (h->hdesc)
            cudaFreeHost(h->hdesc);
        cudaFree(h->astage);
        cudaStreamDestroy(h->s_run);
        if (h->prof)
            cudaFree(h->prof);
        if (h->run_end)
            cudaEventDestroy(h->run_end);
        if (h->last_work)
            cudaEventDestroy(h->last_work);
        cudaStreamDestroy(h->s_plan);
        cudaStreamDestroy(h->h2d);
        cudaStreamDestroy(h->d2h);
        cudaStreamDestroy(h->s_wait);
        delete h;
    });
}

drb_status drb_rb_update_buffer(drb_rb* h, const void* batch, const uint32_t* labels, uint32_t n,
                                uint32_t c, drb_rng* cand, drb_rng* evict,
                                drb_insertion_report* report) {
    DRB_REQUIRE(h && cand && evict && ((batch && labels) || n == 0));
    return guarded([&] {
        if (h->started)
            fail(DRB_ERR_USAGE, "update_buffer: the buffer is driven by its engine once started");
        if (n > h->cfg.max_batch)
            fail(DRB_ERR_USAGE, "update_buffer: batch larger than max_batch");
        device_guard g(h->cfg.device);
        StepParams p = base_params(h);
        p.n = n;
        p.c = c;
        p.batch = static_cast<const uint8_t*>(batch);
        p.labels = labels;
        p.cand_key = cand->key;
        p.evict_key = evict->key;
        p.cand_ctr0 = cand->ctr;
        p.evict_ctr0 = evict->ctr;
        p.mode = kModeUpdate | kModeReport | kModeCtrParams | kModePublish;
        p.wlist = h->wlist;
        p.plist_in = nullptr;
        p.plist_out = nullptr;
        p.vec16 = (p.S % 16 == 0) && (n == 0 || aligned16(batch));
        p.mailbox = nullptr;
        if (launch_sel(p, h->stream) || launch_copy(p, h->grid, h->stream, false))
            fail(DRB_ERR_INTERNAL, std::string("update launch failed: ") + cudaGetErrorString(cudaGetLastError()));
        SelState st{};
        cuda_check(cudaMemcpyAsync(&st, p.sel_out, sizeof st, cudaMemcpyDeviceToHost, h->stream), "state copy");
        std::vector<uint32_t> rep(2ull * h->cfg.n_classes + 2);
        cuda_check(cudaMemcpyAsync(rep.data(), h->report, rep.size() * 4, cudaMemcpyDeviceToHost, h->stream), "report copy");
        cuda_check(cudaStreamSynchronize(h->stream), "update_buffer");
        if (st.error == DRB_ERR_USAGE) {
            // usage_error is raised before any draw and leaves the buffer untouched
            // (rehearsal_buffer.cpp:44-47): discard the produced state.
            fail(DRB_ERR_USAGE, "update_buffer: label out of range (K=" + std::to_string(h->cfg.n_classes) + ")");
        }
        h->cur_sel ^= 1;
        h->ver += 1;
        cand->ctr = st.cand_ctr;
        evict->ctr = st.evict_ctr;
        if (report) {
            const uint32_t K = h->cfg.n_classes;
            if (report->per_class_appends)
                std::memcpy(report->per_class_appends, rep.data(), K * 4);
            if (report->per_class_replacements)
                std::memcpy(report->per_class_replacements, rep.data() + K, K * 4);
            report->appends = rep[2 * K];
            report->replacements = rep[2 * K + 1];
        }
    });
}

drb_status drb_rb_read_slots(drb_rb* h, const drb_read_request* requests, uint32_t count,
                             drb_rng* substitute, void* out, uint32_t* out_labels, uint8_t* status) {
    DRB_REQUIRE(h && substitute && ((requests && out && out_labels && status) || count == 0));
    return guarded([&] {
        device_guard g(h->cfg.device);
        dev_tmp d_req(size_t(count) * 8), d_status(count), d_ctr(8);
        cuda_check(cudaMemcpy(d_req.p, requests, size_t(count) * 8, cudaMemcpyHostToDevice), "req copy");
        const uint64_t* row = reinterpret_cast<const uint64_t*>(h->region + h->layout.off_table) +
                              (h->ver % kTableRing) * uint64_t(h->cfg.world) * h->cfg.n_classes +
                              uint64_t(h->cfg.rank) * h->cfg.n_classes;
        rmode_quiesce(h);
        cuda_check(cudaDeviceSynchronize(), "read_slots order");
        dev_tmp d_occ(size_t(h->cfg.n_classes) * 4);  // the counts of the versioned words
        cuda_check(cudaMemcpy2D(d_occ.p, 4, row, 8, 4, h->cfg.n_classes, cudaMemcpyDeviceToDevice), "occ copy");
        const uint32_t* occ = d_occ.as<uint32_t>();
        if (launch_read_slots(h->slab, h->slab_labels, occ, h->cfg.n_classes, h->cfg.per_class_cap,
                              h->cfg.sample_bytes, d_req.as<uint32_t>(), count, substitute->key,
                              substitute->ctr, static_cast<uint8_t*>(out), out_labels,
                              d_status.as<uint8_t>(), d_ctr.as<uint64_t>(), h->stream))
            fail(DRB_ERR_INTERNAL, "read_slots launch failed");
        cuda_check(cudaStreamSynchronize(h->stream), "read_slots");
        cuda_check(cudaMemcpy(status, d_status.p, count, cudaMemcpyDeviceToHost), "status copy");
        cuda_check(cudaMemcpy(&substitute->ctr, d_ctr.p, 8, cudaMemcpyDeviceToHost), "ctr copy");
    });
}

drb_status drb_rb_snapshot(drb_rb* h, uint32_t* per_class, uint64_t* version) {
    DRB_REQUIRE(h && per_class && version);
    return guarded([&] {
        device_guard g(h->cfg.device);
        rmode_quiesce(h);
        cuda_check(cudaDeviceSynchronize(), "snapshot order");
        const uint64_t* row = reinterpret_cast<const uint64_t*>(h->region + h->layout.off_table) +
                              (h->ver % kTableRing) * uint64_t(h->cfg.world) * h->cfg.n_classes +
                              uint64_t(h->cfg.rank) * h->cfg.n_classes;
        cuda_check(cudaMemcpy2D(per_class, 4, row, 8, 4, h->cfg.n_classes, cudaMemcpyDeviceToHost), "snapshot");
        SelState st{};
        cuda_check(cudaMemcpy(&st, h->sel + h->cur_sel, sizeof st, cudaMemcpyDeviceToHost), "state");
        *version = st.version;
    });
}

drb_status drb_rb_total_stored(drb_rb* h, uint64_t* out) {
    DRB_REQUIRE(h && out);
    return guarded([&] {
        device_guard g(h->cfg.device);
        rmode_quiesce(h);
        cuda_check(cudaDeviceSynchronize(), "order");
        SelState st{};
        cuda_check(cudaMemcpy(&st, h->sel + h->cur_sel, sizeof st, cudaMemcpyDeviceToHost), "state");
        *out = st.total;
    });
}

drb_status drb_rb_cross_class_evictions(drb_rb* h, uint64_t* out) {
    DRB_REQUIRE(h && out);
    return guarded([&] {
        device_guard g(h->cfg.device);
        rmode_quiesce(h);
        cuda_check(cudaDeviceSynchronize(), "order");
        SelState st{};
        cuda_check(cudaMemcpy(&st, h->sel + h->cur_sel, sizeof st, cudaMemcpyDeviceToHost), "state");
        *out = st.cross_class;
    });
}

drb_status drb_rb_device_views(drb_rb* h, void** slab, uint32_t** slab_labels) {
    DRB_REQUIRE(h && slab && slab_labels);
    *slab = h->slab;
    *slab_labels = h->slab_labels;
    return DRB_OK;
}

size_t drb_rb_handle_size(void) { return sizeof(handle_blob); }

drb_status drb_rb_export_handle(drb_rb* h, void* blob, size_t* len) {
    DRB_REQUIRE(h && blob && len);
    if (*len < sizeof(handle_blob)) {
        t_last_error = "export_handle: blob buffer too small";
        *len = sizeof(handle_blob);
        return DRB_ERR_INVALID_ARGUMENT;
    }
    return guarded([&] {
        device_guard g(h->cfg.device);
        handle_blob b{};
        b.magic = kBlobMagic;
        b.version = 1;
        b.pid = int32_t(getpid());
        b.device = h->cfg.device;
        b.rank = h->cfg.rank;
        b.world = h->cfg.world;
        b.region_bytes = h->layout.bytes;
        b.region_ptr = reinterpret_cast<uint64_t>(h->region);
        b.slab_bytes = uint64_t(h->cfg.n_classes) * h->cfg.per_class_cap * h->cfg.sample_bytes;
        b.slab_ptr = reinterpret_cast<uint64_t>(h->slab);
        cuda_check(cudaIpcGetMemHandle(&b.ipc, h->region), "cudaIpcGetMemHandle");
        cuda_check(cudaIpcGetMemHandle(&b.slab_ipc, h->slab), "cudaIpcGetMemHandle (slab)");
        std::memcpy(blob, &b, sizeof b);
        *len = sizeof b;
    });
}

drb_status drb_rb_connect(drb_rb* h, const void* blobs, size_t blob_len) {
    DRB_REQUIRE(h && blobs);
    return guarded([&] {
        const auto& c = h->cfg;
        if (blob_len < sizeof(handle_blob) * c.world)
            fail(DRB_ERR_INVALID_ARGUMENT, "connect: need world blobs");
        if (h->started)
            fail(DRB_ERR_USAGE, "connect: engine already started");
        device_guard g(c.device);
        const auto* all = static_cast<const handle_blob*>(blobs);
        for (uint32_t w = 0; w < c.world; ++w) {
            const handle_blob& b = all[w];
            if (b.magic != kBlobMagic || b.rank != w || b.world != c.world ||
                b.region_bytes != h->layout.bytes)
                fail(DRB_ERR_CONFIG, "connect: blob " + std::to_string(w) + " does not match this configuration");
            if (w == c.rank)
                continue;
            if (b.pid == int32_t(getpid())) {
                if (b.device != c.device) {
                    int can = 0;
                    cuda_check(cudaDeviceCanAccessPeer(&can, c.device, b.device), "peer query");
                    if (!can)
                        fail(DRB_ERR_TRANSPORT, "connect: no peer access between devices");
                    const cudaError_t e = cudaDeviceEnablePeerAccess(b.device, 0);
                    if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled)
                        cuda_check(e, "cudaDeviceEnablePeerAccess");
                    cudaGetLastError();
                }
                h->peers[w] = reinterpret_cast<uint8_t*>(b.region_ptr);
                h->slab_peers[w] = reinterpret_cast<uint8_t*>(b.slab_ptr);
            } else {
                void* p = nullptr;
                cuda_check(cudaIpcOpenMemHandle(&p, b.ipc, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle");
                h->peers[w] = static_cast<uint8_t*>(p);
                h->peer_opened[w] = true;
                void* q = nullptr;
                cuda_check(cudaIpcOpenMemHandle(&q, b.slab_ipc, cudaIpcMemLazyEnablePeerAccess),
                           "cudaIpcOpenMemHandle (slab)");
                h->slab_peers[w] = static_cast<uint8_t*>(q);
                h->slab_opened[w] = true;
            }
        }
        h->connected = true;
    });
}

drb_status drb_rb_start(drb_rb* h) {
    DRB_REQUIRE(h);
    return guarded([&] {
        if (h->started)
            fail(DRB_ERR_USAGE, "engine: already started");
        if (!h->connected)
            fail(DRB_ERR_USAGE, "engine: multi-rank handle not connected");
        h->started = true;
        h->ver0 = h->ver - h->step;  // iteration i uses table version ver0 + i
        h->sel_par0 = h->cur_sel;
        h->plan_par0 = h->cur_plan;
        // Resident engine unless disabled (DRB_PERSIST=0), samples are not 16-byte rows (TMA
        // bulk copies) or the driver has no stream memory operations (its feed); the
        // three-kernel path serves those.
        h->rmode = h->use_persist && memops().ok && h->cfg.sample_bytes % 16 == 0 && h->sm_count >= 4 &&
                   run_smem_bytes(h->cfg.world, h->cfg.n_classes, h->cfg.rep_count, h->cfg.max_batch) <= 227u * 1024u;
        if (h->rmode) {
            device_guard g(h->cfg.device);
            RunCtl rc{};
            rc.sel_done = rc.plan_done = rc.b_done = rc.a_done = rc.admitted = rc.ready = h->step;
            rc.next_step[1] = h->step;  // the first instance is generation 1
            rc.next_desc[1] = 0;
            cuda_check(cudaMemcpy(h->runctl, &rc, sizeof rc, cudaMemcpyHostToDevice), "engine state");
            h->posted = 0;
            h->gen = 0;
            h->alive = false;
            h->released = h->step;
            *mb64(h, kMbHostPosted) = 0;
            *mb64(h, kMbExiting) = 0;
            *mb64(h, kMbDescDone) = 0;
            *mb64(h, kMbReady) = h->step;
            cuda_check(cudaMemset(h->feed_seq, 0, kFeedRing * 8), "feed reset");
        }
    });
}

drb_status drb_rb_shutdown(drb_rb* h) {
    DRB_REQUIRE(h);
    return guarded([&] {
        if (!h->started)
            fail(DRB_ERR_USAGE, "engine: shutdown before start");
        if (h->shut_down)
            fail(DRB_ERR_USAGE, "engine: double shutdown");
        h->shut_down = true;
        device_guard g(h->cfg.device);
        rmode_quiesce(h);  // the resident instance leaves once everything posted is done
        cuda_check(cudaDeviceSynchronize(), "shutdown drain");
        const bool failed = reinterpret_cast<volatile uint32_t*>(h->mailbox)[kMbSticky] != 0;
        if (h->rmode && h->cfg.world > 1 && h->step > 0 && !failed) {
            // Peers may still be pushing this rank's last reps into its m' ring (they run at
            // most a step behind): wait, bounded, for every peer's final announcement, so a
            // drb_rb_destroy after shutdown never frees memory a peer still writes. (Not after
            // a failure: a stalled peer never announces; the three-kernel path announces a
            // step late and keeps the old contract — shut down every rank before destroying.)
            const auto* hdr = reinterpret_cast<const RegionHeader*>(h->region);
            const auto t0 = std::chrono::steady_clock::now();
            for (;;) {
                uint64_t pd[kMaxWorld] = {};
                cuda_check(cudaMemcpy(pd, hdr->pushdone, sizeof pd, cudaMemcpyDeviceToHost), "peer drain");
                bool all = true;
                for (uint32_t w = 0; w < h->cfg.world; ++w)
                    if (w != h->cfg.rank && pd[w] < h->step)
                        all = false;
                if (all)
                    break;
                if (std::chrono::steady_clock::now() - t0 > std::chrono::nanoseconds(h->timeout_ns))
                    fail(DRB_ERR_TRANSPORT, "engine: shutdown: a peer did not finish its last step");
                std::this_thread::sleep_for(std::chrono::microseconds(50));
            }
        }
        h->alive = false;
    });
}

namespace {

// Parameters of engine iteration i (every slot / parity is a function of i, so the three
// kernels of an iteration may be issued at different times).
StepParams iter_params(drb_rb* h, uint64_t i, const void* batch, const uint32_t* labels, uint32_t n) {
    StepParams p = base_params(h);
    const uint64_t v = h->ver0 + i;
    p.tslot_in = uint32_t(v % kTableRing);
    p.tslot_out = uint32_t((v + 1) % kTableRing);
    p.sel_in = h->sel + ((h->sel_par0 + i) & 1);
    p.sel_out = h->sel + ((h->sel_par0 + i + 1) & 1);
    p.plan_in = h->plan + ((h->plan_par0 + i) & 1);
    p.plan_out = h->plan + ((h->plan_par0 + i + 1) & 1);
    p.n = n;
    p.batch = static_cast<const uint8_t*>(batch);
    p.labels = labels;
    p.step = i;
    p.seq = i;
    p.mode = kModeUpdate | kModeAssemble | kModePlan | kModePublish | (h->cfg.world > 1 ? kModePeers : 0u);
    p.aslot = uint32_t(i % h->aug_ring);
    const uint64_t pw = plist_words(h->cfg.world, h->cfg.rep_count);
    const uint64_t ww = wlist_words(h->cfg.max_batch);
    p.plist_in = h->plist + (i % kListRing) * pw;   // X_i, built by plan(i), read by copy(i)
    p.plist_out = h->plist + (i % kListRing) * pw;
    p.wlist = h->wlist + (i % kListRing) * ww;            // W_i
    p.vec16 = (p.S % 16 == 0) && (n == 0 || aligned16(batch));
    return p;
}

constexpr int kE = drb_rb::kEv;
inline int ev_of(uint64_t i) { return int(i % kE); }

// sel(i) on s_sel: table slot (i+1)%6 (own row v=i+1) free once plan(i-4) read it (a peer's
// plan(i-6) precedes its copy(i-6), which precedes my sel(i) through the rendezvous);
// optionally after the caller's prior work on `caller` (m_i produced, m'_{i-3} consumed).
void enqueue_sel(drb_rb* h, uint64_t i, const void* batch, const uint32_t* labels, uint32_t n,
                 cudaStream_t caller, bool wait_caller) {
    StepParams p = iter_params(h, i, batch, labels, n);
    if (wait_caller) {
        cuda_check(cudaEventRecord(h->ev_user[ev_of(i)], caller), "event");
        cuda_check(cudaStreamWaitEvent(h->s_sel, h->ev_user[ev_of(i)], 0), "wait");
    }
    // W slot i%8: copy(i-8) read it. Multi-rank: copy(i-6) complete before sel(i)
    // publishes — every plan(i) entry is pushed into an m' slot whose previous pushes
    // (reps(i-6), any owner) must have landed; each owner orders them before its own sel(i),
    // and plan(i) of every rank waits for all sel(i) rows. (One rank: stream order.)
    if (i >= h->dep_floor + kListRing)
        cuda_check(cudaStreamWaitEvent(h->s_sel, h->ev_copy[ev_of(i - kListRing)], 0), "wait");
    const uint32_t lag = std::min<uint32_t>(h->aug_ring, kTableRing);
    if (h->cfg.world > 1 && i >= h->dep_floor + lag)
        cuda_check(cudaStreamWaitEvent(h->s_sel, h->ev_copy[ev_of(i - lag)], 0), "wait");
    if (i >= h->dep_floor + 4)
        cuda_check(cudaStreamWaitEvent(h->s_sel, h->ev_plan[ev_of(i - 4)], 0), "wait");
    if (launch_sel(p, h->s_sel, h->use_pdl && (h->dbg_bits & 256)))  // DRB_DBG bit 8: PDL sel chain
        fail(DRB_ERR_INTERNAL, std::string("sel launch failed: ") + cudaGetErrorString(cudaGetLastError()));
    cuda_check(cudaEventRecord(h->ev_sel[ev_of(i)], h->s_sel), "event");
    h->ver = h->ver0 + i + 1;
    h->cur_sel = uint32_t((h->sel_par0 + i + 1) & 1);
}

// plan(i) on s_plan: own row v=i+1 from sel(i); X slot i%8 free once copy(i-8) read it.
void enqueue_plan(drb_rb* h, uint64_t i) {
    StepParams p = iter_params(h, i, nullptr, nullptr, 0);
    cuda_check(cudaStreamWaitEvent(h->s_plan, h->ev_sel[ev_of(i)], 0), "wait");
    if (i >= h->dep_floor + kListRing)
        cuda_check(cudaStreamWaitEvent(h->s_plan, h->ev_copy[ev_of(i - kListRing)], 0), "wait");
    if (launch_plan_next(p, h->s_plan, h->use_pdl && (h->dbg_bits & 256)))
        fail(DRB_ERR_INTERNAL, std::string("plan launch failed: ") + cudaGetErrorString(cudaGetLastError()));
    cuda_check(cudaEventRecord(h->ev_plan[ev_of(i)], h->s_plan), "event");
    h->cur_plan = uint32_t((h->plan_par0 + i + 1) & 1);
}

// copy(i) on `s`: W_i from sel(i), X_i from plan(i), slab writes of round i-1 and the reps
// rows of m'_i from copy(i-1).
// prewait_next (inside a run, with copy(i+1) to follow on `s`): s also waits here for
// sel(i+1) / plan(i+1), so copy(i+1)'s only new dependency is copy(i) itself — the edge a
// programmatic (PDL) launch can overlap (sel/plan run iterations ahead; this costs nothing).
// batch_ready: the caller's event after m_i was produced (single steps run their copies on
// the handle's own stream). ready_wait: multi-rank single steps follow the copy with
// peers_wait(i) on s_wait; done[slot] ("m'_i ready") is recorded after it.
void enqueue_copy(drb_rb* h, uint64_t i, const void* batch, const uint32_t* labels, uint32_t n,
                  cudaStream_t s, bool first_of_run, drb_aug* out, cudaEvent_t ev_begin = nullptr,
                  cudaEvent_t ev_end = nullptr, bool prewait_next = false, cudaEvent_t batch_ready = nullptr,
                  bool ready_wait = false) {
    StepParams p = iter_params(h, i, batch, labels, n);
    if (batch_ready)
        cuda_check(cudaStreamWaitEvent(s, batch_ready, 0), "wait");
    if (h->trace) {
        cuda_check(cudaMemsetAsync(h->trace, 0, 32 * 8, s), "trace reset");
        cuda_check(cudaMemsetAsync(h->trace + 14, 0xff, 8, s), "trace reset");
        cuda_check(cudaMemsetAsync(h->trace + 21, 0xff, 16, s), "trace reset");
    }
    const bool prewaited = !first_of_run && h->prewaited == i + 1 && s == h->last_copy_stream;
    if (!prewaited) {
        cuda_check(cudaStreamWaitEvent(s, h->ev_sel[ev_of(i)], 0), "wait");
        cuda_check(cudaStreamWaitEvent(s, h->ev_plan[ev_of(i)], 0), "wait");
    }
    if (prewait_next) {
        cuda_check(cudaStreamWaitEvent(s, h->ev_sel[ev_of(i + 1)], 0), "wait");
        cuda_check(cudaStreamWaitEvent(s, h->ev_plan[ev_of(i + 1)], 0), "wait");
    }
    h->prewaited = prewait_next ? i + 2 : 0;  // (i+1) + 1: 0 means none
    const bool have1 = i >= h->dep_floor + 1;
    // PDL only between this handle's own consecutive copies inside one run: the copy's
    // pre-wait prologue reads m_i, which must not be the output of an arbitrary predecessor.
    const bool pdl = h->use_pdl && !first_of_run && s == h->last_copy_stream && have1;
    if (have1 && s != h->last_copy_stream)
        cuda_check(cudaStreamWaitEvent(s, h->ev_copy[ev_of(i - 1)], 0), "wait");
    // timing events after every dependency: they bracket the copy kernel alone. External
    // records stay real (timeable) records when captured into a graph.
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    cuda_check(cudaStreamIsCapturing(s, &cap), "capture query");
    const unsigned rec_flags = cap == cudaStreamCaptureStatusActive ? cudaEventRecordExternal : 0u;
    if (ev_begin)
        cuda_check(cudaEventRecordWithFlags(ev_begin, s, rec_flags), "event");
    if (launch_copy(p, h->grid, s, pdl))
        fail(DRB_ERR_INTERNAL, std::string("copy launch failed: ") + cudaGetErrorString(cudaGetLastError()));
    if (ev_end)
        cuda_check(cudaEventRecordWithFlags(ev_end, s, rec_flags), "event");
    cuda_check(cudaEventRecord(h->ev_copy[ev_of(i)], s), "event");
    if (cap != cudaStreamCaptureStatusActive) {
        cuda_check(cudaEventRecord(h->last_work, s), "event");
        h->last_work_valid = true;
    }
    if (ready_wait && (p.mode & kModePeers) && i > 0) {
        cuda_check(cudaStreamWaitEvent(h->s_wait, h->ev_copy[ev_of(i)], 0), "wait");
        if (launch_peers_wait(p, h->s_wait))
            fail(DRB_ERR_INTERNAL, std::string("peers_wait launch failed: ") + cudaGetErrorString(cudaGetLastError()));
        cuda_check(cudaEventRecord(h->done[p.aslot], h->s_wait), "event record");
        h->slot_run[p.aslot] = 0;
    } else {
        cuda_check(cudaEventRecord(h->done[p.aslot], s), "event record");
        h->slot_run[p.aslot] = 0;
    }
    h->last_copy_stream = s;
    if (out) {
        out->n = n;
        out->ring_slot = p.aslot;
        out->step = i;
        const uint32_t row0 = h->cfg.max_batch - n;
        out->data = h->region + h->layout.off_aug + uint64_t(p.aslot) * h->layout.aug_slot_bytes +
                    uint64_t(row0) * h->cfg.sample_bytes;
        out->labels = reinterpret_cast<uint32_t*>(h->region + h->layout.off_auglab) +
                      uint64_t(p.aslot) * p.auglab_slot_elems + row0;
    }
    h->step = i + 1;
}

// Host view of the state after h->step iterations (table version, state parities), as the
// three-kernel path keeps it (snapshot, device_error, read_slots read it).
void rmode_advance(drb_rb* h) {
    h->ver = h->ver0 + h->step;
    h->cur_sel = uint32_t((h->sel_par0 + h->step) & 1);
    h->cur_plan = uint32_t((h->plan_par0 + h->step) & 1);
}

// One step through the resident engine: post m_i's descriptor on `s`, then `s`
// waits for "m'_i ready". An unaligned device batch is first copied into a staging slot.
void rmode_step(drb_rb* h, const void* batch, const uint32_t* labels, uint32_t n, cudaStream_t s, drb_aug* out,
                cudaStream_t consumer = nullptr) {
    const uint64_t i = h->step;
    const auto& c = h->cfg;
    const uint8_t* b = static_cast<const uint8_t*>(batch);
    if (n > 0 && !aligned16(batch)) {
        constexpr uint32_t kStage = 4;
        if (!h->astage)
            cuda_check(cudaMalloc(&h->astage, uint64_t(kStage) * c.max_batch * c.sample_bytes), "stage alloc");
        if (i >= kStage)  // the slot's previous batch (step i-4) is no longer read
            rmode_wait(h, i - kStage + 1, s);
        uint8_t* slot = h->astage + (i % kStage) * uint64_t(c.max_batch) * c.sample_bytes;
        cuda_check(cudaMemcpyAsync(slot, batch, uint64_t(n) * c.sample_bytes, cudaMemcpyDeviceToDevice, s), "stage");
        b = slot;
    }
    const uint32_t slot = uint32_t(i % h->aug_ring);
    if (!consumer) {  // one stream: posting m_i releases every earlier m'; then wait for m'_i
        rmode_post(h, b, 0, labels, 0, 1, 0, n, i, 1, s, i + 1, false, true);
    } else {  // producer / consumer streams: the consumer releases what it used, then waits
        rmode_post(h, b, 0, labels, 0, 1, 0, n, i, 1, s, 0, true);
        // the release of consumed m' every `release_every` steps (each stream memory operation
        // costs the consumer stream time; the ring keeps aug_ring - 2 - release_every steps of
        // run-ahead), then the wait for m'_i
        const bool rel = i >= h->released + h->release_every;
        if (rel)
            h->released = i;
        {
            CUstreamBatchMemOpParams ops[2];
            std::memset(ops, 0, sizeof ops);
            uint32_t nop = 0;
            if (rel) {
                ops[nop].writeValue.operation = CU_STREAM_MEM_OP_WRITE_VALUE_64;
                ops[nop].writeValue.address = reinterpret_cast<CUdeviceptr>(&h->runctl->consumed);
                ops[nop].writeValue.value64 = i;  // m'_0 .. m'_{i-1}: everything the consumer was handed
                ops[nop].writeValue.flags = CU_STREAM_WRITE_VALUE_DEFAULT;
                ++nop;
            }
            ops[nop].waitValue.operation = CU_STREAM_MEM_OP_WAIT_VALUE_64;
            ops[nop].waitValue.address = reinterpret_cast<CUdeviceptr>(&h->runctl->ready);
            ops[nop].waitValue.value64 = i + 1;
            ops[nop].waitValue.flags = CU_STREAM_WAIT_VALUE_GEQ;
            ++nop;
            const CUresult r = memops().batch(reinterpret_cast<CUstream>(consumer), nop, ops, 0);
            if (r != CUDA_SUCCESS)
                fail(DRB_ERR_INTERNAL, "consumer wait: cuStreamBatchMemOp failed (" + std::to_string(int(r)) + ")");
        }
    }
    const uint32_t row0 = c.max_batch - n;
    out->n = n;
    out->ring_slot = slot;
    out->step = i;
    out->data = h->region + h->layout.off_aug + uint64_t(slot) * h->layout.aug_slot_bytes + uint64_t(row0) * c.sample_bytes;
    out->labels = reinterpret_cast<uint32_t*>(h->region + h->layout.off_auglab) +
                  uint64_t(slot) * (align_up(h->layout.rows * 4, 256) / 4) + row0;
    h->step = i + 1;
    rmode_advance(h);
}

// `steps` steps over a device ring through the resident engine: one descriptor per 2^31
// steps, then `s` waits until the last m' is ready.
void rmode_run(drb_rb* h, const uint8_t* batches, uint64_t batch_stride, const uint32_t* labels,
               uint64_t label_stride, uint32_t ring, uint32_t n, uint64_t steps, uint64_t first, cudaStream_t s) {
    // The run's last step goes out as its own early-ready descriptor: the stream's wait then ends
    // when m'_{end-1} is complete, without waiting for B(end-1) (which sources its winners
    // from m'_{end-1}, so the caller's ring is free once the wait is over).
    const uint64_t body = steps - 1;
    uint64_t done = 0;
    // DRB_RUN_CHUNK: steps per descriptor (experiments: the per-descriptor cost of the feed)
    static const uint64_t chunk = std::getenv("DRB_RUN_CHUNK") ? std::max<uint64_t>(1, std::strtoull(std::getenv("DRB_RUN_CHUNK"), nullptr, 10)) : (1ull << 31);
    while (done < body) {
        const uint32_t cnt = uint32_t(std::min<uint64_t>(body - done, chunk));
        rmode_post(h, batches, batch_stride, labels, label_stride, ring, uint32_t((first + done) % ring), n,
                   h->step, cnt, s);
        h->step += cnt;
        done += cnt;
    }
    rmode_post(h, batches, batch_stride, labels, label_stride, ring, uint32_t((first + done) % ring), n, h->step, 1, s,
               h->step + 1, false, true);
    h->step += 1;
    // one event for the whole run (its m' ring slots alias it): the host cost of recording
    // R events would sit inside a timed run
    cuda_check(cudaEventRecord(h->run_done, s), "event");
    for (auto& f : h->slot_run)
        f = 1;
    rmode_advance(h);
}

void check_step_args(drb_rb* h, uint32_t n) {
    if (h->shut_down)
        fail(DRB_ERR_USAGE, "engine: update after shutdown");
    if (!h->started)
        fail(DRB_ERR_USAGE, "engine: update before start");
    if (n > h->cfg.max_batch)
        fail(DRB_ERR_USAGE, "engine: batch larger than max_batch");
    check_engine_alive(h);
}

}  // namespace

drb_status drb_rb_step(drb_rb* h, const void* batch, const uint32_t* labels, uint32_t n,
                       void* stream, drb_aug* out) {
    DRB_REQUIRE(h && out && ((batch && labels) || n == 0));
    return guarded([&] {
        check_step_args(h, n);
        device_guard g(h->cfg.device);
        cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : h->stream;
        if (h->rmode) {
            rmode_step(h, batch, labels, n, s, out);
            return;
        }
        const uint64_t i = h->step;
        enqueue_sel(h, i, batch, labels, n, s, true);
        enqueue_plan(h, i);
        // the copies run on the handle's stream, one behind the other (PDL: copy(i)'s batch
        // part overlaps copy(i-1)'s tail); the caller's stream waits for "m'_i ready"
        const bool chained = h->last_copy_stream == h->stream && i >= h->dep_floor + 1;
        enqueue_copy(h, i, batch, labels, n, h->stream, !chained, out, nullptr, nullptr, false,
                     h->ev_user[ev_of(i)], true);
        if (s != h->stream || h->cfg.world > 1)
            cuda_check(cudaStreamWaitEvent(s, h->done[i % h->aug_ring], 0), "wait");
    });
}

drb_status drb_rb_step_split(drb_rb* h, const void* batch, const uint32_t* labels, uint32_t n, void* producer,
                             void* consumer, drb_aug* out) {
    DRB_REQUIRE(h && out && consumer && ((batch && labels) || n == 0));
    return guarded([&] {
        check_step_args(h, n);
        device_guard g(h->cfg.device);
        cudaStream_t sp = producer ? static_cast<cudaStream_t>(producer) : h->stream;
        cudaStream_t sc = static_cast<cudaStream_t>(consumer);
        if (h->rmode) {
            rmode_step(h, batch, labels, n, sp, out, sc);
            return;
        }
        // three-kernel path: a release event per call on the consumer (its use of every m'
        // handed out before); step i refills m'_{i+1-R}'s slot, so the producer waits for the
        // release recorded at call i+2-R (a more recent one for rings deeper than the events)
        const uint64_t i = h->step;
        cuda_check(cudaEventRecord(h->rel[i % drb_rb::kEv], sc), "event");
        const uint64_t R = h->aug_ring;
        if (i + 2 >= R) {
            const uint64_t k = std::max<uint64_t>(i + 2 - R, i + 1 >= drb_rb::kEv ? i + 1 - drb_rb::kEv : 0);
            cuda_check(cudaStreamWaitEvent(sp, h->rel[k % drb_rb::kEv], 0), "wait");
        }
        const drb_status st = drb_rb_step(h, batch, labels, n, sp, out);
        if (st != DRB_OK)
            fail(st, t_last_error);
        cuda_check(cudaStreamWaitEvent(sc, h->done[out->ring_slot], 0), "wait");
    });
}

drb_status drb_rb_run(drb_rb* h, const void* batches, uint64_t batch_stride, const uint32_t* labels,
                      uint64_t label_stride, uint32_t ring, uint32_t n, uint64_t steps, uint64_t first,
                      void* stream, void* const* step_events) {
    DRB_REQUIRE(h && batches && labels && ring > 0);
    return guarded([&] {
        check_step_args(h, n);
        device_guard g(h->cfg.device);
        cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : h->stream;
        const auto* b = static_cast<const uint8_t*>(batches);
        auto bat = [&](uint64_t k) { return b + ((first + k) % ring) * batch_stride; };
        auto lab = [&](uint64_t k) { return labels + ((first + k) % ring) * label_stride; };
        const uint64_t i0 = h->step, end = i0 + steps;
        if (steps == 0)
            return;
        const bool vec = (h->cfg.sample_bytes % 16 == 0) && aligned16(batches) && (batch_stride % 16 == 0);
        h->last_run_persistent = false;
        if (h->rmode) {
            if (step_events)
                fail(DRB_ERR_USAGE, "run: per-step copy events exist only on the three-kernel path (DRB_PERSIST=0)");
            if (vec) {
                rmode_run(h, b, batch_stride, labels, label_stride, ring, n, steps, first, s);
            } else {  // unaligned ring: step by step through the staging copy
                drb_aug aug{};
                for (uint64_t k = 0; k < steps; ++k)
                    rmode_step(h, bat(k), lab(k), n, s, &aug);
            }
            return;
        }
        // Skewed issue order (software pipeline over a resident input ring): sel runs two
        // iterations ahead, plan one, so neither chain waits behind a copy in launch order.
        // Only the first iteration waits for the caller's prior work.
        enqueue_sel(h, i0, bat(0), lab(0), n, s, true);
        if (i0 + 1 < end)
            enqueue_sel(h, i0 + 1, bat(1), lab(1), n, s, false);
        enqueue_plan(h, i0);
        for (uint64_t i = i0; i < end; ++i) {
            if (i + 2 < end)
                enqueue_sel(h, i + 2, bat(i + 2 - i0), lab(i + 2 - i0), n, s, false);
            if (i + 1 < end)
                enqueue_plan(h, i + 1);
            enqueue_copy(h, i, bat(i - i0), lab(i - i0), n, s, i == i0, nullptr,
                         step_events ? static_cast<cudaEvent_t>(step_events[2 * (i - i0)]) : nullptr,
                         step_events ? static_cast<cudaEvent_t>(step_events[2 * (i - i0) + 1]) : nullptr,
                         h->use_pdl && !(h->dbg_bits & 32) && i + 1 < end);
        }
    });
}

}  // extern "C"

struct drb_rb_graph {
    drb_rb* h = nullptr;
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    bool launched = false;
    // resident engine: nothing to capture (a run is one descriptor post and one stream wait,
    // no launches); launch() posts the run
    bool deferred = false;
    const void* batches = nullptr;
    const uint32_t* labels = nullptr;
    uint64_t batch_stride = 0, label_stride = 0, steps = 0, first = 0;
    uint32_t ring = 0, n = 0;
};

extern "C" {

drb_status drb_rb_graph_prepare(drb_rb* h, const void* batches, uint64_t batch_stride,
                                const uint32_t* labels, uint64_t label_stride, uint32_t ring,
                                uint32_t n, uint64_t steps, uint64_t first, void* const* step_events,
                                drb_rb_graph** out) {
    DRB_REQUIRE(h && batches && labels && ring > 0 && out);
    *out = nullptr;
    return guarded([&] {
        device_guard g(h->cfg.device);
        auto gr = std::make_unique<drb_rb_graph>();
        gr->h = h;
        if (h->rmode) {
            check_step_args(h, n);
            if (step_events)
                fail(DRB_ERR_USAGE, "graph_prepare: per-step copy events exist only on the three-kernel path");
            gr->deferred = true;
            gr->batches = batches;
            gr->labels = labels;
            gr->batch_stride = batch_stride;
            gr->label_stride = label_stride;
            gr->steps = steps;
            gr->first = first;
            gr->ring = ring;
            gr->n = n;
            *out = gr.release();
            return;
        }
        // everything issued so far completes first, so the captured steps depend only on
        // each other (no waits on events recorded outside the capture)
        rmode_quiesce(h);
        cuda_check(cudaDeviceSynchronize(), "capture prologue");
        h->dep_floor = h->step;
        cudaStream_t cs = nullptr;
        cuda_check(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking), "capture stream");
        cuda_check(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal), "begin capture");
        drb_status st = drb_rb_run(h, batches, batch_stride, labels, label_stride, ring, n, steps,
                                   first, cs, step_events);
        const std::string err = t_last_error;
        if (st == DRB_OK && steps > 0 && !h->last_run_persistent) {  // join the forked sel/plan streams
            const int e = int((h->step - 1) % drb_rb::kEv);
            if (cudaStreamWaitEvent(cs, h->ev_plan[e], 0) != cudaSuccess)
                st = DRB_ERR_INTERNAL;
        }
        const cudaError_t ce = cudaStreamEndCapture(cs, &gr->graph);
        cudaStreamDestroy(cs);
        if (st != DRB_OK)
            fail(st, err);
        cuda_check(ce, "end capture");
        if (const char* dot = std::getenv("DRB_GRAPH_DOT"))  // diagnostics: the captured DAG
            cudaGraphDebugDotPrint(gr->graph, dot, cudaGraphDebugDotFlagsVerbose);
        cuda_check(cudaGraphInstantiate(&gr->exec, gr->graph, 0), "graph instantiate");
        // upload now: the first launch of a never-uploaded graph pays the upload inside it
        cuda_check(cudaGraphUpload(gr->exec, h->stream), "graph upload");
        cuda_check(cudaStreamSynchronize(h->stream), "graph upload");
        // events recorded during the capture are graph-internal: later steps must not wait
        // on them (graph_launch orders the handle's streams after the whole graph instead)
        h->dep_floor = h->step;
        *out = gr.release();
    });
}

drb_status drb_rb_graph_launch(drb_rb_graph* g, void* stream) {
    DRB_REQUIRE(g);
    return guarded([&] {
        if (g->launched)
            fail(DRB_ERR_USAGE, "graph_launch: a prepared run can be launched once");
        device_guard dg(g->h->cfg.device);
        cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : g->h->stream;
        if (g->deferred) {
            const drb_status st = drb_rb_run(g->h, g->batches, g->batch_stride, g->labels, g->label_stride, g->ring,
                                             g->n, g->steps, g->first, s, nullptr);
            if (st != DRB_OK)
                fail(st, t_last_error);
            g->launched = true;
            return;
        }
        cuda_check(cudaGraphLaunch(g->exec, s), "graph launch");
        cuda_check(cudaEventRecord(g->h->ev_user[0], s), "event");
        cuda_check(cudaEventRecord(g->h->last_work, s), "event");
        g->h->last_work_valid = true;
        for (auto& e : g->h->done)
            cuda_check(cudaEventRecord(e, s), "event");
        for (cudaStream_t o : {g->h->stream, g->h->s_sel, g->h->s_plan})
            if (o != s)
                cuda_check(cudaStreamWaitEvent(o, g->h->ev_user[0], 0), "wait");
        g->launched = true;
    });
}

drb_status drb_rb_graph_destroy(drb_rb_graph* g) {
    if (!g)
        return DRB_OK;
    return guarded([&] {
        device_guard dg(g->h->cfg.device);
        if (g->exec)
            cudaGraphExecDestroy(g->exec);
        if (g->graph)
            cudaGraphDestroy(g->graph);
        delete g;
    });
}

drb_status drb_rb_step_host(drb_rb* h, const void* batch, const uint32_t* labels, uint32_t n,
                            void* out, uint32_t* out_labels, uint32_t* out_count) {
    DRB_REQUIRE(h && out && out_labels && out_count && ((batch && labels) || n == 0));
    return guarded([&] {
        if (n > h->cfg.max_batch)
            fail(DRB_ERR_USAGE, "engine: batch larger than max_batch");
        device_guard g(h->cfg.device);
        const auto& c = h->cfg;
        if (!h->stage) {
            cuda_check(cudaMalloc(&h->stage, 2ull * c.max_batch * c.sample_bytes), "stage alloc");
            cuda_check(cudaMalloc(&h->stage_labels, 2ull * c.max_batch * 4), "stage alloc");
        }
        // Input copy on its own stream into a 2-deep staging ring so the copy of m_{i+1}
        // overlaps step i; the output copy of m'_i runs on a third stream (PCIe is duplex).
        const uint32_t si = uint32_t(h->step & 1);
        uint8_t* st_b = h->stage + uint64_t(si) * c.max_batch * c.sample_bytes;
        uint32_t* st_l = h->stage_labels + uint64_t(si) * c.max_batch;
        cuda_check(cudaStreamWaitEvent(h->h2d, h->in_free[si], 0), "wait");
        cuda_check(cudaMemcpyAsync(st_b, batch, uint64_t(n) * c.sample_bytes, cudaMemcpyHostToDevice, h->h2d), "h2d");
        cuda_check(cudaMemcpyAsync(st_l, labels, uint64_t(n) * 4, cudaMemcpyHostToDevice, h->h2d), "h2d");
        cuda_check(cudaEventRecord(h->h2d_done[si], h->h2d), "event");
        cuda_check(cudaStreamWaitEvent(h->stream, h->h2d_done[si], 0), "wait");
        drb_aug aug{};
        const drb_status st = drb_rb_step(h, st_b, st_l, n, h->stream, &aug);
        if (st != DRB_OK)
            fail(st, t_last_error);
        if (h->rmode)  // (the resident step records no event: the copy-out orders behind this one)
            cuda_check(cudaEventRecord(h->done[aug.ring_slot], h->stream), "event record");
        cuda_check(cudaEventRecord(h->in_free[si], h->stream), "event");
        cuda_check(cudaStreamWaitEvent(h->d2h, h->done[aug.ring_slot], 0), "wait");
        // in place: the caller's batch rows already are m'_i's first n rows; only the
        // representatives (at most r rows, fixed offset n) travel back
        const bool in_place = out == batch && out_labels == labels;
        const uint64_t skip = in_place ? n : 0;
        const uint64_t rows = uint64_t(n) + c.rep_count - skip;
        cuda_check(cudaMemcpyAsync(static_cast<uint8_t*>(out) + skip * c.sample_bytes,
                                   static_cast<const uint8_t*>(aug.data) + skip * c.sample_bytes,
                                   rows * c.sample_bytes, cudaMemcpyDeviceToHost, h->d2h), "d2h");
        cuda_check(cudaMemcpyAsync(out_labels + skip, aug.labels + skip, rows * 4, cudaMemcpyDeviceToHost, h->d2h),
                   "d2h");
        const auto* counts = reinterpret_cast<const uint32_t*>(h->region + h->layout.off_counts);
        cuda_check(cudaMemcpyAsync(out_count, counts + aug.ring_slot, 4, cudaMemcpyDeviceToHost, h->d2h), "d2h");
        // The next step may reuse this m' slot only after the copy-out drained.
        cuda_check(cudaEventRecord(h->done[aug.ring_slot], h->d2h), "event");
        cuda_check(cudaStreamWaitEvent(h->stream, h->done[aug.ring_slot], 0), "wait");
    });
}

drb_status drb_rb_aug_slot(drb_rb* h, uint64_t step, uint32_t n, drb_aug* out) {
    DRB_REQUIRE(h && out);
    return guarded([&] {
        if (n > h->cfg.max_batch)
            fail(DRB_ERR_USAGE, "aug_slot: batch larger than max_batch");
        if (step >= h->step || h->step - step > h->aug_ring)
            fail(DRB_ERR_USAGE, "aug_slot: step " + std::to_string(step) + " is not among the last " +
                                    std::to_string(h->aug_ring) + " enqueued steps");
        const uint32_t slot = uint32_t(step % h->aug_ring);
        const uint32_t row0 = h->cfg.max_batch - n;
        out->n = n;
        out->ring_slot = slot;
        out->step = step;
        out->data = h->region + h->layout.off_aug + uint64_t(slot) * h->layout.aug_slot_bytes +
                    uint64_t(row0) * h->cfg.sample_bytes;
        out->labels = reinterpret_cast<uint32_t*>(h->region + h->layout.off_auglab) +
                      uint64_t(slot) * (align_up(h->layout.rows * 4, 256) / 4) + row0;
    });
}

drb_status drb_rb_aug_count(drb_rb* h, const drb_aug* aug, uint32_t* count) {
    DRB_REQUIRE(h && aug && count);
    return guarded([&] {
        device_guard g(h->cfg.device);
        const auto t0 = std::chrono::steady_clock::now();
        if (h->rmode) {  // the ready publisher mirrors `ready` into host memory: no event per step
            while (*mb64(h, kMbReady) < aug->step + 1) {
                if (reinterpret_cast<volatile uint32_t*>(h->mailbox)[kMbSticky])
                    break;
                std::this_thread::yield();
            }
        } else {
            cuda_check(cudaEventSynchronize(h->slot_run[aug->ring_slot] ? h->run_done : h->done[aug->ring_slot]),
                       "aug wait");
        }
        h->wait_ms += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
        const volatile uint32_t* mb = h->mailbox;
        // `ready` first: the ready publisher writes a slot's error word before it publishes
        // `ready` (failed or not), so an error of this step is visible once `ready` covers it
        const uint64_t rd = h->rmode ? *mb64(h, kMbReady) : ~0ull;
        std::atomic_thread_fence(std::memory_order_acquire);
        const uint32_t e = mb[mb_err(aug->ring_slot, h->aug_ring)];
        *count = mb[mb_count(aug->ring_slot)];
        if (rd < aug->step + 1 || (h->rmode && rd >= kReadyFailed && aug->step >= *mb64(h, kMbFailedAt)))
            fail(DRB_ERR_TRAINING, "engine: round failed with status " + std::to_string(mb[kMbSticky]));
        if (e)
            fail(DRB_ERR_TRAINING, "engine: round failed with status " + std::to_string(e));
    });
}

drb_status drb_rb_synchronize(drb_rb* h) {
    DRB_REQUIRE(h);
    return guarded([&] {
        device_guard g(h->cfg.device);
        if (h->dbg_bits & 1024) {  // diagnostics of the last persistent run
            rmode_quiesce(h);
            cudaDeviceSynchronize();
            RunCtl rc{};
            cudaMemcpy(&rc, h->runctl, sizeof rc, cudaMemcpyDeviceToHost);
            std::fprintf(stderr, "drb run: sel %llu plan %llu b %llu error %u where site %u k %u check %u/%u first k %u\n",
                         (unsigned long long)rc.sel_done, (unsigned long long)rc.plan_done,
                         (unsigned long long)rc.b_done, rc.error, rc.where >> 24, rc.where & 0xffffff,
                         rc.pad[0], rc.pad[2], rc.pad[1]);
            if (h->prof) {
                unsigned long long pr[64];
                cudaMemcpy(pr, h->prof, sizeof pr, cudaMemcpyDeviceToHost);
                for (int c = 0; c < 2; ++c) {
                    const double it = pr[32 * c + 31] ? double(pr[32 * c + 31]) : 1.0;
                    std::fprintf(stderr, "drb prof CTA %d (%llu iterations), cycles/iteration by stamp:", c,
                                 (unsigned long long)pr[32 * c + 31]);
                    for (int x = 0; x < 31; ++x)
                        if (pr[32 * c + x])
                            std::fprintf(stderr, " [%d] %.0f", x, double(pr[32 * c + x]) / it);
                    std::fprintf(stderr, "\n");
                }
            }
        }
        if (h->rmode)  // every posted step's m' ready (the streams that posted them progressed)
            while (*mb64(h, kMbReady) < h->step && !reinterpret_cast<volatile uint32_t*>(h->mailbox)[kMbSticky])
                std::this_thread::yield();
        cuda_check(cudaStreamSynchronize(h->stream), "sync");
        cuda_check(cudaStreamSynchronize(h->s_sel), "sync");
        cuda_check(cudaStreamSynchronize(h->s_plan), "sync");
        cuda_check(cudaStreamSynchronize(h->h2d), "sync");
        cuda_check(cudaStreamSynchronize(h->d2h), "sync");
        for (auto e : h->done)
            cuda_check(cudaEventSynchronize(e), "sync");
        cuda_check(cudaEventSynchronize(h->run_done), "sync");
    });
}

drb_status drb_rb_drain_timings(drb_rb* h, drb_timing* out, uint32_t capacity, uint32_t* count) {
    DRB_REQUIRE(h && count && (out || capacity == 0));
    return guarded([&] {
        *count = 0;
        if (!h->timings || !h->rmode)  // (the three-kernel path records no timings)
            return;
        device_guard g(h->cfg.device);
        rmode_quiesce(h);
        cuda_check(cudaDeviceSynchronize(), "timings order");
        std::vector<uint64_t> t(uint64_t(kTimingRing) * kTimingWords);
        cuda_check(cudaMemcpy(t.data(), h->timings, t.size() * 8, cudaMemcpyDeviceToHost), "timings copy");
        uint64_t i = std::max<uint64_t>(h->timings_drained, h->step > kTimingRing ? h->step - kTimingRing : 0);
        uint32_t n = 0;
        for (; i < h->step && n < capacity; ++i) {
            const uint64_t* r = t.data() + (i % kTimingRing) * kTimingWords;
            auto ms = [](uint64_t a, uint64_t b) { return b >= a && a ? double(b - a) / 1e6 : 0.0; };
            drb_timing& o = out[n++];
            o.iteration = i;
            o.populate_ms = ms(r[1], r[2]);
            o.augment_ms = ms(r[3], r[4]);
            o.latency_ms = ms(r[0], r[4]);
            o.wait_ms = 0.0;
            o.degraded = 0;
            o.pad = 0;
        }
        h->timings_drained = i;
        *count = n;
    });
}

drb_status drb_rb_total_wait_ms(drb_rb* h, double* out) {
    DRB_REQUIRE(h && out);
    *out = h->wait_ms;
    return DRB_OK;
}

drb_status drb_rb_engine_counters(drb_rb* h, uint64_t* iterations, uint64_t* queue_depth, uint64_t* degraded_rounds,
                                  uint64_t* replanned_entries) {
    DRB_REQUIRE(h);
    return guarded([&] {
        device_guard g(h->cfg.device);
        uint64_t pending = 0;  // enqueued rounds whose m' is not ready yet (a non-blocking look)
        if (h->rmode) {
            const uint64_t rd = *mb64(h, kMbReady);
            pending = rd >= kReadyFailed ? 0 : h->step - std::min(h->step, rd);
        } else if (!h->done.empty()) {
            const uint64_t R = h->done.size();
            for (uint64_t x = h->step > R ? h->step - R : 0; x < h->step; ++x)
                pending += cudaEventQuery(h->done[x % R]) == cudaErrorNotReady ? 1 : 0;
            cudaGetLastError();
        }
        if (iterations)
            *iterations = h->step;
        if (queue_depth)
            *queue_depth = pending;
        if (degraded_rounds)  // fail-stop: a round completes on the exact view or fails the engine
            *degraded_rounds = 0;
        if (replanned_entries)  // every owner is reachable over peer memory: nothing is re-planned
            *replanned_entries = 0;
    });
}

drb_status drb_rb_broadcast_sizes(drb_rb* h) {
    DRB_REQUIRE(h);
    // Every round's sel already stored this rank's occupancy row (version i+1) into every
    // peer's table as self-validating words, so the freshest row is always published; the
    // reference's re-broadcast at task boundaries (engine.cpp:256-265) has nothing to resend.
    return DRB_OK;
}

drb_status drb_rb_device_error(drb_rb* h, uint32_t* out) {
    DRB_REQUIRE(h && out);
    return guarded([&] {
        device_guard g(h->cfg.device);
        SelState st{};
        PlanState pst{};
        rmode_quiesce(h);
        cuda_check(cudaDeviceSynchronize(), "order");
        cuda_check(cudaMemcpy(&st, h->sel + h->cur_sel, sizeof st, cudaMemcpyDeviceToHost), "state");
        cuda_check(cudaMemcpy(&pst, h->plan + h->cur_plan, sizeof pst, cudaMemcpyDeviceToHost), "state");
        // the mailbox's sticky word first: the resident engine stops at the failing role, so the
        // state parity the host expects after its posted steps may predate the failure
        const uint32_t sticky = reinterpret_cast<volatile uint32_t*>(h->mailbox)[kMbSticky];
        *out = sticky ? sticky : (st.error ? st.error : pst.error);
    });
}

drb_status drb_rb_trace_read(drb_rb* h, uint64_t* out16) {
    DRB_REQUIRE(h && out16);
    return guarded([&] {
        if (!h->trace)
            fail(DRB_ERR_USAGE, "trace_read: run with DRB_TRACE=1");
        device_guard g(h->cfg.device);
        rmode_quiesce(h);
        cuda_check(cudaDeviceSynchronize(), "trace sync");
        cuda_check(cudaMemcpy(out16, h->trace, 32 * 8, cudaMemcpyDeviceToHost), "trace copy");
    });
}

drb_status drb_rb_timeline_read(drb_rb* h, uint64_t* out, uint32_t* steps) {
    DRB_REQUIRE(h && steps);
    return guarded([&] {
        *steps = h->timeline_steps;
        if (!h->timeline || !out)
            return;
        device_guard g(h->cfg.device);
        rmode_quiesce(h);
        cuda_check(cudaDeviceSynchronize(), "timeline sync");
        cuda_check(cudaMemcpy(out, h->timeline, h->timeline_steps * uint64_t(kTlStride) * 8, cudaMemcpyDeviceToHost), "timeline copy");
    });
}

drb_status drb_rb_engine_info(drb_rb* h, uint32_t* resident, uint64_t* instances, uint64_t* posted,
                              uint32_t* grid) {
    DRB_REQUIRE(h && resident && instances && posted && grid);
    *resident = h->rmode ? 1u : 0u;
    *instances = h->gen;
    *posted = h->posted;
    *grid = h->rmode ? h->run_grid : h->grid;
    return DRB_OK;
}

drb_status drb_rb_launch_info(drb_rb* h, uint32_t* grid, uint32_t* threads, uint32_t* smem) {
    DRB_REQUIRE(h && grid && threads && smem);
    *grid = h->grid;
    *threads = kThreads;
    *smem = h->copy_smem;
    return DRB_OK;
}

}  // extern "C"
