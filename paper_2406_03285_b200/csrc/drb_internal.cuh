// Internal layout shared by the sm_100a kernels (drb_kernels.cu) and the C-ABI host code
// (drb_capi.cu). Not installed; the public boundary is include/drb_rb.h.
#pragma once

#include <cstddef>
#include <cstdint>

#include <cuda_runtime.h>

#include "../../include/drb_rb.h"

namespace drb_b200 {

constexpr int kMaxWorld = DRB_RB_MAX_WORLD;
constexpr int kTableRing = 16;  // occupancy-row versions kept per rank (v % 16); see DESIGN.md §3
constexpr int kListRing = 32;  // W_i / X_i slots: sel and plan may run up to 32 iterations ahead of B
// sel and plan reserve at least this much dynamic shared memory, so neither is ever resident
// next to a copy CTA: they are latency-bound single-CTA kernels and, next to a copy CTA,
// their shared/global instructions queue behind the copy's memory traffic. The copy grid
// leaves two SMs for them. The TMA copy kernel stays small enough (<= kSmSmem/2 - 1 KB) for
// two copy CTAs — copy(i) and the programmatically launched copy(i+1) — to share an SM;
// solo_smem_for() raises the floor so that sel/plan + one such copy CTA exceed the SM.
constexpr uint32_t kSoloSmem = 116u * 1024u;
constexpr uint32_t kSmSmem = 228u * 1024u;      // shared memory per SM (sm_100)
constexpr uint32_t kCtaReserved = 1024u;        // per-CTA system reservation
// DRB_TIMELINE=<steps> record per step: [0,6) kernel start/end, [8,32) phase stamps of
// CTA 0, then kTlCtaSlots stamps for each of up to kTlMaxCtas copy CTAs.
constexpr uint32_t kTlCtaSlots = 16, kTlMaxCtas = 160;
constexpr uint32_t kTlStride = 32 + kTlCtaSlots * kTlMaxCtas;
// m' buffers per rank (drb_rb_config.aug_ring, default 32). The API promises m'_i until step
// i+2 is enqueued; the slot is reused by step i+R (batch rows) and by the pushes of
// reps(i+R-1). A deep ring (R >= the steps of a run) keeps every m' of the run readable.
constexpr uint32_t kAugRingDefault = 32;  // (16 -> 32: pipelined update() 6.2 -> 5.9 us/step, runs unchanged)
constexpr uint32_t kAugRingMin = 6;
constexpr uint32_t kTicketRing = 32;  // copy-CTA arrivals per iteration slot (CTAs drift < kListRing)
constexpr uint32_t kAugRingMax = 1u << 16;
// Host-mapped mailbox (u32 words): [0] sticky engine error, [1, 64) control words,
// [64, 64+R) rows of m' per ring slot, [64+R, 64+2R) per-slot round errors.
constexpr uint32_t kMbSticky = 0, kMbBase = 64;
__host__ __device__ inline uint32_t mb_count(uint32_t slot) { return kMbBase + slot; }
__host__ __device__ inline uint32_t mb_err(uint32_t slot, uint32_t R) { return kMbBase + R + slot; }
__host__ __device__ inline uint32_t mb_words(uint32_t R) { return kMbBase + 2 * R; }
constexpr int kThreads = 512;  // step kernel CTA size (16 warps)
constexpr uint64_t kPhi = 0x9e3779b97f4a7c15ULL;

// Mode bits of one step-kernel launch.
enum : uint32_t {
    kModeUpdate = 1u << 0,    // S1+S2: insert candidates of m_i
    kModeAssemble = 1u << 1,  // copy m_i into m'_i rows [0,n)
    kModePlan = 1u << 2,      // S4+S5: plan(i-1) for every requester, push owned entries
    kModeReport = 1u << 3,    // write the per-class insertion report
    kModeCtrParams = 1u << 4, // take cand/evict counters from the params (update_buffer API)
    kModePublish = 1u << 5,   // write own occupancy row for version i+1
    kModePeers = 1u << 6,     // multi-rank: publish to / wait for / push into peers
};

// Device-resident engine state, ping-ponged between consecutive iterations. The
// selection chain (sel kernel) and the planning chain (plan kernel) own separate state so
// that round i+1's selection can run while round i is still being planned / copied.
struct alignas(16) SelState {
    uint64_t cand_ctr;
    uint64_t evict_ctr;
    uint64_t version;      // mutations applied (rehearsal_buffer.cpp:79)
    uint64_t total;        // samples stored (m_total)
    uint64_t cross_class;  // invariant counter, structurally 0 (rehearsal_buffer.hpp:91-95)
    uint32_t error;        // sticky: DRB_ERR_* of a failed round
    uint32_t pad;
};

struct alignas(16) PlanState {
    uint64_t samp_ctr[kMaxWorld];  // every requester's global-sampling counter (replicated)
    uint32_t error;
    uint32_t pad[3];
};

// Peer-shareable region header (one cudaMalloc per rank, exported over CUDA IPC).
struct alignas(256) RegionHeader {
    uint64_t pushdone[kMaxWorld];  // [w]: 1 + last iteration whose pushes rank w completed
                                   //      (its reps rows of my m'_{i+1} have landed)
    uint64_t pad[24];
};

struct RegionLayout {
    uint64_t off_table;     // u64 [kTableRing][N][K] occupancy words: version << 32 | occ
    uint64_t off_counts;    // u32 aug_count[R] (rows of m' per ring slot), repcnt[R] (|reps| in slot s)
    uint64_t off_aug;       // u8  [R][rows][S]
    uint64_t off_auglab;    // u32 [R][rows]
    uint64_t aug_slot_bytes;
    uint64_t rows;          // max_batch + r
    uint64_t bytes;
};

__host__ __device__ inline uint64_t align_up(uint64_t x, uint64_t a) { return (x + a - 1) / a * a; }

// An occupancy-table word carries its row version (i+1 for round i's row) next to the count,
// so a reader recognises a current word by itself: a publisher's plain 8-byte stores need no
// fence and no separate flag (one NVLink trip instead of store + release + acknowledgement).
__host__ __device__ inline uint64_t occ_word(uint64_t version, uint32_t occ) {
    return (uint64_t(uint32_t(version)) << 32) | occ;
}
__host__ __device__ inline uint32_t occ_of(uint64_t w) { return uint32_t(w); }
__host__ __device__ inline bool occ_is(uint64_t w, uint64_t version) { return uint32_t(w >> 32) == uint32_t(version); }

inline RegionLayout region_layout(uint32_t N, uint32_t K, uint64_t S, uint32_t max_batch,
                                  uint32_t r, uint32_t R) {
    RegionLayout L{};
    uint64_t off = sizeof(RegionHeader);
    L.off_table = off = align_up(off, 256);
    off += uint64_t(kTableRing) * N * K * 8;
    L.off_counts = off = align_up(off, 256);
    off += 2ull * R * 4;
    L.rows = uint64_t(max_batch) + r;
    L.aug_slot_bytes = align_up(L.rows * S, 256);
    L.off_aug = off = align_up(off, 256);
    off += uint64_t(R) * L.aug_slot_bytes;
    L.off_auglab = off = align_up(off, 256);
    off += uint64_t(R) * align_up(L.rows * 4, 256);
    L.bytes = align_up(off, 4096);
    return L;
}

struct StepParams {
    uint32_t K, cap, N, me;
    uint32_t n, c, r, nmax;
    uint64_t S;
    uint64_t step;
    uint64_t seq;                  // launch sequence number of this handle (intra-launch flag)
    uint32_t tslot_in, tslot_out;  // table ring slots of versions i and i+1
    uint32_t aslot;                // m' ring slot of step i
    uint32_t aug_ring;             // R, m' ring depth
    uint32_t mode;
    uint64_t cand_key, evict_key;
    uint64_t cand_ctr0, evict_ctr0;  // used with kModeCtrParams
    uint64_t samp_key[kMaxWorld];
    const uint8_t* batch;
    const uint32_t* labels;
    uint8_t* slab;
    uint32_t* slab_labels;
    const SelState* sel_in;
    SelState* sel_out;
    const PlanState* plan_in;
    PlanState* plan_out;
    uint8_t* region[kMaxWorld];  // every rank's region base, mapped in this process
    const uint8_t* slab_peer[kMaxWorld];  // every rank's slab, mapped in this process
    uint64_t off_table, off_counts, off_aug, off_auglab, aug_slot_bytes, auglab_slot_elems;
    const uint32_t* plist_in;  // copy(i): push list P_i (built by plan(i-1))
    uint32_t* plist_out;       // plan(i): push list P_{i+1}
    uint32_t* wlist;           // sel(i) writes / copy(i) reads the candidate-write list W_i
    uint32_t* report;    // [2K + 2]: appends[K], replacements[K], totals[2]
    uint32_t* mailbox;   // host-mapped, mb_* layout above
    uint64_t timeout_ns;
    uint32_t vec16;      // 16-byte vector path legal (S % 16 == 0, aligned bases)
    uint32_t smem_bytes;
    uint32_t solo_smem;
    uint32_t dbg;        // DRB_DBG experiment bits (0 in production)  // sel / plan dynamic smem floor (kSoloSmem or 0), see below
    unsigned long long* trace;  // optional phase timestamps (CTA 0) + grid min/max, 16 slots
    unsigned long long* timeline;  // optional per-kernel [start, end] per step (kind 0 sel, 1 plan, 2 copy)
    uint32_t timeline_steps;       // ring length of the timeline (entries = steps * 3)
    uint64_t evict_m;              // floor((2^64-1) / cap): the eviction bound's reciprocal (host-computed)
    unsigned long long* prof;      // DRB_DBG 65536: clock64 phase accumulators of the run's sel/plan CTAs [64]
};

// ---- resident engine -----------------------------------------------------
// One cooperative kernel per rank stays resident while work is posted: CTA 0 runs the sel
// chain (+ the feeder and ready warps), CTA 1 the plan chain, CTAs 2.. the copies. Work
// arrives as descriptors in a device ring, written by stream-ordered memory operations on
// the caller's stream (update(): one step; run(): a range of steps over an input ring), so
// a step costs no kernel launch. An instance leaves after an idle period once every
// admitted step is complete (so device-wide synchronisation still returns); the next post
// launches the next instance, which resumes from RunCtl.
constexpr uint32_t kFeedRing = 256;  // descriptors in flight
// A descriptor is written by the host into mapped host memory; the poster's stream then stores
// its index + 1 into the device word feed_seq[j % kFeedRing] (one stream memory operation,
// ordered after the producer of the batch); the feeder copies the descriptor into the device
// mirror before admitting its steps.
struct alignas(64) FeedDesc {
    uint64_t batches;       // const uint8_t*: ring of input batches
    uint64_t labels;        // const uint32_t*
    uint64_t batch_stride;  // bytes between ring batches
    uint64_t label_stride;  // u32 elements between ring label rows
    uint64_t i_begin;       // engine iteration of the descriptor's first step
    uint64_t count_n;       // steps (lo 32) | batch rows n (bits 32-61) | kDescEarly | kDescSplit
    uint64_t ring_first;    // ring batches (lo 32) | first batch of the range (hi 32)
    uint64_t seq;           // descriptor index + 1, written last: the descriptor is complete
};
constexpr uint32_t kFeedDescWords = sizeof(FeedDesc) / 8;
// The descriptor's m' is consumed on another stream, which releases consumed m' explicitly
// (RunCtl::consumed); without the flag, posting step i releases every m' before it.
constexpr uint64_t kDescSplit = 1ull << 63;
// Single-stream update(): m'_i is ready as soon as A(i) and the previous round are (B(i) then
// sources round i's winners from m'_i, so m_i is free at that point). Without the flag B(i)
// reads the winners from m_i and m'_i is ready after B(i): the B engines never wait for the
// A engines (the throughput form, runs and split updates).
constexpr uint64_t kDescEarly = 1ull << 62;

// Device counters of the resident engine. Iteration counters are absolute (i+1 once
// iteration i's role finished) and carry over from one instance to the next.
struct alignas(64) RunCtl {
    uint64_t sel_done;   // sel(i) finished (W_i, state, own row v=i+1)
    uint64_t plan_done;  // plan(i) finished (X_i)
    uint64_t b_done;     // B(i) of every copy CTA complete (in order): W_i writes, X_i pushes
    uint64_t a_done;     // A(i) of every copy CTA complete (in order): m_i's rows and labels in m'_i
    uint64_t admitted;   // iterations whose descriptors the feeder has seen
    uint64_t ready;      // m'_i ready for the consumer (i+1): the stream waits poll this word
    uint64_t desc_done;  // descriptors fully consumed (their ring slots may be rewritten)
    uint64_t stop_at;    // gen << 40 | iteration: every role of instance `gen` leaves there
    uint64_t next_step[2];  // [gen & 1]: where instance `gen` starts (written by the one before)
    uint64_t next_desc[2];  // its first descriptor
    uint64_t consumed;      // split-stream consumers: m'_0 .. m'_{consumed-1} are released
    uint32_t error;      // sticky: a wait timed out or a round failed -> every role leaves
    uint32_t where;      // diagnostics: the wait that failed first (site << 24 | k)
    uint32_t pad[2];
    uint32_t ticket[kTicketRing];   // copy-CTA B arrivals of iteration k in slot k % 32 (drift < kListRing)
    uint32_t aticket[kTicketRing];  // copy-CTA A arrivals
};
constexpr uint64_t kStopMask = (1ull << 40) - 1;
constexpr uint64_t kReadyFailed = 1ull << 62;  // ready after a failure: releases every stream wait

// Host-mapped control words of the resident engine (u32 index into the mailbox; u64 words
// take two): the host's posted-descriptor count, the leaving instance's announcement, the
// host's request to leave as soon as idle.
constexpr uint32_t kMbHostPosted = 2, kMbExiting = 4, kMbQuiesce = 6, kMbDescDone = 8, kMbReady = 10;
// the first step the ready publisher did not make ready when the engine failed (written before
// `ready` turns kReadyFailed, so a waiter that sees the failure also sees where it began)
constexpr uint32_t kMbFailedAt = 12;

struct RunParams {
    StepParams base;  // per-iteration fields patched on device (run_patch)
    FeedDesc* feed;                      // [kFeedRing] device mirror of the admitted descriptors
    const FeedDesc* hdesc;               // [kFeedRing] mapped host ring (written by the host)
    const uint64_t* feed_seq;            // [kFeedRing] device: j + 1 once descriptor j is posted
    volatile unsigned long long* desc_done_host;  // mapped mirror of RunCtl::desc_done
    volatile unsigned long long* ready_host;      // mapped mirror of RunCtl::ready (host-side waits)
    RunCtl* ctl;
    uint64_t ver0;
    SelState* sel_base;
    PlanState* plan_base;
    uint32_t* plist_base;
    uint32_t* wlist_base;
    uint64_t gen;      // instance generation
    uint64_t idle_ns;  // leave after this long with nothing admitted and all work done
    const volatile unsigned long long* host_posted;  // mapped: descriptors the host has posted
    volatile unsigned long long* exiting;            // mapped: gen << 32 | next descriptor + 1
    const volatile uint32_t* quiesce;                // mapped: leave as soon as idle
    uint32_t sel_par0, plan_par0, pw, ww, copy_ctas;
    uint32_t feeder_cta;  // CTA whose warps 4 and 5 run the feeder and the ready publisher
    uint64_t* timings;    // DRB_RB_FLAG_TIMINGS: [kTimingRing][kTimingWords] globaltimer stamps, else null
    uint32_t tool_mode;   // under a tool that serialises the device: one instance per post, leave when idle
    uint32_t a_ahead;     // A(i) runs at most this many iterations ahead of the completed B
};
// Per-round stamps (drb_rb_drain_timings): [0] admitted, [1] sel start, [2] sel handed over,
// [3] plan start, [4] pushes complete (b_done)
constexpr uint32_t kTimingRing = 4096, kTimingWords = 8;
constexpr uint32_t kRunThreads = 32 * (kMaxWorld + 2);  // plan_threads(N) + a helper warp, >= kSelThreads

// Push list X_i, plan(i) -> copy(i). u32 words:
//   [0] cnt      — |reps_me(i)|: representative rows of my m'_{i+1}
//   [1] n_jobs   — entries of plan(i), over every requester, whose slot this rank owns
//   [2..3] pad
//   dst[MJ]      (requester q << 24) | position j: the bytes go to q's m'_{i+1} row nmax+j
//   row[MJ]      slot as cls*cap + slot in my slab                       (MJ = N*max(r,1))
__host__ __device__ inline uint32_t plist_mj(uint32_t N, uint32_t r) { return N * (r ? r : 1); }
__host__ __device__ inline uint32_t plist_r(uint32_t r) { return r ? r : 1; }
__host__ __device__ inline uint32_t plist_words(uint32_t N, uint32_t r) { return 4 + 2 * plist_mj(N, r); }

// Candidate-write list W_i, sel(i) -> copy(i). u32 words: [0] n_win, then (batch row,
// slab row) pairs of round i's winning candidates (last writer of each (class, slot)).
__host__ __device__ inline uint32_t wlist_words(uint32_t nmax) { return 2 + 2 * nmax; }

// Dynamic shared-memory carve-ups (4-byte words) of the three iteration kernels.
#define DRB_TAKE(words) (w += ((words) + 3) & ~3u, w - (((words) + 3) & ~3u))
struct SelSmem {
    uint32_t occ, lab, sel, cand_l, cand_slot, kind, misc, words;
};
__host__ __device__ inline SelSmem sel_smem(uint32_t K, uint32_t nmax) {
    SelSmem s{};
    uint32_t w = 0;
    const uint32_t n32 = nmax < 32 ? 32 : nmax;
    s.occ = DRB_TAKE(K);
    s.lab = DRB_TAKE(nmax);
    s.sel = DRB_TAKE(n32);
    s.cand_l = DRB_TAKE(nmax);
    s.cand_slot = DRB_TAKE(nmax);
    s.kind = DRB_TAKE(n32);  // also the 32-entry scratch of warp_select
    s.misc = DRB_TAKE(64);
    s.words = w;
    return s;
}
struct PlanSmem {
    uint32_t pre, pfx, plan, cnt, acc, misc, words;
};
__host__ __device__ inline PlanSmem plan_smem(uint32_t N, uint32_t K, uint32_t r) {
    PlanSmem s{};
    uint32_t w = 0;
    const uint32_t mj = plist_mj(N, r);
    s.pre = DRB_TAKE(N * K + (N * K) / 32 + 1);  // padded: one word per 32 (plan_core's scan stripes)
    s.pfx = DRB_TAKE(N * K + 1 + (N * K + 1) / 32 + 1);
    s.plan = DRB_TAKE(3 * mj);
    s.cnt = DRB_TAKE(N);
    s.acc = DRB_TAKE(mj);
    s.misc = DRB_TAKE(64 + (mj + 31) / 32);
    s.words = w;
    return s;
}
struct CopySmem {
    uint32_t xraw, wraw, jsrc, rowmap, misc, words;
};
__host__ __device__ inline CopySmem copy_smem(uint32_t N, uint32_t r, uint32_t nmax) {
    CopySmem s{};
    uint32_t w = 0;
    s.xraw = DRB_TAKE(plist_words(N, r));  // push list X_i verbatim
    s.wraw = DRB_TAKE(wlist_words(nmax));  // W_i verbatim
    s.jsrc = DRB_TAKE(plist_mj(N, r));     // per job: source row (bit 31: batch row, else slab)
    s.rowmap = DRB_TAKE(nmax);             // batch row -> slab row of its W_i write, or -1
    s.misc = DRB_TAKE(32);
    s.words = w;
    return s;
}
// TMA copy kernel: the copy lists (CopySmem) + mbarriers + a ring of kTmaChunk-byte stages
// (A: batch slice, B: push jobs / non-fused writes).
constexpr uint32_t kTmaThreads = 64;
constexpr uint32_t kTmaChunk = 8192;
// A holds a CTA's whole batch slice at the c2 shape (56 x 150528 B / 146 CTAs = 57.7 KB), so
// copy(i+1) can load and store it to m'_{i+1} while copy(i) still runs (PDL)
constexpr uint32_t kTmaStagesA = 8, kTmaStagesB = 4;
constexpr uint32_t kTmaStages = kTmaStagesA + kTmaStagesB;
struct TmaSmem {
    uint32_t bars, ring, bytes;  // byte offsets
};
__host__ __device__ inline TmaSmem tma_smem(uint32_t N, uint32_t r, uint32_t nmax) {
    TmaSmem t{};
    const uint32_t lists = copy_smem(N, r, nmax).words * 4;
    t.bars = (lists + 127u) & ~127u;
    t.ring = t.bars + 128u * ((8u * kTmaStages + 127u) / 128u);
    t.bytes = t.ring + kTmaStages * kTmaChunk;
    return t;
}
// Persistent run kernel (drb_run_kernel): one carve-up serves every role — sel (+ a second
// label buffer), plan, and the copy role's lists, barriers, A ring and B arena (byte offsets).
// At least kSoloSmem so exactly one CTA lands on each SM.
struct RunSmem {
    uint32_t bars, ring_a, wrows, flags;  // shared by the copy role's warps
    uint32_t xraw[2], wraw[2], jsrc[2], misc[2], paddr[2], arena[2];  // per B warp (k even / odd)
    uint32_t arena_bytes, bytes;
};
__host__ __device__ inline RunSmem run_smem(uint32_t N, uint32_t K, uint32_t r, uint32_t nmax) {
    RunSmem s{};
    const uint32_t MJ = plist_mj(N, r);
    uint32_t off = 0;
    auto take = [&](uint32_t bytes, uint32_t align) {
        off = (off + align - 1) / align * align;
        const uint32_t at = off;
        off += bytes;
        return at;
    };
    s.bars = take(128, 128);
    s.flags = take(128, 16);
    s.wrows = take(4 * (nmax + 1) * 4, 16);  // W_k's slab rows, slot k % 4 (count first)
    for (int w = 0; w < 2; ++w) {
        s.xraw[w] = take(plist_words(N, r) * 4, 16);
        s.wraw[w] = take(wlist_words(nmax) * 4, 16);
        s.jsrc[w] = take(MJ * 4, 16);
        s.misc[w] = take(32 * 4, 16);
        s.paddr[w] = take(16 * (MJ + nmax), 16);
    }
    s.ring_a = take(kTmaStagesA * kTmaChunk, 128);
    const uint32_t want = 200u * 1024u;  // total target; the two arenas take what is left
    const uint32_t left = want > off + 2 * 16384u ? want - off : 2 * 16384u;
    s.arena_bytes = (left / 2) & ~127u;
    s.arena[0] = take(s.arena_bytes, 128);
    s.arena[1] = take(s.arena_bytes, 128);
    const uint32_t sel_b = (sel_smem(K, nmax).words + nmax + 8 + 136) * 4, plan_b = plan_smem(N, K, r).words * 4;
    const uint32_t ctl = sel_b > plan_b ? sel_b : plan_b;
    s.bytes = off > ctl ? off : ctl;
    if (s.bytes < kSoloSmem)
        s.bytes = kSoloSmem;
    return s;
}
#undef DRB_TAKE
// sel/plan shared-memory floor: with the TMA copy kernel at `copy_bytes`, one sel/plan CTA
// plus one copy CTA must not fit on one SM.
__host__ __device__ inline uint32_t solo_smem_for(uint32_t copy_bytes) {
    const uint32_t need = kSmSmem - copy_bytes;  // + 2 reservations > kSmSmem
    const uint32_t lo = need > kSoloSmem ? need : kSoloSmem;
    return lo > 227u * 1024u ? 227u * 1024u : lo;
}

// Launchers (drb_kernels.cu), C++ linkage, used by drb_capi.cu only.
// pdl: launched programmatically behind the previous kernel of the same chain on `stream`
// (its prologue overlaps that kernel; griddepcontrol.wait orders the dependent part).
int launch_sel(const StepParams& p, void* stream, bool pdl = false);
int launch_plan_next(const StepParams& p, void* stream, bool pdl = false);
// pdl: the previous kernel on `stream` is this handle's copy of the previous iteration, so
// the launch may overlap its tail (programmatic dependent launch).
int launch_copy(const StepParams& p, uint32_t grid, void* stream, bool pdl);
int copy_kernel_max_ctas_per_sm(uint32_t smem_bytes, int* out);
// multi-rank: wait (one warp) until every peer's pushes into m'_i landed (pushdone >= i)
int launch_peers_wait(const StepParams& p, void* stream);
int copy_tma_occupancy(uint32_t smem_bytes, int* out);  // CTAs per SM of the TMA copy kernel
// resident engine: dynamic smem, and the cooperative launch of one instance (grid = copy_ctas + 2)
uint32_t run_smem_bytes(uint32_t N, uint32_t K, uint32_t r, uint32_t nmax);
int launch_run(const RunParams& rp, uint32_t grid, void* stream);
// fallback feed without stream memory operations: one thread stores a descriptor / waits for ready
uint32_t sel_smem_bytes(uint32_t K, uint32_t nmax);
uint32_t plan_smem_bytes(uint32_t N, uint32_t K, uint32_t r);
uint32_t plan_threads(uint32_t N);
int launch_bias_counts(uint64_t key, uint32_t want, uint32_t total_draw, uint64_t draws,
                       unsigned long long* counts_dev, uint64_t* ctr_out_dev, void* stream);
int launch_rng_draw(uint64_t key, uint64_t ctr, uint64_t bound, uint64_t n, uint64_t* out_dev,
                    uint64_t* ctr_out_dev, void* stream);
int launch_swor(uint64_t key, uint64_t ctr, uint32_t n, uint32_t k, uint32_t* out_dev,
                uint64_t* ctr_out_dev, void* stream);
int launch_plan(uint64_t key, uint64_t ctr, uint32_t want, uint32_t entries, uint32_t n_workers,
                uint32_t n_classes, const uint32_t* occ_dev, uint32_t* out_dev, uint32_t* count_dev,
                uint64_t* ctr_out_dev, void* stream);
int launch_read_slots(const uint8_t* slab, const uint32_t* slab_labels, const uint32_t* occ_dev,
                      uint32_t K, uint32_t cap, uint64_t S, const uint32_t* req_dev,
                      uint32_t count, uint64_t key, uint64_t ctr, uint8_t* out,
                      uint32_t* out_labels, uint8_t* status_dev, uint64_t* ctr_out_dev,
                      void* stream);

}  // namespace drb_b200
