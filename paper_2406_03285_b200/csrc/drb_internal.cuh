// Internal layout shared by the sm_100a kernels (drb_kernels.cu) and the C-ABI host code
// (drb_capi.cu). Not installed; the public boundary is include/drb_rb.h.
#pragma once

#include <cstddef>
#include <cstdint>

#include <cuda_runtime.h>

#include "../../include/drb_rb.h"

namespace drb_b200 {

constexpr int kMaxWorld = DRB_RB_MAX_WORLD;
constexpr int kTableRing = 6;  // occupancy-row versions kept per rank (v % 6); see DESIGN.md §4
constexpr int kListRing = 4;   // W_i / P_i slots: sel and plan may run up to 4 iterations ahead
// Every iteration kernel (sel, plan, copy) reserves at least this much dynamic shared
// memory, so no two of them are ever resident on one SM: sel and plan are latency-bound
// single-CTA kernels and, next to a copy CTA, their shared/global instructions queue behind
// the copy's memory traffic in the SM's LSU pipe. The copy grid leaves two SMs for them.
constexpr uint32_t kSoloSmem = 116u * 1024u;
// DRB_TIMELINE=<steps> record per step: [0,6) kernel start/end, [8,32) phase stamps of
// CTA 0, then kTlCtaSlots stamps for each of up to kTlMaxCtas copy CTAs.
constexpr uint32_t kTlCtaSlots = 8, kTlMaxCtas = 160;
constexpr uint32_t kTlStride = 32 + kTlCtaSlots * kTlMaxCtas;
constexpr int kAugRing = 3;    // m' buffers per rank; m'_i valid until step i+2 is enqueued
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
    uint64_t occ_flag[kMaxWorld];  // [w]: latest occupancy version rank w published here
    uint64_t done[kMaxWorld];      // [w]: 1 + last iteration whose copy rank w completed
                                   //      (its slab writes of that round are visible)
    uint64_t readdone[kMaxWorld];  // [w]: 1 + last iteration whose pulls rank w completed
    uint64_t ticket;               // local: CTA completion tickets (last-CTA detection)
    uint64_t rticket;              // local: CTA tickets after the pull phase
    uint32_t aug_count[4];         // local: rows of m' per ring slot (device copy)
    uint64_t pad[2];
};

struct RegionLayout {
    uint64_t off_table;     // u32 [kTableRing][N][K]
    uint64_t off_aug;       // u8  [kAugRing][rows][S]
    uint64_t off_auglab;    // u32 [kAugRing][rows]
    uint64_t aug_slot_bytes;
    uint64_t rows;          // max_batch + r
    uint64_t bytes;
};

__host__ __device__ inline uint64_t align_up(uint64_t x, uint64_t a) { return (x + a - 1) / a * a; }

inline RegionLayout region_layout(uint32_t N, uint32_t K, uint64_t S, uint32_t max_batch,
                                  uint32_t r) {
    RegionLayout L{};
    uint64_t off = sizeof(RegionHeader);
    L.off_table = off = align_up(off, 256);
    off += uint64_t(kTableRing) * N * K * 4;
    L.rows = uint64_t(max_batch) + r;
    L.aug_slot_bytes = align_up(L.rows * S, 256);
    L.off_aug = off = align_up(off, 256);
    off += kAugRing * L.aug_slot_bytes;
    L.off_auglab = off = align_up(off, 256);
    off += uint64_t(kAugRing) * align_up(L.rows * 4, 256);
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
    uint64_t off_table, off_aug, off_auglab, aug_slot_bytes, auglab_slot_elems;
    const uint32_t* plist_in;  // copy(i): push list P_i (built by plan(i-1))
    uint32_t* plist_out;       // plan(i): push list P_{i+1}
    uint32_t* wlist;           // sel(i) writes / copy(i) reads the candidate-write list W_i
    uint32_t* report;    // [2K + 2]: appends[K], replacements[K], totals[2]
    uint32_t* mailbox;   // host-mapped: [kAugRing] counts, [kAugRing] errors
    uint64_t timeout_ns;
    uint32_t vec16;      // 16-byte vector path legal (S % 16 == 0, aligned bases)
    uint32_t smem_bytes;
    uint32_t solo_smem;
    uint32_t dbg;        // DRB_DBG experiment bits (0 in production)  // sel / plan dynamic smem floor (kSoloSmem or 0), see below
    unsigned long long* trace;  // optional phase timestamps (CTA 0) + grid min/max, 16 slots
    unsigned long long* timeline;  // optional per-kernel [start, end] per step (kind 0 sel, 1 plan, 2 copy)
    uint32_t timeline_steps;       // ring length of the timeline (entries = steps * 3)
};

// Pull list handed from plan(i-1) to copy(i). u32 words:
//   [0] cnt      — this rank's representatives of round i-1 (= rows pulled into m'_i)
//   [1] n_remote — rows of MY slab that other requesters read this round
//   [2..3] pad
//   owner[R], row[R]      this rank's plan in draw order (pulled into m'_i row nmax+j);
//                         row = cls*cap + slot in the owner's slab          (R = max(r,1))
//   rrow[MJ], rmask[MJ]   remote-read rows of my slab, bit w = requester w reads it
__host__ __device__ inline uint32_t plist_mj(uint32_t N, uint32_t r) { return N * (r ? r : 1); }
__host__ __device__ inline uint32_t plist_r(uint32_t r) { return r ? r : 1; }
__host__ __device__ inline uint32_t plist_words(uint32_t N, uint32_t r) {
    return 4 + 2 * plist_r(r) + 2 * plist_mj(N, r);
}

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
    s.pre = DRB_TAKE(N * K);
    s.pfx = DRB_TAKE(N * K + 1);
    s.plan = DRB_TAKE(3 * mj);
    s.cnt = DRB_TAKE(N);
    s.acc = DRB_TAKE(mj);
    s.misc = DRB_TAKE(64 + (mj + 31) / 32);
    s.words = w;
    return s;
}
struct CopySmem {
    uint32_t praw, wraw, post, win, defer, rowmap, misc, words;
};
__host__ __device__ inline CopySmem copy_smem(uint32_t N, uint32_t r, uint32_t nmax) {
    CopySmem s{};
    uint32_t w = 0;
    s.praw = DRB_TAKE(plist_words(N, r));   // pull list verbatim
    s.wraw = DRB_TAKE(wlist_words(nmax));   // W_i verbatim
    s.post = DRB_TAKE(plist_r(r));          // per pulled rep: local overwrite after the read
    s.win = DRB_TAKE(2 * nmax);             // candidate writes nobody reads this round
    s.defer = DRB_TAKE(3 * nmax);           // writes to rows remote requesters read
    s.rowmap = DRB_TAKE(nmax);              // batch row -> slab row of its safe write, or -1
    s.misc = DRB_TAKE(32);
    s.words = w;
    return s;
}
// TMA copy kernel: the copy lists (CopySmem) + mbarriers + a ring of kTmaChunk-byte stages
// (A: batch slice, B: pulls / safe writes, C: the round-i bytes of pulled rows).
constexpr uint32_t kTmaThreads = 64;
constexpr uint32_t kTmaChunk = 16384;
constexpr uint32_t kTmaStagesA = 6, kTmaStagesB = 2;
constexpr uint32_t kTmaStages = kTmaStagesA + kTmaStagesB;  // C mirrors B: ring slots [kTmaStages, +B)
struct TmaSmem {
    uint32_t bars, ring, bytes;  // byte offsets
};
__host__ __device__ inline TmaSmem tma_smem(uint32_t N, uint32_t r, uint32_t nmax) {
    TmaSmem t{};
    const uint32_t lists = copy_smem(N, r, nmax).words * 4;
    t.bars = (lists + 127u) & ~127u;
    t.ring = t.bars + 128u * ((8u * (kTmaStages + kTmaStagesB) + 127u) / 128u);
    t.bytes = t.ring + (kTmaStages + kTmaStagesB) * kTmaChunk;
    return t;
}
#undef DRB_TAKE

// Launchers (drb_kernels.cu), C++ linkage, used by drb_capi.cu only.
int launch_sel(const StepParams& p, void* stream);
int launch_plan_next(const StepParams& p, void* stream);
// pdl: the previous kernel on `stream` is this handle's copy of the previous iteration, so
// the launch may overlap its tail (programmatic dependent launch).
int launch_copy(const StepParams& p, uint32_t grid, void* stream, bool pdl);
int copy_kernel_max_ctas_per_sm(uint32_t smem_bytes, int* out);
uint32_t sel_smem_bytes(uint32_t K, uint32_t nmax);
uint32_t plan_smem_bytes(uint32_t N, uint32_t K, uint32_t r);
uint32_t plan_threads(uint32_t N);
int launch_rng_draw(uint64_t key, uint64_t ctr, uint64_t bound, uint64_t n, uint64_t* out_dev,
                    uint64_t* ctr_out_dev, void* stream);
int launch_swor(uint64_t key, uint64_t ctr, uint32_t n, uint32_t k, uint32_t* out_dev,
                uint64_t* ctr_out_dev, void* stream);
int launch_plan(uint64_t key, uint64_t ctr, uint32_t want, uint32_t n_workers, uint32_t n_classes,
                const uint32_t* occ_dev, uint32_t* out_dev, uint32_t* count_dev,
                uint64_t* ctr_out_dev, void* stream);
int launch_read_slots(const uint8_t* slab, const uint32_t* slab_labels, const uint32_t* occ_dev,
                      uint32_t K, uint32_t cap, uint64_t S, const uint32_t* req_dev,
                      uint32_t count, uint64_t key, uint64_t ctr, uint8_t* out,
                      uint32_t* out_labels, uint8_t* status_dev, uint64_t* ctr_out_dev,
                      void* stream);

}  // namespace drb_b200
