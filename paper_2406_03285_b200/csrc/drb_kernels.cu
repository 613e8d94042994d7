// sm_100a kernels of the distributed rehearsal buffer (arXiv 2406.03285 hot path).
//
// One engine iteration i on one rank is three kernels:
//   * sel(i):  S1+S2 update_buffer(m_i)          proj/src/buffer/rehearsal_buffer.cpp:14-86
//              publish occupancy row v=i+1       proj/src/engine/engine.cpp:108-136
//   * plan(i): size rendezvous v=i+1             proj/src/sampler/size_table.cpp:66-100
//              S4 plan(i) for every requester    proj/src/sampler/sampler.cpp:39-68 (+ locate,
//                                                proj/src/sampler/size_table.cpp:29-39)
//   * copy(i): m_i -> m'_i, the slab writes of round i, and S5: every owned slot of plan(i)
//              at version i+1 pushed into its requester's m'_{i+1}
//                                                proj/src/sampler/sampler.cpp:111-232 (fetch),
//                                                proj/src/engine/engine.cpp:215-251 (serve),
//              so m'_i = m_i ++ reps(i-1)        proj/src/sampler/sampler.cpp:234-240
// The RNG decisions are bit-identical to proj/src/core/rng.cpp:12-53 and are evaluated
// warp-parallel over consecutive counters (exact rejection semantics; see warp_* below).

#include <cuda_runtime.h>

#include <cstdint>

#include "drb_internal.cuh"

// Timeline / trace / phase-profile stamps (DRB_TIMELINE, DRB_TRACE, DRB_DBG 65536) exist only
// in the instrumented build (-DDRB_INSTRUMENT=1, tools/): every site costs the control chains
// instruction fetch and issue slots even when switched off at run time.
#ifndef DRB_INSTRUMENT
#define DRB_INSTRUMENT 0
#endif
// Critical-chain experiment (tools/): -DDRB_DELAY=1/2/3 adds ~1 us per iteration to the sel /
// plan / B chain of the persistent run; the chain whose delay moves the step time is the bound.
#ifndef DRB_DELAY
#define DRB_DELAY 0
#endif

namespace drb_b200 {

namespace {

constexpr unsigned kFull = 0xffffffffu;

__device__ __forceinline__ void delay_exp(int chain) {
    if (DRB_DELAY == chain) {
        const long long t0 = clock64();
        while (clock64() - t0 < 2000) {
        }
    }
}

__device__ __forceinline__ uint64_t mix64(uint64_t z) {  // rng.cpp:12-17
    z += kPhi;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

// Value of the draw whose post-increment counter is `ctr` (rng.cpp:41-43).
__device__ __forceinline__ uint64_t draw_at(uint64_t key, uint64_t ctr) {
    return mix64(key ^ (ctr * kPhi));
}

// Sequential bounded(n) (rng.cpp:45-53); advances ctr by the draws consumed.
__device__ uint64_t bounded_seq(uint64_t key, uint64_t& ctr, uint64_t n) {
    const uint64_t thr = (0ull - n) % n;
    for (;;) {
        const uint64_t v = draw_at(key, ++ctr);
        if (v >= thr)
            return v % n;
    }
}

// Exact v mod d for a 32-bit d, without the generic 64-bit division routine: with
// m = floor((2^64-1)/d) (one division, shared by every lane that reduces by the same d),
// q = umulhi(v, m) undershoots floor(v/d) by at most 2. The rejection threshold of
// bounded(d) is (2^64 - d) mod d = reduce(0 - d) (rng.cpp:45-53).
struct reducer {
    uint64_t d, m;
    __device__ explicit reducer(uint64_t d_) : d(d_), m(~0ull / d_) {}
    __device__ reducer(uint64_t d_, uint64_t m_) : d(d_), m(m_) {}  // m precomputed (= ~0 / d)
    __device__ __forceinline__ uint64_t mod(uint64_t v) const {
        uint64_t r = v - __umul64hi(v, m) * d;
        r = r >= d ? r - d : r;
        return r >= d ? r - d : r;
    }
    __device__ __forceinline__ uint64_t thr() const { return mod(0ull - d); }
};
// v mod d for d < 2^16 from three 32-bit remainders: v = hi*2^32 + lo and
// (hi mod d)*(2^32 mod d) < 2^32.
__device__ __forceinline__ uint32_t mod_small(uint64_t v, uint32_t d) {
    const uint32_t c = (0u - d) % d;  // 2^32 mod d
    const uint32_t hi = static_cast<uint32_t>(v >> 32) % d, lo = static_cast<uint32_t>(v) % d;
    return ((hi * c) % d + lo) % d;
}
// i mod R for the m' ring (R <= 2^16) in 32-bit arithmetic: no 64-bit division routine on the
// per-step paths
__device__ __forceinline__ uint32_t ring_slot(uint64_t i, uint32_t R) { return mod_small(i, R); }
__device__ __forceinline__ uint32_t thr_small(uint32_t d) {  // 2^64 mod d = (2^32 mod d)^2 mod d
    const uint32_t c = (0u - d) % d;
    return (c * c) % d;
}

__device__ __forceinline__ uint64_t globaltimer() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__device__ __forceinline__ uint64_t ld_acquire_sys(const uint64_t* p) {
    uint64_t v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void st_release_sys(uint64_t* p, uint64_t v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ uint4 ld_stream(const uint4* p) {
    uint4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p));
    return v;
}

// S1 — partial Fisher–Yates selection (rehearsal_buffer.cpp:14-26), one full warp.
// Fast path (k <= 32, no rejection in the k draws): lane j evaluates draw j
// (counter ctr+1+j, bound n-j) in parallel and the swap sequence is resolved without
// materialising the permutation:
//   A(j)   = value at position j just before swap j
//          = A(m) for the latest m<j with s_m == j, else j          (pointer jumping)
//   sel[j] = A(q) for the latest q<j with s_q == s_j, else s_j.
// Any rejected draw (probability < k*2^-32) falls back to the literal sequential loop.
// The fast path alone (k <= 32, n < 2^16): sel[0..k) for draws ctr+1..ctr+k; false (sel
// untouched) if any of them is rejected. `idx` is 32 words of scratch.
__device__ bool warp_select_fast(uint64_t key, uint64_t ctr, uint32_t n, uint32_t k, uint32_t* sel,
                                 uint32_t* idx) {
    const int lane = threadIdx.x & 31;
    {
        const uint32_t j = lane;
        uint32_t s = 0xffffffffu;
        bool ok = true;
        if (j < k) {  // n <= 4096 (max_batch): 32-bit remainders
            const uint32_t nj = n - j;
            const uint64_t v = draw_at(key, ctr + 1 + j);
            ok = v >= thr_small(nj);
            s = j + mod_small(v, nj);
        }
        if (__ballot_sync(kFull, !ok) == 0) {
            // q: latest earlier lane drawing the same target (one match instruction)
            const unsigned same = __match_any_sync(kFull, s);
            const unsigned lt = (1u << lane) - 1u;
            const int q = (j < k && (same & lt)) ? 31 - __clz(same & lt) : -1;
            // pa(j): latest earlier lane m whose target s_m == j (s_m > m), via smem max
            int* last = reinterpret_cast<int*>(idx);
            last[lane] = -1;
            __syncwarp();
            if (j < k && s < 32 && s != j)
                atomicMax(&last[s], lane);
            __syncwarp();
            const int pa = j < k ? last[lane] : -1;
            __syncwarp();
            int par = pa >= 0 ? pa : lane;
#pragma unroll
            for (int it = 0; it < 5; ++it)
                par = __shfl_sync(kFull, par, par);
            const uint32_t aq = __shfl_sync(kFull, static_cast<uint32_t>(par), q < 0 ? 0 : q);
            if (j < k)
                sel[j] = q >= 0 ? aq : s;
            __syncwarp();
            return true;
        }
    }
    return false;
}

__device__ void warp_select(uint64_t key, uint64_t& ctr, uint32_t n, uint32_t k, uint32_t* sel,
                            uint32_t* idx) {
    const int lane = threadIdx.x & 31;
    if (k == 0)
        return;
    // (mod_small needs n < 2^16; max_batch <= 4096)
    if (k <= 32 && n < 65536u && warp_select_fast(key, ctr, n, k, sel, idx)) {
        ctr += k;
        return;
    }
    for (uint32_t i = lane; i < n; i += 32)
        idx[i] = i;
    __syncwarp();
    if (lane == 0) {
        for (uint32_t j = 0; j < k; ++j) {
            const uint32_t s = j + static_cast<uint32_t>(bounded_seq(key, ctr, n - j));
            const uint32_t t = idx[j];
            idx[j] = idx[s];
            idx[s] = t;
            sel[j] = idx[j];
        }
    }
    ctr = __shfl_sync(kFull, ctr, 0);
    __syncwarp();
}

// S2 — per-candidate class slot assignment in selection order (rehearsal_buffer.cpp:55-80),
// one full warp, 32 candidates per pass. Candidate t of class L with in-batch rank rho
// appends at occ[L]+rho while that is < cap; otherwise it replaces slot
// evict.bounded(cap) — eviction draws are consumed only by replacements, in selection
// order (exclusive prefix over the replacement ballot; rejected draws are skipped via
// __fns over the validity ballot, which is exact because every replacement draws with the
// same bound cap). occ[] (shared) is updated in place to the post-update occupancy.
__device__ void warp_assign(uint64_t ekey, uint64_t& ectr, uint32_t cap, uint64_t cap_m, uint32_t k,
                            const uint32_t* sel, const uint32_t* lab, uint32_t* occ,
                            uint32_t* cand_l, uint32_t* cand_slot, uint32_t* scratch,
                            uint32_t* kind, uint32_t& appends) {
    const int lane = threadIdx.x & 31;
    const reducer red = cap_m ? reducer(cap, cap_m) : reducer(cap);
    const uint64_t thr = red.thr();
    const unsigned lt = (1u << lane) - 1u;
    appends = 0;
    for (uint32_t base = 0; base < k; base += 32) {
        const uint32_t t = base + lane;
        const bool act = t < k;
        const uint32_t L = act ? lab[sel[t]] : 0xffffffffu;
        // in-batch rank of this candidate within its class, and whether it is the last
        const unsigned same = __match_any_sync(kFull, L);
        const uint32_t rho = __popc(same & lt);
        const bool last_of_class = (same >> lane) == 1u;
        const uint32_t o = act ? occ[L] : 0;
        __syncwarp();
        const bool app = act && (o + rho < cap);
        const bool rep = act && !app;
        const unsigned rmask = __ballot_sync(kFull, rep);
        const uint32_t R = __popc(rmask);
        const uint32_t e = __popc(rmask & lt);
        uint32_t slot = o + rho;
        if (R) {
            const uint64_t v = draw_at(ekey, ectr + 1 + lane);
            const bool valid = v >= thr;
            const unsigned vmask = __ballot_sync(kFull, valid);
            if (static_cast<uint32_t>(__popc(vmask)) >= R) {
                // the e-th replacement takes the e-th valid draw: valid lanes deposit their value
                // by valid-rank, replacements pick theirs up (no per-lane __fns)
                const uint32_t vr = __popc(vmask & lt);
                if (valid && vr < R)
                    scratch[vr] = static_cast<uint32_t>(red.mod(v));
                __syncwarp();
                if (rep)
                    slot = scratch[e];
                ectr += __ffs(__ballot_sync(kFull, valid && vr == R - 1));  // past the R-th valid draw
                __syncwarp();
            } else {
                if (lane == 0)
                    for (uint32_t x = 0; x < R; ++x)
                        scratch[x] = static_cast<uint32_t>(bounded_seq(ekey, ectr, cap));
                ectr = __shfl_sync(kFull, ectr, 0);
                __syncwarp();
                if (rep)
                    slot = scratch[e];
            }
        }
        if (act) {
            cand_l[t] = L;
            cand_slot[t] = slot;
            kind[t] = app ? 1u : 0u;
            if (last_of_class)
                occ[L] = min(cap, o + rho + 1);
        }
        appends += __popc(__ballot_sync(kFull, app));
        __syncwarp();
    }
}

// S4 — plan(want, view) draws (sampler.cpp:39-61) for one requester, one full warp.
// Draws are bounded(total) on consecutive counters; lane l holds counter ctr+1+l.
// Rejected draws are skipped, duplicates (of accepted flats or of earlier lanes in the
// same batch) consume their counter without producing an entry — exactly the
// `while (|out| < want) { f = bounded(total); if (insert(f)) out.push(locate(f)); }`
// loop. The counter advances to the draw that completed the plan. Exhaustion
// (want >= total) lists every slot in flat order with no draws. Returns the entry count;
// acc[] receives the flat indices in draw order.
__device__ uint32_t warp_plan_draw(uint64_t key, uint64_t& ctr, uint32_t want, uint32_t total,
                                   uint32_t* acc) {
    const int lane = threadIdx.x & 31;
    const unsigned lt = (1u << lane) - 1u;
    if (want == 0 || total == 0)
        return 0;
    if (want >= total) {
        #pragma unroll 1
        for (uint32_t j = lane; j < total; j += 32)
            acc[j] = j;
        __syncwarp();
        return total;
    }
    const reducer red(total);
    const uint64_t thr = red.thr();
    uint32_t got = 0;
    while (got < want) {
        const uint64_t v = draw_at(key, ctr + 1 + lane);
        const bool ok = v >= thr;
        const uint32_t f = static_cast<uint32_t>(red.mod(v));
        // duplicate of an earlier valid lane in this batch? (rejected lanes get a unique
        // key above any flat index, total < 2^31)
        const unsigned same = __match_any_sync(kFull, ok ? f : 0x80000000u + lane);
        bool dup = !ok || (same & lt) != 0;
        for (uint32_t a = 0; a < got; ++a)
            if (acc[a] == f)
                dup = true;
        const unsigned nm = __ballot_sync(kFull, !dup);
        const uint32_t c = __popc(nm);
        const uint32_t need = want - got;
        const uint32_t rank = __popc(nm & lt);
        __syncwarp();
        if (c >= need) {
            if (!dup && rank < need)
                acc[got + rank] = f;
            // the lane holding the need-th new flat (one ballot, not __fns)
            ctr += __ffs(__ballot_sync(kFull, !dup && rank == need - 1));
            got = want;
        } else {
            if (!dup)
                acc[got + rank] = f;
            ctr += 32;
            got += c;
        }
        __syncwarp();
    }
    return want;
}

// locate (size_table.cpp:29-39): flat -> (owner, class, slot) by binary search over the
// exclusive prefix pfx[0..NK] (largest i with pfx[i] <= f), one warp.
// Shared-memory index with one pad word per 32: a lane's contiguous stripe of a prefix array
// (lane * per + i) then falls on distinct banks (K = 1000 puts 32 words in every stripe).
template <bool kPad>
__device__ __forceinline__ uint32_t pidx(uint32_t x) { return kPad ? x + (x >> 5) : x; }

template <bool kPad = false>
__device__ void warp_locate(const uint32_t* acc, uint32_t cnt, const uint32_t* pfx, uint32_t NK,
                            uint32_t K, uint32_t* plan) {
    const int lane = threadIdx.x & 31;
    for (uint32_t j = lane; j < cnt; j += 32) {
        const uint32_t f = acc[j];
        uint32_t lo = 0, hi = NK;
        while (hi - lo > 1) {
            const uint32_t mid = (lo + hi) >> 1;
            if (pfx[pidx<kPad>(mid)] <= f)
                lo = mid;
            else
                hi = mid;
        }
        plan[3 * j] = lo / K;
        plan[3 * j + 1] = lo % K;
        plan[3 * j + 2] = f - pfx[pidx<kPad>(lo)];
    }
    __syncwarp();
}

// Exclusive prefix of a[0..n) into out[0..n] (out[n] = total), one warp: each lane scans a
// contiguous stripe, then a warp scan of the stripe totals.
template <bool kPad = false>
__device__ uint32_t warp_exclusive_scan(const uint32_t* a, uint32_t n, uint32_t* out) {
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t per = (n + 31) / 32;
    const uint32_t b0 = min(n, lane * per), b1 = min(n, b0 + per);
    uint32_t s = 0;
    for (uint32_t i = b0; i < b1; ++i)
        s += a[pidx<kPad>(i)];
    uint32_t x = s;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(kFull, x, o);
        if (lane >= static_cast<uint32_t>(o))
            x += y;
    }
    uint32_t excl = x - s;
    for (uint32_t i = b0; i < b1; ++i) {
        out[pidx<kPad>(i)] = excl;
        excl += a[pidx<kPad>(i)];
    }
    const uint32_t total = __shfl_sync(kFull, x, 31);
    if (lane == 0)
        out[pidx<kPad>(n)] = total;
    __syncwarp();
    return total;
}

template <typename V>
__device__ __forceinline__ V ld_vec(const V* p) {
    if constexpr (sizeof(V) == 16) {
        const uint4 v = ld_stream(reinterpret_cast<const uint4*>(p));
        return *reinterpret_cast<const V*>(&v);
    } else {
        return __ldg(p);
    }
}

// Diagnostics: sel / plan stamp slots 0-8, copy CTA 0 slots 16-19 (DRB_TRACE=1).
// Timeline (DRB_TIMELINE=<steps>): grid-wide first start / last end of each kernel of
// each step, as globaltimer ns; works inside CUDA graphs.
__device__ __forceinline__ void tl_mark(const StepParams& p, int kind, bool end) {
#if DRB_INSTRUMENT
    if (p.timeline && threadIdx.x == 0) {
        unsigned long long* e = p.timeline + (p.step & (p.timeline_steps - 1)) * kTlStride + 2 * kind;
        if (end)
            atomicMax(e + 1, globaltimer());
        else
            atomicMin(e, globaltimer());
    }
#endif
}

// per-CTA copy stamps (timeline mode): slot s of this CTA, written by the calling thread
__device__ __forceinline__ void cta_mark(const StepParams& p, int slot) {
#if DRB_INSTRUMENT
    if (p.timeline && blockIdx.x < kTlMaxCtas) {
        uint64_t t;  // "memory": not reordered with the surrounding loads / stores
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)::"memory");
        p.timeline[(p.step & (p.timeline_steps - 1)) * kTlStride + 32 + blockIdx.x * kTlCtaSlots + slot] = t;
    }
#endif
}

// DRB_DBG 65536: cycles since `t` into prof slot `slot` of this control CTA (lane 0 of the
// calling warp), then t = now. Free of memory traffic when profiling is off.
__device__ __forceinline__ void prof_span(const StepParams& p, int slot, unsigned long long& t) {
#if DRB_INSTRUMENT
    if (p.prof && blockIdx.x <= 1 && (threadIdx.x & 31) == 0) {
        const unsigned long long now = clock64();
        if (t)
            atomicAdd(p.prof + 32 * blockIdx.x + slot, now - t);
        t = now;
    }
#endif
}

__device__ __forceinline__ void trace_at(const StepParams& p, int slot) {
#if DRB_INSTRUMENT
    // CTA 0 (sel, plan and the copy's first CTA); CTA 1 too: the plan role of a persistent run
    if (p.prof && blockIdx.x <= 1 && threadIdx.x == 0) {  // cycles since this CTA's previous stamp
        __shared__ unsigned long long prof_prev;
        const unsigned long long now = clock64();
        if (slot != 12 && slot != 13)  // 12/13: loop tops (start the chain)
            atomicAdd(p.prof + 32 * blockIdx.x + slot, now - prof_prev);
        else
            atomicAdd(p.prof + 32 * blockIdx.x + slot, prof_prev ? now - prof_prev : 0ull);
        atomicAdd(p.prof + 32 * blockIdx.x + 31, slot == 12 || slot == 13 ? 1ull : 0ull);
        prof_prev = now;
    }
    if (blockIdx.x <= 1 && (threadIdx.x & 31) == 0) {
        if (p.trace)
            p.trace[slot] = globaltimer();
        if (p.timeline)  // phase stamps of the pipelined run: slots 8.. of the step's record
            p.timeline[(p.step & (p.timeline_steps - 1)) * kTlStride + 8 + slot] = globaltimer();
    }
#endif
}

}  // namespace

// ======================================================================================
// One engine iteration i on one rank is three kernels, pipelined across iterations
// (DESIGN.md §3):
//   sel(i)   1 CTA  : S1+S2 of round i (rehearsal_buffer.cpp:14-86), the candidate-write
//                     list W_i, round-(i+1) selection state, occupancy row v=i+1 published
//                     (engine.cpp:108-136)                        — chained only on sel(i-1)
//   plan(i)  1 CTA  : size rendezvous v=i+1 (size_table.cpp:66-100), S4 plan(i) for every
//                     requester (sampler.cpp:39-68), the push list X_i, labels of
//                     m'_{i+1}'s representatives                  — chained only on plan(i-1)
//   copy(i)  grid   : m_i -> m'_i rows, W_i into the slab, and the pushes of X_i (slots at
//                     version i+1 into each requester's m'_{i+1})
// so copy(i) starts with every list it needs already in memory, and sel(i+1) / plan(i+1)
// run concurrently with copy(i) on their own streams.
// ======================================================================================

constexpr uint32_t kSelThreads = 128;

// m' ring slot counts of this rank: aug_count[R] then repcnt[R]
__device__ __forceinline__ uint32_t* counts_of(const StepParams& p) {
    return reinterpret_cast<uint32_t*>(p.region[p.me] + p.off_counts);
}
// How far a rank's sel(i) may run ahead of every peer's pushes (multi-rank): the table slot
// its row overwrites (kTableRing versions) and the m' slot plan(i) refills (R slots).
__device__ __forceinline__ uint32_t aug_lag(uint32_t R) { return R < kTableRing ? R : kTableRing; }

// Spin (thread-level) until *flag >= want or the timeout; returns false on timeout.
__device__ bool wait_flag(const uint64_t* flag, uint64_t want, uint64_t timeout_ns) {
    const uint64_t t0 = globaltimer();
    while (ld_acquire_sys(flag) < want) {
        if (globaltimer() - t0 > timeout_ns)
            return false;
        __nanosleep(32);
    }
    return true;
}

struct SelView {  // sel's shared-memory arrays (sel_smem carve-up)
    uint32_t *occ, *lab, *sel, *cand_l, *cand_slot, *kind, *misc;
    SelState* st;
};
__device__ __forceinline__ SelView sel_view(uint32_t* sm, const StepParams& p) {
    const SelSmem L = sel_smem(p.K, p.nmax);
    SelView v;
    v.occ = sm + L.occ;
    v.lab = sm + L.lab;
    v.sel = sm + L.sel;
    v.cand_l = sm + L.cand_l;
    v.cand_slot = sm + L.cand_slot;
    v.kind = sm + L.kind;
    v.misc = sm + L.misc;
    v.st = reinterpret_cast<SelState*>(v.misc + 16);
    return v;
}

// sel(i) after its loads (one full warp): S1+S2 on occ (own occupancy row, version i, updated
// in place to version i+1) and lab (labels of m_i, `bad` if any is >= K), the candidate-write
// list W_i, the round-(i+1) selection state (p.sel_out, and *v.st in place), stored slot
// labels, the published occupancy row v=i+1 and the insertion report.
// spec (persistent run): a selection computed ahead for the counter spec_ctr (k = min(c, n)
// draws, no rejection); used when it matches this round's counter and k.
__device__ void sel_core(const StepParams& p, const SelView& v, bool bad, const uint32_t* spec = nullptr,
                         uint64_t spec_ctr = ~0ull, bool peers_checked = false) {
    const uint32_t lane = threadIdx.x & 31;
    const unsigned lt = (1u << lane) - 1u;
    const uint32_t N = p.N, K = p.K, me = p.me, n = p.n, cap = p.cap;
    const uint32_t NK = N * K;
    const bool do_update = p.mode & kModeUpdate;
    const bool do_publish = p.mode & kModePublish;
    const bool multi = (p.mode & kModePeers) && N > 1;
    SelState* st = v.st;
    uint32_t *occ = v.occ, *sel = v.sel, *cand_l = v.cand_l, *cand_slot = v.cand_slot, *kind = v.kind;
    trace_at(p, 1);
    const bool dead = st->error != 0;  // sticky: a failed round kills the engine
    const uint32_t k = (!dead && do_update && !bad && n > 0) ? min(p.c, n) : 0;
    uint64_t cand_ctr = (p.mode & kModeCtrParams) ? p.cand_ctr0 : st->cand_ctr;
    uint64_t evict_ctr = (p.mode & kModeCtrParams) ? p.evict_ctr0 : st->evict_ctr;
    uint32_t appends = 0;
    if (k > 0) {
        if (spec && spec_ctr == cand_ctr && k <= 32) {  // S1 already drawn for this counter
            sel = const_cast<uint32_t*>(spec);
            cand_ctr += k;
        } else {
            warp_select(p.cand_key, cand_ctr, n, k, sel, kind);
        }
        trace_at(p, 2);
        warp_assign(p.evict_key, evict_ctr, cap, p.evict_m, k, sel, v.lab, occ, cand_l, cand_slot, v.misc + 32, kind,
                    appends);
    }
    trace_at(p, 3);
    unsigned long long pt = 0;
    prof_span(p, 14, pt);
    // W_i: winners = last writer of each (class, slot) in selection order, ballot-ordered
    uint32_t* wl = p.wlist;
    uint32_t n_win = 0;
#pragma unroll 1
    for (uint32_t base = 0; base < k; base += 32) {
        const uint32_t t = base + lane;
        bool w = false;
        uint32_t key = 0;
        if (k <= 32) {  // one match: no later candidate of the same (class, slot)
            key = t < k ? cand_l[t] * cap + cand_slot[t] : 0x80000000u + lane;  // slots < 2^31
            const unsigned same = __match_any_sync(kFull, key);
            w = t < k && (same >> lane) == 1u;
        } else if (t < k) {
            key = cand_l[t] * cap + cand_slot[t];
            w = true;
#pragma unroll 1
            for (uint32_t u = t + 1; u < k && w; ++u)
                w = cand_l[u] * cap + cand_slot[u] != key;
        }
        const unsigned m = __ballot_sync(kFull, w);
        if (w) {
            const uint32_t pos = n_win + __popc(m & lt);
            wl[2 + 2 * pos] = sel[t];
            wl[3 + 2 * pos] = key;
        }
        n_win += __popc(m);
    }
    if (lane == 0)
        wl[0] = n_win;
    prof_span(p, 14, pt);
    // round-(i+1) selection state
    const uint32_t err = dead ? st->error : ((bad && do_update) ? DRB_ERR_USAGE : 0u);
    __syncwarp();
    if (lane == 0) {
        SelState o;
        o.cand_ctr = cand_ctr;
        o.evict_ctr = evict_ctr;
        o.version = st->version + k;  // one per mutation (rehearsal_buffer.cpp:79)
        o.total = st->total + appends;
        o.cross_class = st->cross_class;
        o.error = err;
        o.pad = 0;
        *p.sel_out = o;
        *st = o;
        if (p.mailbox && err)
            reinterpret_cast<volatile uint32_t*>(p.mailbox)[kMbSticky] = err;
    }
    prof_span(p, 15, pt);
#pragma unroll 1
    for (uint32_t t = lane; t < k; t += 32)  // stored label == class (class-partitioned)
        p.slab_labels[cand_l[t] * cap + cand_slot[t]] = cand_l[t];
    prof_span(p, 16, pt);
    if (do_publish && !dead) {  // publish_row(i): version i+1 (engine.cpp:108-136)
        uint64_t* tout = reinterpret_cast<uint64_t*>(p.region[me] + p.off_table) +
                         uint64_t(p.tslot_out) * NK + uint64_t(me) * K;
#pragma unroll 1
        for (uint32_t x = lane; x < K; x += 32)
            tout[x] = occ_word(p.step + 1, occ[x]);
        if (multi) {
            // Every peer finished copy(i-6) (it announced pushdone >= i-5): its plan(i-6) no
            // longer reads the table slot this row overwrites, and its pushes into the m'
            // slot that plan(i) refills have landed. Normally long true: sel runs ahead.
            const uint32_t lag = aug_lag(p.aug_ring);
            if (!peers_checked && p.step >= lag && lane < N && lane != me &&
                !wait_flag(&reinterpret_cast<const RegionHeader*>(p.region[me])->pushdone[lane],
                           p.step - (lag - 1), p.timeout_ns) &&
                p.mailbox)
                reinterpret_cast<volatile uint32_t*>(p.mailbox)[kMbSticky] = DRB_ERR_TRANSPORT;
            __syncwarp();
#pragma unroll 1
            for (uint32_t w = 0; w < N; ++w) {
                if (w == me)
                    continue;
                uint64_t* pt = reinterpret_cast<uint64_t*>(p.region[w] + p.off_table) +
                               uint64_t(p.tslot_out) * NK + uint64_t(me) * K;
#pragma unroll 1
                for (uint32_t x = lane; x < K; x += 32)  // self-validating words: no flag, no fence
                    pt[x] = occ_word(p.step + 1, occ[x]);
            }
        }
    }
    prof_span(p, 17, pt);
    if (p.mode & kModeReport) {  // insertion_report (rehearsal_buffer.hpp:17-26)
#pragma unroll 1
        for (uint32_t x = lane; x < 2 * K + 2; x += 32)
            p.report[x] = 0;
        __syncwarp();
        __threadfence_block();
#pragma unroll 1
        for (uint32_t t = lane; t < k; t += 32) {
            const bool app = kind[t] != 0;
            atomicAdd(&p.report[(app ? 0 : K) + cand_l[t]], 1u);
            atomicAdd(&p.report[2 * K + (app ? 0 : 1)], 1u);
        }
    }
    __syncwarp();
    prof_span(p, 18, pt);
    trace_at(p, 4);
}

// labels of m_i into v.lab (all threads of the CTA, stride T); returns this thread's "bad"
__device__ __forceinline__ int sel_load_labels(const StepParams& p, const SelView& v, uint32_t T) {
    int any_bad = 0;
#pragma unroll 1
    for (uint32_t x = threadIdx.x; x < p.n; x += T) {
        const uint32_t l = __ldg(p.labels + x);
        v.lab[x] = l;
        any_bad |= l >= p.K;
    }
    return any_bad;
}

__global__ void __launch_bounds__(kSelThreads) drb_sel_kernel(const __grid_constant__ StepParams p) {
    extern __shared__ __align__(128) uint32_t sm[];
    const SelView v = sel_view(sm, p);
    const uint32_t tid = threadIdx.x, warp = tid >> 5;
    const uint64_t* tin = reinterpret_cast<const uint64_t*>(p.region[p.me] + p.off_table) +
                          uint64_t(p.tslot_in) * p.N * p.K + uint64_t(p.me) * p.K;
    trace_at(p, 0);
    tl_mark(p, 0, false);
    // No griddepcontrol.launch_dependents here (nor in plan): a copy launched with the PDL
    // attribute turns ALL its captured in-edges programmatic, and copy(i) reads W_i / X_i
    // before its griddepcontrol.wait — so sel/plan must trigger their dependents only by
    // completing. (Measured: PDL on the sel/plan chains themselves does not pay either.)
    // Under PDL the labels of m_i would load while sel(i-1) still runs; state and the own
    // occupancy row (version i) come from sel(i-1) and load after griddepcontrol.wait.
    const int any_bad = sel_load_labels(p, v, kSelThreads);
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (tid < sizeof(SelState) / 8)
        reinterpret_cast<uint64_t*>(v.st)[tid] = __ldcg(reinterpret_cast<const uint64_t*>(p.sel_in) + tid);
#pragma unroll 1
    for (uint32_t x = tid; x < p.K; x += kSelThreads)
        v.occ[x] = occ_of(__ldcg(tin + x));
    const bool bad = __syncthreads_or(any_bad) != 0;  // usage_error before any draw (:44-47)
    if (warp != 0)
        return;
    sel_core(p, v, bad);
    tl_mark(p, 0, true);
}

struct PlanView {  // plan's shared-memory arrays (plan_smem carve-up)
    uint32_t *pre, *pfx, *plan, *cnt, *acc, *misc, *maskP;
    PlanState* st;
};
__device__ __forceinline__ PlanView plan_view(uint32_t* sm, const StepParams& p) {
    const PlanSmem L = plan_smem(p.N, p.K, p.r);
    PlanView v;
    v.pre = sm + L.pre;
    v.pfx = sm + L.pfx;
    v.plan = sm + L.plan;
    v.cnt = sm + L.cnt;
    v.acc = sm + L.acc;
    v.misc = sm + L.misc;
    v.st = reinterpret_cast<PlanState*>(v.misc + 16);
    v.maskP = v.misc + 64;
    return v;
}

// __syncthreads (bar 0) or a named barrier over the first `threads` threads
__device__ __forceinline__ void cta_bar(uint32_t bar, uint32_t threads) {
    if (bar == 0)
        __syncthreads();
    else
        asm volatile("bar.sync %0, %1;" ::"r"(bar), "r"(threads) : "memory");
}

// plan(i) after the size rendezvous (threads [0, T), T >= 32*(N+1), synchronising on barrier
// `bar` — 0 for __syncthreads): the view
// v=i+1 from the table, S4 for every requester (p.plan_out and *v.st updated in place),
// labels of m'_{i+1}'s reps, the push list X_i. v.misc[0] = rendezvous status.
__device__ void plan_core(const StepParams& p, const PlanView& v, uint32_t T, uint32_t bar) {
    uint32_t *pre = v.pre, *pfx = v.pfx, *plan = v.plan, *cnt = v.cnt, *acc = v.acc, *misc = v.misc,
             *maskP = v.maskP;
    PlanState* st = v.st;
    const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const unsigned lt = (1u << lane) - 1u;
    const uint32_t N = p.N, K = p.K, me = p.me, cap = p.cap, r = p.r;
    const uint32_t NK = N * K;
    const uint32_t MJ = plist_mj(N, r);
    // size rendezvous for v = i+1 (size_table.cpp:66-100 / engine.cpp:152): every word of
    // every row at this version (own row from sel(i); peers' rows land over NVLink),
    // bounded by timeout_ns
    const uint64_t* tv1 = reinterpret_cast<const uint64_t*>(p.region[me] + p.off_table) +
                          uint64_t(p.tslot_out) * NK;
    {
        // kU words per thread in flight per pass (each word validates itself: no ordering
        // between them), then a spin only on the words that have not landed yet — one round
        // trip for the whole view instead of one per NK/T words (K = 1000 at c3)
        constexpr uint32_t kU = 16;
        uint64_t t0 = 0;
        uint32_t part = 0;  // this thread's share of the view's total (no separate sum pass)
#pragma unroll 1
        for (uint32_t base = tid; base < NK; base += T * kU) {
            uint64_t w[kU];
#pragma unroll
            for (uint32_t u = 0; u < kU; ++u)
                w[u] = base + u * T < NK ? *reinterpret_cast<const volatile uint64_t*>(tv1 + base + u * T) : 0;
#pragma unroll
            for (uint32_t u = 0; u < kU; ++u) {
                const uint32_t x = base + u * T;
                if (x >= NK)
                    break;
                while (!occ_is(w[u], p.step + 1)) {
                    if (t0 == 0)
                        t0 = globaltimer();
                    else if (globaltimer() - t0 > p.timeout_ns) {
                        misc[0] = DRB_ERR_TRANSPORT;
                        break;
                    }
                    __nanosleep(32);
                    w[u] = *reinterpret_cast<const volatile uint64_t*>(tv1 + x);
                }
                pre[pidx<true>(x)] = occ_of(w[u]);  // (padded: the scan reads stripes)
                part += occ_of(w[u]);
            }
        }
        part = __reduce_add_sync(kFull, part);  // T is a multiple of 32
        if (lane == 0)
            misc[2 + warp] = part;  // misc[2 .. 2 + T/32): per-warp totals (T/32 <= 9)
    }
    cta_bar(bar, T);
    trace_at(p, 6);
    const bool dead = st->error != 0;
    uint32_t* out = p.plist_out;
    if (dead) {
        if (tid < sizeof(PlanState) / 8)
            reinterpret_cast<uint64_t*>(p.plan_out)[tid] = reinterpret_cast<const uint64_t*>(st)[tid];
        if (tid == 0) {
            out[0] = 0;
            out[1] = 0;
        }
        return;
    }
    // S4 plan(i): warps 1..N draw for requester q = warp-1; warp 0 builds the prefix
    unsigned long long pt = 0;
    if (warp == 1)
        prof_span(p, 14, pt);
    if (warp >= 1 && warp <= N) {
        const uint32_t q = warp - 1;
        uint64_t ctr = st->samp_ctr[q];
        const uint32_t total = __reduce_add_sync(kFull, lane < T / 32 ? misc[2 + lane] : 0u);
        if (warp == 1)
        prof_span(p, 14, pt);
        const uint32_t c = warp_plan_draw(p.samp_key[q], ctr, r, total, acc + q * r);
        prof_span(p, 15, pt);
        if (lane == 0) {
            cnt[q] = c;
            p.plan_out->samp_ctr[q] = ctr;
            st->samp_ctr[q] = ctr;
        }
    } else if (warp == 0) {
        warp_exclusive_scan<true>(pre, NK, pfx);
    }
    cta_bar(bar, T);
    if (warp == 1)
        prof_span(p, 16, pt);
    if (warp >= 1 && warp <= N) {
        const uint32_t q = warp - 1;
        warp_locate<true>(acc + q * r, cnt[q], pfx, NK, K, plan + 3 * q * r);
        prof_span(p, 17, pt);
        if (q == me && (p.mode & kModeAssemble)) {  // labels of m'_{i+1}'s reps (stored label == class)
            const uint32_t nslot = (p.aslot + 1) % p.aug_ring;
            uint32_t* al = reinterpret_cast<uint32_t*>(p.region[me] + p.off_auglab) +
                           uint64_t(nslot) * p.auglab_slot_elems;
#pragma unroll 1
            for (uint32_t j = lane; j < cnt[q]; j += 32)
                al[p.nmax + j] = plan[3 * (q * r + j) + 1];
            if (lane == 0)  // |reps(i)|: the rows m'_{i+1} gets after its batch (repcnt, counts_of)
                counts_of(p)[p.aug_ring + nslot] = cnt[q];
        }
        prof_span(p, 18, pt);
    }
    cta_bar(bar, T);
    if (warp == 1)
        prof_span(p, 19, pt);
    trace_at(p, 7);
    // Push list X_i for copy(i): every entry (q, j) of plan(i), over all requesters q (own
    // plan included), whose slot this rank owns, in (q, j) order. copy(i) stores the slot's
    // version-(i+1) bytes into q's m'_{i+1} row nmax+j (sampler.cpp:111-232 serve + fetch,
    // as one-sided stores from the owner).
    const uint32_t NR = N * r;
    uint32_t* jdst = out + 4;
    uint32_t* jrow = out + 4 + MJ;
    for (uint32_t base = warp * 32; base < NR; base += T) {
        const uint32_t e = base + lane;
        bool own = false;
        if (e < NR) {
            const uint32_t q = e / r, j = e - q * r;
            own = j < cnt[q] && plan[3 * e] == me;
        }
        const unsigned m = __ballot_sync(kFull, own);
        if (lane == 0)
            maskP[base >> 5] = m;
    }
    cta_bar(bar, T);
    for (uint32_t base = warp * 32; base < NR; base += T) {
        const unsigned m = maskP[base >> 5];
        if (!((m >> lane) & 1u))
            continue;
        uint32_t pos = __popc(m & lt);
#pragma unroll 1
        for (uint32_t b2 = 0; b2 < (base >> 5); ++b2)
            pos += __popc(maskP[b2]);
        const uint32_t e = base + lane, q = e / r, j = e - q * r;
        jdst[pos] = (q << 24) | j;
        jrow[pos] = plan[3 * e + 1] * cap + plan[3 * e + 2];
    }
    if (tid == 0) {
        uint32_t nj = 0;
#pragma unroll 1
        for (uint32_t b2 = 0; b2 < (NR + 31) / 32; ++b2)
            nj += __popc(maskP[b2]);
        out[0] = cnt[me];
        out[1] = nj;
        p.plan_out->error = misc[0];
        st->error = misc[0];
        if (misc[0] && p.mailbox)  // rendezvous failure: the engine is dead from here
            reinterpret_cast<volatile uint32_t*>(p.mailbox)[kMbSticky] = misc[0];
    }
    trace_at(p, 8);
}

__global__ void drb_plan_next_kernel(const __grid_constant__ StepParams p) {
    extern __shared__ __align__(128) uint32_t sm[];
    const PlanView v = plan_view(sm, p);
    uint32_t* misc = v.misc;
    PlanState* st = v.st;
    const uint32_t tid = threadIdx.x;
    trace_at(p, 5);
    tl_mark(p, 1, false);
    asm volatile("griddepcontrol.wait;" ::: "memory");  // plan(i-1): the sampling counters
    if (tid < sizeof(PlanState) / 8)
        reinterpret_cast<uint64_t*>(st)[tid] = __ldcg(reinterpret_cast<const uint64_t*>(p.plan_in) + tid);
    if (tid == 0)
        misc[0] = 0;
    __syncthreads();
    plan_core(p, v, blockDim.x, 0);  // (the size rendezvous is plan_core's versioned view load)
    tl_mark(p, 1, true);
}

__device__ __forceinline__ void mailbox_fail(const StepParams& p, uint32_t err) {
    if (p.mailbox) {
        volatile uint32_t* mb = p.mailbox;
        mb[mb_err(p.aslot, p.aug_ring)] = err;
        mb[kMbSticky] = err;
    }
}

// ---- copy(i) ------------------------------------------------------------------------------
// m'_i = m_i ++ reps(i-1) is assembled by two launches: copy(i) writes m_i's rows, and
// copy(i-1) of every owner already wrote reps(i-1) into m'_i's representative rows. A rep
// of plan(i) is the content of its slot at version i+1 (S5), i.e. after round i's writes:
// for a slot in W_i that is the winning candidate's batch row, otherwise the slab row as it
// is now (round i does not touch it). So copy(i) reads every slot it serves *while* it
// writes W_i — no read-before-write hazard exists — and stores the bytes straight into the
// requester's m'_{i+1} row nmax+j: its own (HBM) or a peer's (P2P stores over NVLink).
//   A  m_i -> m'_i rows [nmax-n, nmax); a batch row that won a slot also -> its slab row
//   B  push jobs of X_i (plan(i)): version-(i+1) slot bytes -> requester's m'_{i+1} row;
//      without assembly (update_buffer API) the W_i writes instead
// Cross-rank: after its pushes complete, the last CTA of copy(i) release-stores
// pushdone[me] = i+1 into every peer's header; copy(i) does not finish before every
// peer's pushdone >= i (their reps(i-1) rows of m'_i landed). Nothing waits on a peer
// before moving bytes.

// Copy CTA, warp 0: wait for the staged lists (cp.async), resolve each push job's source
// (winner batch row if its slot is written this round, else the slab row) and the
// batch-row -> slab-row map of the fused W_i writes; publish misc[0..1] and the ready flag.
__device__ void copy_parse(const StepParams& p, const uint32_t* xraw, const uint32_t* wraw, uint32_t* jsrc,
                           int* rowmap, uint32_t* misc, volatile uint32_t* ready, bool do_push, bool do_update,
                           bool fuse) {
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t MJ = plist_mj(p.N, p.r);
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncwarp();
    const uint32_t nj = do_push ? xraw[1] : 0;
    const uint32_t n_win = do_update ? wraw[0] : 0;
    const uint32_t* jrow = xraw + 4 + MJ;
    if (n_win <= 32) {  // lane t holds winner t's slot; one ballot per job (winners hold distinct slots)
        const uint32_t wslot = lane < n_win ? wraw[3 + 2 * lane] : ~0u;
#pragma unroll 1
        for (uint32_t x = 0; x < nj; ++x) {
            const uint32_t row = jrow[x];
            const unsigned hit = __ballot_sync(kFull, wslot == row);
            if (lane == 0)
                jsrc[x] = hit ? 0x80000000u | wraw[2 + 2 * (__ffs(hit) - 1)] : row;
        }
    } else {
#pragma unroll 1
        for (uint32_t x = lane; x < nj; x += 32) {
            const uint32_t row = jrow[x];
            uint32_t src = row;
#pragma unroll 1
            for (uint32_t t = 0; t < n_win; ++t)
                if (wraw[3 + 2 * t] == row) {
                    src = 0x80000000u | wraw[2 + 2 * t];
                    break;
                }
            jsrc[x] = src;
        }
    }
    if (fuse) {
#pragma unroll 1
        for (uint32_t x = lane; x < p.n; x += 32)
            rowmap[x] = -1;
        __syncwarp();
#pragma unroll 1
        for (uint32_t t = lane; t < n_win; t += 32)
            rowmap[wraw[2 + 2 * t]] = static_cast<int>(wraw[3 + 2 * t]);
    }
    if (lane == 0) {
        misc[0] = nj;
        misc[1] = fuse ? 0u : n_win;
    }
    __syncwarp();
    __threadfence_block();
    if (lane == 0) {
        *ready = 1;
        cta_mark(p, 1);
    }
    trace_at(p, 20);
}

// CTA 0, warp 0, after griddepcontrol.wait: m'_i's batch labels, its row count
// n + |reps(i-1)| (|reps(i-1)| left by copy(i-1) in repcnt) and |reps(i)| for copy(i+1).
__device__ void copy_counts(const StepParams& p, const uint32_t* xraw) {
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t row0 = p.nmax - p.n;
    uint32_t* al = reinterpret_cast<uint32_t*>(p.region[p.me] + p.off_auglab) + uint64_t(p.aslot) * p.auglab_slot_elems;
#pragma unroll 1
    for (uint32_t x = lane; x < p.n; x += 32)
        al[row0 + x] = __ldg(p.labels + x);
    if (lane == 0) {
        uint32_t* aug_count = counts_of(p);
        uint32_t* repcnt = aug_count + p.aug_ring;
        const uint32_t prev = p.step > 0 ? repcnt[p.aslot] : 0u;
        aug_count[p.aslot] = p.n + prev;
        repcnt[(p.aslot + 1) % p.aug_ring] = xraw[0];
        if (p.mailbox) {
            volatile uint32_t* mb = p.mailbox;
            mb[mb_count(p.aslot)] = p.n + prev;
            mb[mb_err(p.aslot, p.aug_ring)] = 0;
        }
    }
}

// Multi-rank hand-off of the pushes:
//   copy(i) start (CTA 0, warp 0, after griddepcontrol.wait: copy(i-1) complete, so are its
//     stores into the peers' m'_i — kernel completion): pushdone[me] = i at every peer,
//     after a system fence;
//   peers_wait(i), a one-warp kernel off the copy chain: every peer announced pushdone >= i
//     (their reps(i-1) rows of my m'_i landed). The consumer's "m'_i ready" event follows it,
//     so no copy ever waits on a peer's progress.
__device__ void copy_announce_peers(const StepParams& p) {
    const uint32_t lane = threadIdx.x & 31;
    if (p.step == 0)
        return;
    __threadfence_system();
    __syncwarp();
    if (lane < p.N && lane != p.me)
        st_release_sys(&reinterpret_cast<RegionHeader*>(p.region[lane])->pushdone[p.me], p.step);
}
__device__ void copy_wait_peers(const StepParams& p) {
    const uint32_t lane = threadIdx.x & 31;
    RegionHeader* hdr = reinterpret_cast<RegionHeader*>(p.region[p.me]);
    if (p.step == 0)
        return;
    bool ok = true;
    if (lane < p.N && lane != p.me)
        ok = wait_flag(&hdr->pushdone[lane], p.step, p.timeout_ns);
    if (__any_sync(kFull, !ok) && lane == 0)
        mailbox_fail(p, DRB_ERR_TRANSPORT);
}

__global__ void peers_wait_kernel(const __grid_constant__ StepParams p) {
    if (threadIdx.x < 32)
        copy_wait_peers(p);
}

__device__ __forceinline__ uint8_t* push_dst(const StepParams& p, uint32_t dst, uint32_t next_slot) {
    const uint32_t q = dst >> 24, j = dst & 0xffffffu;
    return p.region[q] + p.off_aug + uint64_t(next_slot) * p.aug_slot_bytes + uint64_t(p.nmax + j) * p.S;
}

// LSU path (any S % 4 == 0): grid-stride vector copies over the same lists.
template <typename V>
__global__ void __launch_bounds__(kThreads, 1) drb_copy_kernel(const __grid_constant__ StepParams p) {
    extern __shared__ __align__(128) uint32_t sm[];
    const CopySmem L = copy_smem(p.N, p.r, p.nmax);
    uint32_t* xraw = sm + L.xraw;
    uint32_t* wraw = sm + L.wraw;
    uint32_t* jsrc = sm + L.jsrc;
    int* rowmap = reinterpret_cast<int*>(sm + L.rowmap);
    uint32_t* misc = sm + L.misc;
    volatile uint32_t* ready = misc + 6;

    const uint32_t tid = threadIdx.x, warp = tid >> 5;
    const uint32_t N = p.N, me = p.me, n = p.n;
    const uint64_t S = p.S;
    const uint32_t nvec = static_cast<uint32_t>(S / sizeof(V));
    const bool do_assemble = p.mode & kModeAssemble;
    const bool do_push = (p.mode & kModePlan) && p.plist_in;
    const bool do_update = p.mode & kModeUpdate;
    const bool multi = (p.mode & kModePeers) && N > 1;
    const uint32_t part = blockIdx.x, parts = gridDim.x;
    const V* batch = reinterpret_cast<const V*>(p.batch);
    V* slab = reinterpret_cast<V*>(p.slab);
    V* asm_dst = reinterpret_cast<V*>(p.region[me] + p.off_aug + uint64_t(p.aslot) * p.aug_slot_bytes) +
                 uint64_t(p.nmax - n) * nvec;
    const uint32_t next_slot = (p.aslot + 1) % p.aug_ring;
    const uint32_t* jdst = xraw + 4;

    tl_mark(p, 2, false);
    if (tid == 0)
        cta_mark(p, 0);
    asm volatile("griddepcontrol.launch_dependents;");
    if (tid < 16)
        misc[tid] = 0;
    const uint32_t pw = do_push ? plist_words(N, p.r) : 0;
    const uint32_t ww = do_update ? wlist_words(p.nmax) : 0;
    if (warp == 0) {
#pragma unroll 1
        for (uint32_t x = tid; x < pw; x += 32)
            asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(xraw + x))),
                         "l"(p.plist_in + x)
                         : "memory");
#pragma unroll 1
        for (uint32_t x = tid; x < ww; x += 32)
            asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(wraw + x))),
                         "l"(p.wlist + x)
                         : "memory");
        asm volatile("cp.async.commit_group;" ::: "memory");
    }
    __syncthreads();
    const bool fuse = do_assemble;
    if (warp == 0) {
        copy_parse(p, xraw, wraw, jsrc, rowmap, misc, ready, do_push, do_update, fuse);
        if (blockIdx.x == 0) {
            asm volatile("griddepcontrol.wait;" ::: "memory");
            if (multi)
                copy_announce_peers(p);
            if (do_assemble)
                copy_counts(p, xraw);
        }
    }
    __syncthreads();
    asm volatile("griddepcontrol.wait;" ::: "memory");  // copy(i-1) complete (slab at version i)
    // A: m_i -> m'_i (+ fused W_i slab writes)
    const uint32_t tva = do_assemble ? n * nvec : 0;
    const uint32_t alo = static_cast<uint32_t>(uint64_t(tva) * part / parts);
    const uint32_t ahi = static_cast<uint32_t>(uint64_t(tva) * (part + 1) / parts);
    constexpr int U = sizeof(V) == 16 ? 4 : 8;
#pragma unroll 1
    for (uint32_t g0 = alo + tid; g0 < ahi; g0 += U * kThreads) {
        V v[U];
#pragma unroll
        for (int u = 0; u < U; ++u)
            if (g0 + u * kThreads < ahi)
                v[u] = ld_vec(batch + g0 + u * kThreads);
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint32_t gv = g0 + u * kThreads;
            if (gv < ahi) {
                asm_dst[gv] = v[u];
                const uint32_t row = gv / nvec;
                const int key = rowmap[row];
                if (key >= 0)
                    slab[uint64_t(key) * nvec + (gv - row * nvec)] = v[u];
            }
        }
    }
    if (tid == 32)
        cta_mark(p, 5);
    // B: push jobs, then (no assembly) the W_i writes
    const uint32_t nj = misc[0], nw = misc[1];
    const uint32_t pv = nj * nvec;
    const uint32_t tvb = pv + nw * nvec;
    const uint32_t blo = static_cast<uint32_t>(uint64_t(tvb) * part / parts);
    const uint32_t bhi = static_cast<uint32_t>(uint64_t(tvb) * (part + 1) / parts);
#pragma unroll 1
    for (uint32_t gv = blo + tid; gv < bhi; gv += kThreads) {
        if (gv < pv) {
            const uint32_t x = gv / nvec, o = gv - x * nvec;
            const uint32_t s = jsrc[x];
            const V* src = (s >> 31) ? batch + uint64_t(s & 0x7fffffffu) * nvec : slab + uint64_t(s) * nvec;
            reinterpret_cast<V*>(push_dst(p, jdst[x], next_slot))[o] = ld_vec(src + o);
        } else {
            const uint32_t t = (gv - pv) / nvec, o = (gv - pv) - t * nvec;
            slab[uint64_t(wraw[3 + 2 * t]) * nvec + o] = ld_vec(batch + uint64_t(wraw[2 + 2 * t]) * nvec + o);
        }
    }
    if (tid == 32)
        cta_mark(p, 6);
    if (p.timeline) {
        __syncthreads();
        tl_mark(p, 2, true);
        if (tid == 0)
            cta_mark(p, 7);
    }
}

// ---- TMA bulk-copy path (S % 16 == 0) ---------------------------------------------------
// The same copy(i) moved by the SM's TMA engine: 1-D cp.async.bulk global->shared
// (mbarrier completion) and shared->global (bulk groups), so the bytes in flight per SM
// are bounded by the shared-memory ring, not by the L1 miss-tracking capacity that
// throttles 16-byte vector loads. Two elected threads issue everything:
//   warp 1 lane 0  A: batch slice -> ring -> m'_i rows; after griddepcontrol.wait the same
//                  ring bytes -> slab rows of the W_i winners (rowmap)
//   warp 0         staged lists (copy_parse), CTA 0's counts; lane 0 B: push jobs
//                  (slot bytes -> ring -> requester's m'_{i+1} row, local HBM or a peer's)
//                  and, without assembly, the W_i writes
// Everything before griddepcontrol.wait (list staging and parsing, A's loads and m'_i
// stores) is independent of copy(i-1), so under PDL it overlaps copy(i-1)'s tail: the
// kernel is sized (<= half an SM's shared memory) for two co-resident CTAs.
__device__ __forceinline__ uint64_t min64(uint64_t a, uint64_t b) { return a < b ? a : b; }
__device__ __forceinline__ uint32_t smem_u32(const void* ptr) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(ptr));
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes)
                 : "memory");
}
// Wait for phase `parity` of barrier b to complete. Bounded: a bulk copy that never lands
// (a fault) must not hang the GPU — after timeout_ns the wait gives up and returns false.
__device__ __forceinline__ bool mbar_wait(uint64_t* b, uint32_t parity, uint64_t timeout_ns = 4000000000ull) {
    uint32_t ok = 0;
    uint64_t t0 = 0;
    for (uint32_t spin = 0;; ++spin) {
        asm volatile(
            "{\n .reg .pred q;\n mbarrier.try_wait.parity.shared::cta.b64 q, [%1], %2;\n selp.u32 %0, 1, 0, q;\n}"
            : "=r"(ok)
            : "r"(smem_u32(b)), "r"(parity)
            : "memory");
        if (ok)
            return true;
        if (spin == 64)
            t0 = globaltimer();
        else if (spin > 64 && (spin & 63) == 0 && globaltimer() - t0 > timeout_ns)
            return false;
    }
}
// Per-barrier phase bits of an engine thread: barrier x of a ring is waited on with bit x,
// which then flips (a partially used window leaves the other barriers' phases alone).
__device__ __forceinline__ uint32_t take_phase(uint32_t& bits, uint32_t x) {
    const uint32_t ph = (bits >> x) & 1u;
    bits ^= 1u << x;
    return ph;
}

__device__ __forceinline__ void bulk_load(void* dst_smem, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst_smem)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void bulk_store(void* dst, const void* src_smem, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src_smem)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read_all() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

__global__ void __launch_bounds__(kTmaThreads, 1) drb_copy_tma_kernel(const __grid_constant__ StepParams p) {
    extern __shared__ __align__(128) uint32_t sm[];
    const CopySmem L = copy_smem(p.N, p.r, p.nmax);
    uint32_t* xraw = sm + L.xraw;
    uint32_t* wraw = sm + L.wraw;
    uint32_t* jsrc = sm + L.jsrc;
    int* rowmap = reinterpret_cast<int*>(sm + L.rowmap);
    uint32_t* misc = sm + L.misc;
    const TmaSmem T = tma_smem(p.N, p.r, p.nmax);
    uint64_t* bars = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(sm) + T.bars);
    uint8_t* ring = reinterpret_cast<uint8_t*>(sm) + T.ring;

    const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t N = p.N, me = p.me, n = p.n;
    const uint64_t S = p.S;
    const bool do_assemble = p.mode & kModeAssemble;
    const bool do_push = (p.mode & kModePlan) && p.plist_in;
    const bool do_update = p.mode & kModeUpdate;
    const bool multi = (p.mode & kModePeers) && N > 1;
    const uint32_t part = blockIdx.x, parts = gridDim.x;
    const uint8_t* batch = reinterpret_cast<const uint8_t*>(p.batch);
    uint8_t* slab = reinterpret_cast<uint8_t*>(p.slab);
    uint8_t* my_aug = p.region[me] + p.off_aug + uint64_t(p.aslot) * p.aug_slot_bytes;
    const uint32_t next_slot = (p.aslot + 1) % p.aug_ring;
    const uint32_t row0 = p.nmax - n;
    const uint32_t* jdst = xraw + 4;
    volatile uint32_t* ready = misc + 6;

    tl_mark(p, 2, false);
    if (tid == 0)
        cta_mark(p, 0);
    asm volatile("griddepcontrol.launch_dependents;");
    if (tid < 16)
        misc[tid] = 0;
    if (tid == 0 || tid == 32) {  // each engine thread owns its barriers
        const uint32_t b0 = tid == 0 ? kTmaStagesA : 0, b1 = tid == 0 ? kTmaStages : kTmaStagesA;
        for (uint32_t b = b0; b < b1; ++b)
            mbar_init(bars + b, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    const uint32_t pw = do_push ? plist_words(N, p.r) : 0;
    const uint32_t ww = do_update ? wlist_words(p.nmax) : 0;
    if (warp == 0) {
#pragma unroll 1
        for (uint32_t x = lane; x < pw; x += 32)
            asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(xraw + x)), "l"(p.plist_in + x)
                         : "memory");
#pragma unroll 1
        for (uint32_t x = lane; x < ww; x += 32)
            asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(wraw + x)), "l"(p.wlist + x)
                         : "memory");
        asm volatile("cp.async.commit_group;" ::: "memory");
    }
    __syncthreads();  // misc / ready zeroed, barriers initialised, list loads issued
    if (tid == 32)
        cta_mark(p, 8);

    const uint32_t CH = kTmaChunk;
    if (warp == 1) {
        // ---- A engine: batch bytes [alo, ahi) of this CTA -> m'_i (+ W_i winners' slab rows) ----
        if (lane == 0) {
            const uint64_t a16 = (do_assemble && !(p.dbg & 128)) ? (uint64_t(n) * S) >> 4 : 0;  // 128: no bytes
            const uint64_t alo = (a16 * part / parts) << 4, ahi = (a16 * (part + 1) / parts) << 4;
            const uint32_t nA = static_cast<uint32_t>((ahi - alo + CH - 1) / CH);
            uint8_t* dst = my_aug + uint64_t(row0) * S;
            uint32_t ph_bits = 0;  // phase of each A barrier
            bool lists = false;
            for (uint32_t w0 = 0; w0 < nA; w0 += kTmaStagesA) {
                const uint32_t w1 = min(nA, w0 + kTmaStagesA);
                if (w0 > 0)
                    bulk_wait_read_all();  // the ring's previous window has been stored
                for (uint32_t k = w0; k < w1; ++k) {
                    const uint64_t off = alo + uint64_t(k) * CH;
                    const uint32_t len = static_cast<uint32_t>(min64(CH, ahi - off));
                    uint64_t* bar = bars + (k - w0);
                    mbar_expect_tx(bar, len);
                    bulk_load(ring + (k - w0) * CH, batch + off, len, bar);
                }
                if (w0 == 0)
                    cta_mark(p, 2);
                for (uint32_t k = w0; k < w1; ++k) {  // m'_i rows as soon as each piece lands
                    const uint64_t off = alo + uint64_t(k) * CH;
                    const uint32_t len = static_cast<uint32_t>(min64(CH, ahi - off));
                    if (!mbar_wait(bars + (k - w0), take_phase(ph_bits, k - w0)))
                        mailbox_fail(p, DRB_ERR_INTERNAL);
                    if (k == 0)
                        cta_mark(p, 11);
                    bulk_store(dst + off, ring + (k - w0) * CH, len);
                }
                bulk_commit();
                if (w0 == 0)
                    cta_mark(p, 5);
                if (!lists) {  // slab rows: after copy(i-1) (its reads of them) and the lists
                    asm volatile("griddepcontrol.wait;" ::: "memory");
                    while (*ready == 0)
                        __nanosleep(20);
                    __threadfence_block();
                    lists = true;
                    cta_mark(p, 3);
                }
                for (uint32_t k = w0; k < w1; ++k) {  // W_i winners among these rows
                    uint64_t off = alo + uint64_t(k) * CH;
                    const uint64_t end = off + min64(CH, ahi - off);
                    while (off < end) {
                        const uint32_t row = static_cast<uint32_t>(off / S);
                        const uint64_t rend = min64(end, uint64_t(row + 1) * S);
                        const int key = rowmap[row];
                        if (key >= 0)
                            bulk_store(slab + uint64_t(key) * S + (off - uint64_t(row) * S),
                                       ring + (k - w0) * CH + (off - (alo + uint64_t(k) * CH)),
                                       static_cast<uint32_t>(rend - off));
                        off = rend;
                    }
                }
                bulk_commit();
            }
            bulk_wait_read_all();
            cta_mark(p, 6);
        }
    } else if (warp == 0) {
        copy_parse(p, xraw, wraw, jsrc, rowmap, misc, ready, do_push, do_update, do_assemble);
        asm volatile("griddepcontrol.wait;" ::: "memory");  // copy(i-1) complete: slab at version i
        if (lane == 0)
            cta_mark(p, 10);
        if (multi && blockIdx.x == 0)
            copy_announce_peers(p);
        if (blockIdx.x == 0 && do_assemble)
            copy_counts(p, xraw);
        if (lane == 0) {
            // ---- B engine: push jobs (+ non-fused W_i writes) ----
            uint8_t* ringB = ring + kTmaStagesA * CH;
            uint64_t* barB = bars + kTmaStagesA;
            const uint32_t nj = misc[0];
            const uint64_t pv = uint64_t(nj) * S;
            const uint64_t sv = uint64_t(misc[1]) * S;
            const uint64_t b16 = (p.dbg & 128) ? 0 : (pv + sv) >> 4;
            const uint64_t blo = (b16 * part / parts) << 4, bhi = (b16 * (part + 1) / parts) << 4;
            uint32_t use = 0;      // window count
            uint32_t ph_bits = 0;  // phase of each B barrier
            uint64_t off = blo;
            while (off < bhi) {
                // one window: up to kTmaStagesB pieces, each inside one row and <= CH
                uint64_t poff[kTmaStagesB];
                uint32_t plen[kTmaStagesB], m = 0;
                while (m < kTmaStagesB && off < bhi) {
                    const bool is_job = off < pv;
                    const uint64_t base = is_job ? 0 : pv;
                    const uint32_t j = static_cast<uint32_t>((off - base) / S);
                    const uint64_t rend = min64(bhi, base + uint64_t(j + 1) * S);
                    const uint32_t len = static_cast<uint32_t>(min64(CH, rend - off));
                    const uint64_t o = off - base - uint64_t(j) * S;
                    const uint8_t* src;
                    if (is_job) {
                        const uint32_t s = jsrc[j];
                        src = ((s >> 31) ? batch + uint64_t(s & 0x7fffffffu) * S : slab + uint64_t(s) * S) + o;
                    } else {
                        src = batch + uint64_t(wraw[2 + 2 * j]) * S + o;
                    }
                    poff[m] = off;
                    plen[m] = len;
                    mbar_expect_tx(barB + m, len);
                    bulk_load(ringB + m * CH, src, len, barB + m);
                    off += len;
                    ++m;
                }
                if (use == 0)
                    cta_mark(p, 4);
                for (uint32_t x = 0; x < m; ++x) {
                    const bool is_job = poff[x] < pv;
                    const uint64_t base = is_job ? 0 : pv;
                    const uint32_t j = static_cast<uint32_t>((poff[x] - base) / S);
                    const uint64_t o = poff[x] - base - uint64_t(j) * S;
                    uint8_t* dst = is_job ? push_dst(p, jdst[j], next_slot) + o
                                          : slab + uint64_t(wraw[3 + 2 * j]) * S + o;
                    if (!mbar_wait(barB + x, take_phase(ph_bits, x)))
                        mailbox_fail(p, DRB_ERR_INTERNAL);
                    bulk_store(dst, ringB + x * CH, plen[x]);
                }
                bulk_commit();
                bulk_wait_read_all();  // the ring is reused by the next window
                ++use;
            }
            cta_mark(p, 9);
        }
    }
    asm volatile("griddepcontrol.wait;" ::: "memory");
    __syncthreads();  // all bulk stores of this CTA issued and sourced
    if (p.timeline) {
        __syncthreads();
        tl_mark(p, 2, true);
        if (tid == 0)
            cta_mark(p, 7);
    }
}

// ---- resident engine (drb_rb_step / drb_rb_run) ---------------------------------
// One cooperative instance (all CTAs co-resident) stays resident while work is posted: CTA 0
// loops the sel chain (warps 0-3), the feeder (warp 4) and the ready publisher (warp 5); CTA 1
// the plan chain; CTAs 2.. the copies. The hand-offs that the three-kernel path expresses as
// launches and stream events are device counters in RunCtl (absolute: i+1 once iteration i's
// role finished). Work arrives as descriptors (FeedDesc) written by stream-ordered memory
// operations on the caller's stream; the feeder admits their steps in order, every role
// follows `admitted`. The selection / sampling state stays in shared memory across
// iterations, the next labels are fetched while the current selection runs, and nothing is
// launched per step. Every decision is the same code as the three-kernel path (sel_core,
// plan_core, copy_parse, the push-at-source copy), so the outputs are bit-identical.
//   sel(i)   waits B(i-8) (W slot), plan(i-4) (table slot); multi-rank B(i-6) of every rank
//            (the pushes into the m' slot that plan(i)'s requesters refill)
//   plan(i)  waits sel(i), B(i-8) (X slot), peers' occupancy rows v=i+1
//   A(i)     (batch -> m'_i) waits B(i-R+1) (its ring slot's previous m' is complete)
//   B(i)     (W_i writes, X_i pushes, by byte column) waits sel(i), plan(i) only
//   ready(i) (m'_i complete: the consumer's stream wait) = A(i), B(i) on every copy CTA and,
//            multi-rank, every peer's B(i-1) (its pushes of reps(i-1) into m'_i)
// An instance leaves once it has been idle (everything admitted is ready, nothing posted)
// for idle_ns, after a handshake with the host over mapped memory (the host relaunches when
// it posts behind a leaving instance); every role stops at the same iteration, and the next
// instance resumes there.
__device__ __forceinline__ uint64_t ld_acquire_gpu(const uint64_t* p) {
    uint64_t v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_gpu(uint64_t* p, uint64_t v) {
    asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ bool run_failed(const RunParams& rp) {
    return *reinterpret_cast<volatile const uint32_t*>(&rp.ctl->error) != 0;
}
// Fail the engine (first failure wins the diagnostics) and make it visible to the host.
__device__ void run_fail(const RunParams& rp, uint32_t err, uint32_t where) {
    if (atomicCAS(&rp.ctl->error, 0u, err) == 0)
        rp.ctl->where = where;
    if (rp.base.mailbox) {
        volatile uint32_t* mb = rp.base.mailbox;
        mb[kMbSticky] = err;
    }
}

// *f >= want, or false once the engine failed / the wait timed out (then the engine fails).
// Only waits on admitted iterations use this: those complete unless a peer stalls.
__device__ bool run_wait(const uint64_t* f, uint64_t want, const RunParams& rp, bool sys, uint64_t* got = nullptr) {
    uint64_t v = sys ? ld_acquire_sys(f) : ld_acquire_gpu(f);
    if (v >= want) {  // satisfied: no timer read
        if (got)
            *got = v;
        return true;
    }
    const uint64_t t0 = globaltimer();
    for (;;) {
        v = sys ? ld_acquire_sys(f) : ld_acquire_gpu(f);
        if (v >= want) {
            if (got)
                *got = v;
            return true;
        }
        if (run_failed(rp))
            return false;
        if (globaltimer() - t0 > rp.base.timeout_ns) {
            run_fail(rp, DRB_ERR_TRANSPORT, (9u << 24) | uint32_t(want & 0xffffff));
            return false;
        }
        __nanosleep(20);
    }
}
__device__ __forceinline__ uint64_t back(uint64_t k, uint64_t d) { return k >= d ? k - d : 0; }

// Every peer's word words[w] >= want (w != me, w < N), one thread. `seen` caches the smallest
// value observed (peers advance in lockstep, so one look usually covers many later waits). The
// words are read with relaxed loads issued together (one round trip for all peers, not one
// acquire each); a word still short is then waited for (bounded, acquire). With `fence`, one
// fence.acq_rel.sys after a fresh look is the acquire for the relaxed reads (a system fence
// costs microseconds: callers that publish with a system-scope release next pass false — the
// release's fence follows the reads).
__device__ bool wait_peers(const uint64_t* words, uint32_t N, uint32_t me, uint64_t want, const RunParams& rp,
                           uint64_t& seen, bool fence) {
    if (seen >= want)
        return true;
    uint64_t v[kMaxWorld];
#pragma unroll
    for (uint32_t w = 0; w < kMaxWorld; ++w) {
        v[w] = ~0ull;
        if (w < N && w != me)
            asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v[w]) : "l"(words + w) : "memory");
    }
    uint64_t lo = ~0ull;
#pragma unroll
    for (uint32_t w = 0; w < kMaxWorld; ++w) {
        if (v[w] < want && !run_wait(words + w, want, rp, true, &v[w]))
            return false;
        lo = v[w] < lo ? v[w] : lo;
    }
    if (fence)
        asm volatile("fence.acq_rel.sys;" ::: "memory");
    seen = lo;
    return true;
}

// Iteration i is admitted (its descriptor is visible), or false: this instance stops at or
// before i, or the engine failed. Unbounded: an idle engine waits here for the next post.
__device__ bool wait_admit(const RunParams& rp, uint64_t& seen, uint64_t i) {
    if (seen > i)
        return true;
#pragma unroll 1
    for (uint32_t spin = 0;; ++spin) {
        seen = ld_acquire_gpu(&rp.ctl->admitted);
        if (seen > i)
            return true;
        const uint64_t st = *reinterpret_cast<volatile const uint64_t*>(&rp.ctl->stop_at);
        if ((st >> 40) == (rp.gen & 0xffffffu) && (st & kStopMask) <= i)
            return false;
        if (run_failed(rp))
            return false;
        __nanosleep(spin < 256 ? 32 : 256);
    }
}

// The descriptor holding iteration i (roles advance through the ring in order).
struct FeedCursor {
    uint64_t j, ib;
    uint32_t cnt, n, ring, first;
    bool early;  // kDescEarly
    const uint8_t* batches;
    const uint32_t* labels;
    uint64_t bstride, lstride;
};
__device__ __forceinline__ void cursor_init(FeedCursor& c, uint64_t i0, uint64_t j0) {
    c.j = j0 - 1;  // (wraps for j0 = 0; the first seek advances to j0)
    c.ib = i0;
    c.cnt = 0;
}
__device__ void cursor_seek(FeedCursor& c, const RunParams& rp, uint64_t i) {
    while (i >= c.ib + c.cnt) {
        ++c.j;
        const FeedDesc* d = rp.feed + (c.j % kFeedRing);
        c.batches = reinterpret_cast<const uint8_t*>(__ldcg(&d->batches));
        c.labels = reinterpret_cast<const uint32_t*>(__ldcg(&d->labels));
        c.bstride = __ldcg(&d->batch_stride);
        c.lstride = __ldcg(&d->label_stride);
        c.ib = __ldcg(&d->i_begin);
        const uint64_t cn = __ldcg(&d->count_n), rf = __ldcg(&d->ring_first);
        c.cnt = static_cast<uint32_t>(cn);
        c.n = static_cast<uint32_t>(cn >> 32) & 0x3fffffffu;
        c.early = (cn & kDescEarly) != 0;
        c.ring = static_cast<uint32_t>(rf);
        c.first = static_cast<uint32_t>(rf >> 32);
    }
}
__device__ __forceinline__ uint64_t cursor_slot(const FeedCursor& c, uint64_t i) {
    return (c.first + static_cast<uint32_t>(i - c.ib)) % c.ring;
}
__device__ __forceinline__ const uint8_t* cursor_batch(const FeedCursor& c, uint64_t i) {
    return c.batches + cursor_slot(c, i) * c.bstride;
}
__device__ __forceinline__ const uint32_t* cursor_labels(const FeedCursor& c, uint64_t i) {
    return c.labels + cursor_slot(c, i) * c.lstride;
}

// StepParams of engine iteration i, as iter_params() on the host (batch fields: feed_patch)
__device__ void run_patch(StepParams& p, const RunParams& rp, uint64_t i) {
    const uint64_t v = rp.ver0 + i;
    p.tslot_in = static_cast<uint32_t>(v % kTableRing);
    p.tslot_out = static_cast<uint32_t>((v + 1) % kTableRing);
    p.sel_in = rp.sel_base + ((rp.sel_par0 + i) & 1);
    p.sel_out = rp.sel_base + ((rp.sel_par0 + i + 1) & 1);
    p.plan_in = rp.plan_base + ((rp.plan_par0 + i) & 1);
    p.plan_out = rp.plan_base + ((rp.plan_par0 + i + 1) & 1);
    p.step = i;
    p.seq = i;
    p.aslot = ring_slot(i, p.aug_ring);
    p.plist_in = rp.plist_base + (i % kListRing) * rp.pw;
    p.plist_out = const_cast<uint32_t*>(p.plist_in);
    p.wlist = rp.wlist_base + (i % kListRing) * rp.ww;
}
__device__ __forceinline__ void feed_patch(StepParams& p, const FeedCursor& c, uint64_t i) {
    p.batch = cursor_batch(c, i);
    p.labels = cursor_labels(c, i);
    p.n = c.n;
}

// per-CTA timeline stamp of engine iteration i (timeline mode), any thread
__device__ __forceinline__ void run_mark(const RunParams& rp, uint64_t i, int slot) {
#if DRB_INSTRUMENT
    const StepParams& p = rp.base;
    if (p.timeline && blockIdx.x < kTlMaxCtas)
        p.timeline[(i & (p.timeline_steps - 1)) * kTlStride + 32 + blockIdx.x * kTlCtaSlots + slot] = globaltimer();
#endif
}

__device__ __forceinline__ void named_bar(uint32_t id, uint32_t threads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(threads) : "memory");
}

// Per-round timing stamp (drb_rb_drain_timings), one thread, only when enabled.
__device__ __forceinline__ void tstamp(const RunParams& rp, uint64_t i, uint32_t slot) {
    if (rp.timings)
        rp.timings[(i % kTimingRing) * kTimingWords + slot] = globaltimer();
}

// Waits on run counters keep the last value seen, so a satisfied wait costs no memory trip.
struct SeenFlag {
    const uint64_t* f;
    uint64_t seen;
};
__device__ __forceinline__ bool wait_seen(SeenFlag& s, uint64_t want, const RunParams& rp, bool sys = false) {
    if (s.seen >= want)
        return true;
    return run_wait(s.f, want, rp, sys, &s.seen);  // (the value that satisfied the wait: no second load)
}

__device__ __forceinline__ bool poll_seen(SeenFlag& s, uint64_t want) {  // one acquire load at most
    if (s.seen >= want)
        return true;
    s.seen = ld_acquire_gpu(s.f);
    return s.seen >= want;
}

__device__ __forceinline__ void st_release_cta(volatile unsigned long long* p, uint64_t v) {
    asm volatile("st.release.cta.shared.u64 [%0], %1;" ::"r"(smem_u32(const_cast<unsigned long long*>(p))), "l"(v)
                 : "memory");
}
__device__ __forceinline__ uint64_t ld_acquire_cta(const volatile unsigned long long* p) {
    uint64_t v;
    asm volatile("ld.acquire.cta.shared.u64 %0, [%1];" : "=l"(v) : "r"(smem_u32(const_cast<unsigned long long*>(p)))
                 : "memory");
    return v;
}

// A publisher warp (lane 0) for a control CTA: whenever the compute warps hand over
// iteration k (smem `ready` = k+1, release at CTA scope), it release-stores the run counter
// (`done` = i0+k+1, GPU scope — this is the store that waits for the compute warps' global
// writes to be acknowledged, so they don't) and refreshes the counters the compute warps
// check next (`seen`, acquire). It leaves when the compute warps raise `stop`.
__device__ void run_publisher(const RunParams& rp, uint64_t i0, volatile unsigned long long* ready, uint64_t* done,
                              volatile unsigned long long* seen, const uint64_t* s0, const uint64_t* s1,
                              volatile const uint32_t* stop) {
#pragma unroll 1
    for (uint64_t k = 0;; ++k) {
#pragma unroll 1
        for (uint32_t spin = 0; ld_acquire_cta(ready) < k + 1; ++spin) {
            if (*stop) {  // the role left: publish a hand-over that raced with the stop, then leave
                __threadfence_block();
                if (ld_acquire_cta(ready) >= k + 1)
                    break;
                return;
            }
            if ((spin & 63) == 63 && run_failed(rp))
                return;
            seen[0] = ld_acquire_gpu(s0);  // keep the compute warps' view fresh while waiting
            seen[1] = ld_acquire_gpu(s1);
            if (spin > 4096)  // idle engine: back off
                __nanosleep(256);
        }
        st_release_gpu(done, i0 + k + 1);
        seen[0] = ld_acquire_gpu(s0);
        seen[1] = ld_acquire_gpu(s1);
    }
}

// The feeder (one lane): admits posted descriptors in order, and ends the instance when idle.
__device__ void run_feeder(const RunParams& rp, uint64_t i0, uint64_t j0) {
    // The whole warp runs this loop in lockstep (every value below is warp-uniform). Lanes 0-7
    // poll the sequence words of the next eight descriptors together; the posted prefix of them
    // is fetched in one PCIe round trip (four 16-byte reads per descriptor, on lanes 4d..4d+3)
    // and admitted in order, so a producer that runs ahead is admitted a batch at a time.
    const uint32_t lane = threadIdx.x & 31;
    uint64_t j = j0, admitted = i0, idle_t0 = 0;
    uint64_t released = i0;  // m' below this are released by implicit (single-stream) posts
    bool failed = false;
    const uint32_t R = rp.base.aug_ring;
    constexpr uint32_t kBatch = 32 / (kFeedDescWords / 2);  // descriptors per round trip
#pragma unroll 1
    for (uint32_t spin = 0;; ++spin) {
        uint32_t posted = 0;
        if (lane < kBatch)
            posted = ld_acquire_sys(rp.feed_seq + ((j + lane) % kFeedRing)) == j + lane + 1;  // stream order
        const uint32_t cnt = __ffs(~__ballot_sync(kFull, posted)) - 1;  // posted prefix j .. j+cnt-1
        if (cnt > 0) {
            __syncwarp();  // (the polling lanes' acquires order every lane's descriptor reads)
            // the descriptors from mapped host memory, then the device mirror the roles read
            const uint32_t d = lane / (kFeedDescWords / 2), part = lane % (kFeedDescWords / 2);
            uint64_t lo = 0, hi = 0;
            if (d < cnt) {
                const uint64_t* hs = reinterpret_cast<const uint64_t*>(rp.hdesc + ((j + d) % kFeedRing));
                asm volatile("ld.relaxed.sys.global.v2.u64 {%0, %1}, [%2];" : "=l"(lo), "=l"(hi) : "l"(hs + 2 * part)
                             : "memory");
            }
            uint64_t consumed = 0;
            if (lane == 0)
                consumed = ld_acquire_sys(&rp.ctl->consumed);
            consumed = __shfl_sync(kFull, consumed, 0);
            uint32_t took = 0;
            bool blocked = false;
#pragma unroll 1
            for (; took < cnt; ++took) {
                uint64_t w[kFeedDescWords];
#pragma unroll
                for (uint32_t x = 0; x < kFeedDescWords / 2; ++x) {
                    w[2 * x] = __shfl_sync(kFull, lo, took * (kFeedDescWords / 2) + x);
                    w[2 * x + 1] = __shfl_sync(kFull, hi, took * (kFeedDescWords / 2) + x);
                }
                if (w[5] & kDescSplit) {
                    // plan(i)/B(i) refill m'_{i+1}'s slot, last handed out as m'_{i+1-R}: its
                    // consumer (another stream) must have released it
                    const uint64_t need = w[4] + 2 >= R ? w[4] + 2 - R : 0;
                    if (released < need && consumed < need) {
                        blocked = true;
                        break;
                    }
                } else if (w[4] > released) {
                    released = w[4];
                }
                admitted = w[4] + static_cast<uint32_t>(w[5]);  // i_begin + count
                if (lane == 0) {
                    uint64_t* dd = reinterpret_cast<uint64_t*>(rp.feed + ((j + took) % kFeedRing));
#pragma unroll
                    for (uint32_t x = 0; x < kFeedDescWords; ++x)
                        dd[x] = w[x];
                    if (rp.timings)
                        for (uint64_t x = w[4]; x < admitted && x < w[4] + kTimingRing; ++x)
                            tstamp(rp, x, 0);
                    run_mark(rp, w[4], 13);
                }
            }
            if (took > 0) {
                if (lane == 0) {
                    st_release_gpu(&rp.ctl->admitted, admitted);
                }
                j += took;
                idle_t0 = 0;
                spin = 0;
                continue;
            }
            if (blocked) {  // posted work is waiting for its consumer: not idle
                idle_t0 = 0;
                __nanosleep(128);
                continue;
            }
        }
        uint32_t act = 0;  // 0: keep polling, 1: failed, 2: leave
        if (lane == 0) {
            if (run_failed(rp)) {
                act = 1;
            } else if (ld_acquire_gpu(&rp.ctl->ready) < admitted) {  // work in flight: not idle
                idle_t0 = 0;
            } else {
                const uint64_t now = globaltimer();
                if (idle_t0 == 0)
                    idle_t0 = now;
                if (rp.tool_mode) {  // every post launches its own instance: nothing to hand over
                    act = 2;
                } else if (*rp.quiesce != 0 || now - idle_t0 >= rp.idle_ns) {
                    // Leave. Announce it in host memory first, then look for a post already on
                    // its way (the host raises host_posted before it enqueues the descriptor's
                    // memory operations, then reads `exiting`): of the two, at least one sees
                    // the other, so either this instance stays or the host launches the next
                    // one behind it.
                    *rp.exiting = (rp.gen << 32) | (j + 1);
                    asm volatile("fence.sc.sys;" ::: "memory");
                    if (*rp.host_posted > j) {
                        *rp.exiting = 0;  // stay (a relaunch the host may already have queued finds no work)
                        idle_t0 = 0;
                    } else {
                        act = 2;
                    }
                }
            }
        }
        act = __shfl_sync(kFull, act, 0);
        if (act == 1) {
            failed = true;
            break;
        }
        if (act == 2)
            break;
        __nanosleep(spin < 512 ? 64 : 512);
    }
    if (lane == 0) {
        if (!failed) {
            rp.ctl->next_step[(rp.gen + 1) & 1] = admitted;
            rp.ctl->next_desc[(rp.gen + 1) & 1] = j;
        }
        st_release_gpu(&rp.ctl->stop_at, ((rp.gen & 0xffffffu) << 40) | admitted);
    }
}

// CTA 0 warp 5: ready(i) — m'_i complete — in order, for the consumers' stream waits.
__device__ void run_ready(const RunParams& rp, uint64_t i0, uint64_t j0) {
    // m'_i = m_i ++ reps(i-1) is complete once A(i) (its batch rows and labels, every CTA),
    // B(i-1) (the reps this rank owns; plan(i-1) wrote their labels and |reps(i-1)|) and every
    // peer's B(i-1) (the reps it owns) are. The caller's m_i is free once sel(i) has read its
    // labels and B(i) no longer reads it: for early-ready steps B(i) sources the winners from
    // m'_i, so B(i) may still run; otherwise ready(i) also waits for B(i).
    const StepParams& b = rp.base;
    const bool multi = (b.mode & kModePeers) && b.N > 1;
    const RegionHeader* hdr = reinterpret_cast<const RegionHeader*>(b.region[b.me]);
    const uint32_t* repcnt = reinterpret_cast<const uint32_t*>(b.region[b.me] + b.off_counts) + b.aug_ring;
    uint32_t* aug_count = reinterpret_cast<uint32_t*>(b.region[b.me] + b.off_counts);
    uint64_t adm = 0;
    SeenFlag ad{&rp.ctl->a_done, 0}, bd{&rp.ctl->b_done, 0}, sd{&rp.ctl->sel_done, 0};
    uint64_t peers_seen = 0;
    FeedCursor c;
    cursor_init(c, i0, j0);
    uint64_t i = i0;
#pragma unroll 1
    for (;; ++i) {
        if (!wait_admit(rp, adm, i))
            break;
        cursor_seek(c, rp, i);
        // early-ready steps: A(i), the previous round and sel(i); otherwise B(i), which implies
        // them (every CTA's arrival for B(i) waited for its A(i); B(i) followed sel(i))
        bool ok = c.early ? wait_seen(ad, i + 1, rp) && wait_seen(bd, i, rp) && wait_seen(sd, i + 1, rp)
                          : wait_seen(bd, i + 1, rp);
        if (ok && multi && i > 0)
            ok = wait_peers(hdr->pushdone, b.N, b.me, i, rp, peers_seen, false);
        if (!ok) {  // the engine failed: every admitted m' not yet ready reports it
            if (b.mailbox) {
                volatile uint32_t* mb = b.mailbox;
                const uint32_t err = *reinterpret_cast<volatile const uint32_t*>(&rp.ctl->error);
                for (uint64_t x = i; x < adm && x < i + b.aug_ring; ++x)
                    mb[mb_err(ring_slot(x, b.aug_ring), b.aug_ring)] = err ? err : DRB_ERR_INTERNAL;
            }
            break;
        }
        const uint32_t slot = ring_slot(i, b.aug_ring);
        const uint32_t cnt = c.n + (i > 0 ? __ldcg(repcnt + slot) : 0u);  // n + |reps(i-1)|
        aug_count[slot] = cnt;
        if (b.mailbox) {
            volatile uint32_t* mb = b.mailbox;
            mb[mb_count(slot)] = cnt;
            mb[mb_err(slot, b.aug_ring)] = 0;
        }
        st_release_sys(&rp.ctl->ready, i + 1);
        *rp.ready_host = i + 1;  // (after the system-scope release: the host sees m'_i complete)
        run_mark(rp, i, 14);
        if (i + 1 == c.ib + c.cnt) {  // a descriptor's last step: once its B is done too, no role
                                      // reads the descriptor again and the host may reuse its slot
            if (!wait_seen(bd, i + 1, rp))
                break;
            st_release_gpu(&rp.ctl->desc_done, c.j + 1);
            *rp.desc_done_host = c.j + 1;
        }
    }
    if (run_failed(rp)) {  // release every stream (and host) still waiting for an m' of this engine
        if (b.mailbox)
            *reinterpret_cast<volatile unsigned long long*>(b.mailbox + kMbFailedAt) = i;
        __threadfence_system();
        st_release_sys(&rp.ctl->ready, kReadyFailed);
        *rp.ready_host = kReadyFailed;
    }
}

// CTA 0: the sel chain. Warp 0 runs sel(i), warp 2 draws round i+1's selection ahead,
// warp 3 fetches the labels of m_{i+1}; warp 1 publishes sel_done and keeps b_done /
// plan_done fresh in shared memory; warps 4 and 5 are the feeder and the ready publisher.
__device__ void run_sel_role(const RunParams& rp, uint32_t* sm, StepParams& sp, uint32_t* flag, uint64_t i0,
                             uint64_t j0) {
    const uint32_t tid = threadIdx.x, warp = tid >> 5;
    if (warp == 4 && rp.feeder_cta == 0) {
        run_feeder(rp, i0, j0);  // (the whole warp)
        return;
    }
    if (warp == 5 && rp.feeder_cta == 0) {
        if ((tid & 31) == 0)
            run_ready(rp, i0, j0);
        return;
    }
    if (tid >= kSelThreads)
        return;
    const StepParams& b = rp.base;
    const uint32_t N = b.N, me = b.me;
    const bool multi = (b.mode & kModePeers) && N > 1;
    const uint32_t lag = aug_lag(b.aug_ring);
    SelView v = sel_view(sm, b);
    uint32_t* lab2 = sm + sel_smem(b.K, b.nmax).words;  // second label buffer (prefetch)
    uint32_t* labs[2] = {v.lab, lab2};
    volatile unsigned long long* seen =  // [0] b_done, [1] plan_done as last loaded; [2] ready
        reinterpret_cast<volatile unsigned long long*>(sm + ((sel_smem(b.K, b.nmax).words + b.nmax + 1) & ~1u));
    // Speculative S1 (warp 2 draws round k+1's selection during round k; it depends only on
    // the candidate counter, which round k advances by min(c, n_k) unless a draw is rejected
    // or the round inserts nothing): sx[0..1] the counter each parity's selection was drawn
    // for (~0: none), sx[2] the counter at the start of the current round; spec_sel[2][32].
    unsigned long long* sx = const_cast<unsigned long long*>(seen) + 4;
    uint32_t* spec_sel = reinterpret_cast<uint32_t*>(sx + 4);
    uint32_t* spec_tmp = spec_sel + 64;
    // step hand-over between tid 0 and the other warps: [0] current n, [1] next n (or ~0:
    // step k+1 not admitted yet), [2..3] next labels pointer, [4] stop, [5] bad of m_k,
    // [6] bad of the prefetched m_{k+1}, [7] labels of step k already in labs[k & 1]
    volatile uint32_t* hx = reinterpret_cast<volatile uint32_t*>(spec_tmp + 32);
    FeedCursor cur, nxt;  // tid 0's
    uint64_t adm_seen = 0, peers_seen = 0;
    if (tid == 0) {
        sp = b;
        run_patch(sp, rp, i0);
        seen[0] = 0;
        seen[1] = 0;
        seen[2] = 0;
        sx[0] = ~0ull;
        sx[1] = ~0ull;
        for (int x = 0; x < 8; ++x)
            hx[x] = 0;
        cursor_init(cur, i0, j0);
        cursor_init(nxt, i0, j0);
    }
    named_bar(1, kSelThreads);
    {  // state and the own occupancy row at the start of the instance
        const uint64_t* tin = reinterpret_cast<const uint64_t*>(sp.region[me] + sp.off_table) +
                              uint64_t(sp.tslot_in) * N * sp.K + uint64_t(me) * sp.K;
        if (tid < sizeof(SelState) / 8)
            reinterpret_cast<uint64_t*>(v.st)[tid] = __ldcg(reinterpret_cast<const uint64_t*>(sp.sel_in) + tid);
        for (uint32_t x = tid; x < sp.K; x += kSelThreads)
            v.occ[x] = occ_of(__ldcg(tin + x));
        named_bar(1, kSelThreads);
    }
    if (warp == 1) {
        if (tid == 32)
            run_publisher(rp, i0, seen + 2, &rp.ctl->sel_done, seen, &rp.ctl->b_done, &rp.ctl->plan_done, hx + 4);
        return;
    }
    const RegionHeader* hdr = reinterpret_cast<const RegionHeader*>(b.region[me]);
#pragma unroll 1
    for (uint64_t k = 0;; ++k) {  // warps 0, 2, 3 (barrier 1, 96 threads)
        const uint64_t i = i0 + k;
        if (tid == 0) {
            trace_at(sp, 12);
            run_mark(rp, i, 0);
            uint64_t as = adm_seen;
            bool ok = wait_admit(rp, as, i);
            if (ok && v.st->error) {  // round i-1 failed (a label >= K): it was still delivered;
                                      // nothing after it runs (engine.cpp:67-68,74-80)
                run_fail(rp, v.st->error, (1u << 24) | uint32_t(i & 0xffffff));
                ok = false;
            }
            if (ok) {
                run_patch(sp, rp, i);
                if (nxt.cnt != 0 && i >= nxt.ib && i < nxt.ib + nxt.cnt)
                    cur = nxt;  // looked ahead in round i-1 (no second descriptor load)
                else
                    cursor_seek(cur, rp, i);
                feed_patch(sp, cur, i);
                hx[0] = sp.n;
                // W slot (i-8) / m' slot (multi, i-6) / table slot (plan(i-4)) free
                // W slot: B(i-32) complete (multi-rank: the m' / table lag); table slot: plan(i-15)
                const uint64_t wb = i0 + back(k, multi ? lag - 1 : kListRing - 1), wp = i0 + back(k, kTableRing - 2);
                if (seen[0] < wb)
                    ok = run_wait(&rp.ctl->b_done, wb, rp, false);
                if (ok && seen[1] < wp)
                    ok = run_wait(&rp.ctl->plan_done, wp, rp, false);
                run_mark(rp, i, 1);
                if (ok && multi && i >= lag)  // peers' B(i-lag) complete (m' slot)
                    ok = wait_peers(hdr->pushdone, N, me, i - lag + 1, rp, peers_seen, true);
                // step i+1 already posted: its batch size and labels for the look-ahead warps
                hx[1] = ~0u;
                if (ok && (as > i + 1 || ((as = ld_acquire_gpu(&rp.ctl->admitted)) > i + 1))) {
                    cursor_seek(nxt, rp, i + 1);
                    hx[1] = nxt.n;
                    const uint32_t* lp = cursor_labels(nxt, i + 1);
                    hx[2] = static_cast<uint32_t>(reinterpret_cast<uint64_t>(lp));
                    hx[3] = static_cast<uint32_t>(reinterpret_cast<uint64_t>(lp) >> 32);
                }
            }
            adm_seen = as;
            __threadfence_block();  // sel(k-1)'s hand-over is visible before the stop
            hx[4] = ok ? 0u : 1u;
            sx[2] = v.st->cand_ctr;  // written by this thread in sel_core(k-1)
        }
        named_bar(1, 96);
        if (hx[4])
            return;
        v.lab = labs[k & 1];
        if (!hx[7]) {  // labels of m_i were not prefetched: load them now (all three warps)
            const uint32_t n = hx[0];
            const uint32_t t = tid < 32 ? tid : tid - 32;  // warps 0, 2, 3 -> 0..95
            int bad = 0;
            for (uint32_t x = t; x < n; x += 96) {
                const uint32_t l = __ldg(sp.labels + x);
                v.lab[x] = l;
                bad |= l >= sp.K;
            }
            if (bad)
                atomicOr(const_cast<uint32_t*>(hx + 5), 1u);
            named_bar(1, 96);
        }
        const uint32_t nn = hx[1];
        if (warp == 0) {
            tl_mark(sp, 0, false);
            trace_at(sp, 0);
            if (tid == 0) {
                run_mark(rp, i, 2);
                tstamp(rp, i, 1);
            }
            // (the peers' pushdone for the table / m' slot was checked before the hand-over)
            sel_core(sp, v, hx[5] != 0, spec_sel + 32 * (k & 1), sx[k & 1], true);
            delay_exp(1);
            __syncwarp();
            unsigned long long pt = 0;
            prof_span(sp, 19, pt);
            if (tid == 0) {
                st_release_cta(seen + 2, k + 1);  // hand sel(k) to the publisher
                tstamp(rp, i, 2);
                run_mark(rp, i, 3);
                tl_mark(sp, 0, true);
            }
            prof_span(sp, 19, pt);
        } else if (warp == 2) {  // warp 2: S1 of round k+1, ahead
            uint64_t drawn = ~0ull;
            const uint32_t kk = min(sp.c, hx[0]);   // round k's draws (counter advance)
            if (nn != ~0u) {
                const uint32_t k1 = min(sp.c, nn);  // round k+1's draws
                if (kk > 0 && k1 > 0 && k1 <= 32 && nn < 65536u) {
                    const uint64_t c1 = sx[2] + kk;
                    if (warp_select_fast(sp.cand_key, c1, nn, k1, spec_sel + 32 * ((k + 1) & 1), spec_tmp))
                        drawn = c1;
                }
            }
            if (tid == 64)
                sx[(k + 1) & 1] = drawn;
        } else if (nn != ~0u) {  // warp 3: labels of m_{k+1}
            const uint32_t* lp =
                reinterpret_cast<const uint32_t*>(uint64_t(hx[2]) | (uint64_t(hx[3]) << 32));
            int bad = 0;
            for (uint32_t x = tid - 96; x < nn; x += 32) {
                const uint32_t l = __ldg(lp + x);
                labs[(k + 1) & 1][x] = l;
                bad |= l >= sp.K;
            }
            if (__any_sync(kFull, bad) && tid == 96)
                hx[6] = 1u;
        }
        unsigned long long pt2 = 0;
        if (warp == 0)
            prof_span(sp, 20, pt2);
        named_bar(1, 96);
        if (warp == 0)
            prof_span(sp, 20, pt2);
        if (tid == 0) {
            hx[7] = nn != ~0u ? 1u : 0u;  // step k+1's labels are in labs[(k+1) & 1]
            hx[5] = hx[6];
            hx[6] = 0;
            run_mark(rp, i, 4);
        }
    }
}

// CTA 1: the plan chain. plan_core runs on the first plan_threads(N) threads (named barrier
// 3); a helper warp publishes plan_done and keeps sel_done / b_done fresh.
__device__ void run_plan_role(const RunParams& rp, uint32_t* sm, StepParams& sp, uint32_t* flag, uint64_t i0) {
    const uint32_t tid = threadIdx.x, warp = tid >> 5;
    const PlanView v = plan_view(sm, rp.base);
    const uint32_t T = 32 * (rp.base.N + 1 < 3 ? 3 : rp.base.N + 1);  // plan_threads(N) <= kRunThreads - 32
    const uint32_t helper = kRunThreads / 32 - 1;
    volatile unsigned long long* seen = reinterpret_cast<volatile unsigned long long*>(flag + 2);  // [0] sel, [1] b, [2] ready
    volatile uint32_t* stop = flag;  // [0]
    if (tid == 0) {
        sp = rp.base;
        run_patch(sp, rp, i0);
        seen[0] = 0;
        seen[1] = 0;
        seen[2] = 0;
        flag[0] = 0;
    }
    __syncthreads();
    if (warp == helper) {
        if ((tid & 31) == 0)
            run_publisher(rp, i0, seen + 2, &rp.ctl->plan_done, seen, &rp.ctl->sel_done, &rp.ctl->b_done, stop);
        return;
    }
    if (tid >= T)
        return;
    if (tid < sizeof(PlanState) / 8)
        reinterpret_cast<uint64_t*>(v.st)[tid] = __ldcg(reinterpret_cast<const uint64_t*>(sp.plan_in) + tid);
    uint64_t adm = 0;
#pragma unroll 1
    for (uint64_t k = 0;; ++k) {
        const uint64_t i = i0 + k;
        if (tid == 0) {
            trace_at(sp, 13);
            run_mark(rp, i, 0);
            bool ok = wait_admit(rp, adm, i);
            if (ok) {
                run_patch(sp, rp, i);
                if (seen[0] < i + 1)  // sel(i)
                    ok = run_wait(&rp.ctl->sel_done, i + 1, rp, false);
                if (ok && seen[1] < i0 + back(k, kListRing - 1))  // X slot: B(i-32) complete
                    ok = run_wait(&rp.ctl->b_done, i0 + back(k, kListRing - 1), rp, false);
            }
            run_mark(rp, i, 1);
            flag[1] = ok ? 0u : 1u;
            v.misc[0] = 0;
        }
        cta_bar(3, T);
        if (flag[1]) {
            if (tid == 0) {
                __threadfence_block();
                flag[0] = 1;  // the publisher leaves too
            }
            return;
        }
        tl_mark(sp, 1, false);
        trace_at(sp, 5);
        if (tid == 0)
            tstamp(rp, i, 3);
        plan_core(sp, v, T, 3);
        delay_exp(2);
        cta_bar(3, T);
        if (tid == 0) {
            st_release_cta(seen + 2, k + 1);  // hand plan(k) to the publisher
            tl_mark(sp, 1, true);
            run_mark(rp, i, 3);
        }
    }
}

// B(k) of a copy CTA is complete: fence, arrive. Copy CTAs are not in lockstep, so arrivals
// are counted per iteration (slot k % 8); the last arrival of iteration i releases b_done =
// i+1 once b_done = i (in order) and, multi-rank, pushdone = i+1 at every peer.
// a_done = max(a_done, v) with release semantics: A(i) of every CTA is complete. Two chains
// raise it — the A ticket of early-ready steps, the B arrivals of the others (whose CTA
// arrivals wait for their own A(i)) — and A is in order per CTA, so the maximum is exact.
__device__ __forceinline__ void raise_a_done(const RunParams& rp, uint64_t v) {
    asm volatile("red.release.gpu.global.max.u64 [%0], %1;" ::"l"(&rp.ctl->a_done), "l"(v) : "memory");
}
// Returns true for the last arrival (b_done = i+1 published). a_too: every arrival of this
// iteration also waited for its CTA's A(i), so the last one raises a_done too.
__device__ bool run_b_arrive(const RunParams& rp, const StepParams& p, uint64_t k, uint64_t i, bool multi,
                             bool a_too) {
    asm volatile("fence.proxy.async.global;" ::: "memory");  // the bulk stores, for generic-proxy readers
    uint32_t* t = &rp.ctl->ticket[k % kTicketRing];
    uint32_t old;
    // acq_rel at GPU scope: the last arrival observes every arrival's (completed) stores, local
    // and remote; its one system-scope fence below makes them all visible to the peers before
    // the pushdone words (cumulativity), so no arrival pays a system-scope atomic
    asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(old) : "l"(t) : "memory");
    if (old + 1 == rp.copy_ctas) {
        *reinterpret_cast<volatile uint32_t*>(t) = 0;  // slot reused by iteration k+32
        if (!run_wait(&rp.ctl->b_done, i, rp, false))
            return false;
        (void)multi;  // pushdone at the peers: run_peer_publisher, off this chain
        if (a_too)
            raise_a_done(rp, i + 1);
        st_release_gpu(&rp.ctl->b_done, i + 1);
        tstamp(rp, i, 4);
        run_mark(rp, i, 9);
        return true;
    }
    return false;
}

// Cross-warp progress of a copy CTA's engines (shared memory, per iteration parity).
struct BFlags {
    unsigned long long landed[2];    // k+1: B(k)'s loads landed (its reads are done)
    unsigned long long complete[2];  // k+1: B(k)'s stores complete
    unsigned long long parsed[4];    // k+1 in slot k % 4: W_k's slab rows published in wrows[k % 4]
    unsigned long long a_local;      // k+1: this CTA's A(k) complete (m_i's slice and labels in m'_i)
};
// Bounded like every other wait: gives up once the run failed or after timeout_ns (then
// fails the run, recording `site` and the iteration), so no role can spin forever.
__device__ bool smem_wait_ge(const volatile unsigned long long* f, uint64_t want, const RunParams& rp,
                             uint32_t site, uint64_t k) {
    uint64_t t0 = 0;
    for (uint32_t spin = 0; *f < want; ++spin) {
        if ((spin & 255) == 255) {
            if (run_failed(rp))
                return false;
            const uint64_t now = globaltimer();
            if (t0 == 0)
                t0 = now;
            else if (now - t0 > rp.base.timeout_ns) {
                run_fail(rp, DRB_ERR_INTERNAL, (site << 24) | uint32_t(k & 0xffffff));
                return false;
            }
        }
        __nanosleep(20);
    }
    return true;
}

// B(k)'s stores are complete (after bulk_wait_all): hand them to the CTA's arrival warp. The
// proxy fence orders the async-proxy stores before the CTA-scope release; the arrival warp's
// acquire and its GPU-scope acq_rel ticket atomic carry them on (cumulativity).
__device__ __forceinline__ void b_complete(volatile BFlags* fl, uint64_t k) {
    asm volatile("fence.proxy.async.global;" ::: "memory");
    st_release_cta(&fl->complete[k & 1], k + 1);
}

// One B engine (a warp) of a copy CTA, for the instance's iterations k = wsel, wsel+2, ...:
// the W_i writes and X_i pushes on this CTA's byte column [c0, c1). The two B warps
// alternate, so B(k+1) issues its loads while B(k) drains; what must stay ordered between
// consecutive iterations on the same slab bytes is ordered through BFlags:
//   a slot pushed in k that W_{k-1} wrote        -> B(k-1)'s stores complete first
//   a W_k row that X_{k-1} read                  -> B(k-1)'s loads landed before k's stores
//   a W_k row that W_{k-1} also wrote            -> B(k-1)'s stores complete first
__device__ void run_b_warp(const RunParams& rp, uint32_t* sm, const RunSmem& R, StepParams& sp, uint32_t wsel,
                           uint64_t i0, uint64_t j0) {
    const uint32_t lane = threadIdx.x & 31;
    const StepParams& b = rp.base;
    uint8_t* base8 = reinterpret_cast<uint8_t*>(sm);
    uint32_t* xraw = reinterpret_cast<uint32_t*>(base8 + R.xraw[wsel]);
    uint32_t* wraw = reinterpret_cast<uint32_t*>(base8 + R.wraw[wsel]);
    uint32_t* jsrc = reinterpret_cast<uint32_t*>(base8 + R.jsrc[wsel]);
    uint32_t* misc = reinterpret_cast<uint32_t*>(base8 + R.misc[wsel]);
    uint64_t* paddr = reinterpret_cast<uint64_t*>(base8 + R.paddr[wsel]);
    uint8_t* arena = base8 + R.arena[wsel];
    uint32_t* wrows = reinterpret_cast<uint32_t*>(base8 + R.wrows);
    volatile BFlags* fl = reinterpret_cast<volatile BFlags*>(base8 + R.flags);
    uint64_t* barB = reinterpret_cast<uint64_t*>(base8 + R.bars) + kTmaStagesA + wsel;
    volatile uint32_t* ready = misc + 6;
    const uint32_t part = blockIdx.x - 2, parts = rp.copy_ctas;
    const uint64_t S = b.S;
    const uint64_t c16 = S >> 4;
    const uint64_t c0 = (c16 * part / parts) << 4, c1 = (c16 * (part + 1) / parts) << 4;
    const uint32_t clen = static_cast<uint32_t>(c1 - c0);
    const uint32_t per_win = clen ? R.arena_bytes / clen : 0;
    const uint32_t pw = plist_words(b.N, b.r), ww = wlist_words(b.nmax), nslot = b.nmax + 1;
    SeenFlag pdone{&rp.ctl->plan_done, 0}, adone{&rp.ctl->a_done, 0};  // (plan_done > i implies sel_done > i)
    uint64_t adm = 0;
    FeedCursor cur;
    cursor_init(cur, i0, j0);
    uint32_t phB = 0;
    int64_t prev_k = -1;  // this warp's previous iteration (stores not yet drained)
    bool fetched = false;  // this iteration's lists already in flight (prefetched by the previous one)
    if (lane == 0)
        sp = b;
    auto fetch_lists = [&](uint64_t i) {  // W_i and X_i -> wraw / xraw (cp.async, one group)
        const uint32_t* xs = rp.plist_base + (i % kListRing) * rp.pw;
        const uint32_t* ws = rp.wlist_base + (i % kListRing) * rp.ww;
        for (uint32_t x = lane; x < pw; x += 32)
            asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(xraw + x)), "l"(xs + x) : "memory");
        for (uint32_t x = lane; x < ww; x += 32)
            asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(wraw + x)), "l"(ws + x) : "memory");
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
#pragma unroll 1
    for (uint64_t k = wsel;; k += 2) {
        const uint64_t i = i0 + k;
        bool ok = true;
        // Before waiting for a step that is not posted yet, complete the previous one: its
        // stores would otherwise stay in flight (and b_done, ready behind them) until the
        // next post arrives.
        if (prev_k >= 0) {
            bool posted = false;
            if (lane == 0)
                posted = adm > i || (adm = ld_acquire_gpu(&rp.ctl->admitted)) > i;
            if (!__shfl_sync(kFull, posted ? 1 : 0, 0)) {
                bulk_wait_all();
                __syncwarp();
                if (lane == 0)
                    b_complete(fl, uint64_t(prev_k));
                prev_k = -1;
            }
        }
        if (lane == 0) {
            ok = wait_admit(rp, adm, i);
            if (ok) {
                run_patch(sp, rp, i);
                cursor_seek(cur, rp, i);
                feed_patch(sp, cur, i);
                if (!fetched)
                    ok = wait_seen(pdone, i + 1, rp);  // plan(i) followed sel(i): implies sel_done > i
            }
        }
        if (!__shfl_sync(kFull, ok ? 1 : 0, 0))
            break;
        delay_exp(3);
        __syncwarp();
        tl_mark(sp, 2, false);
        if (lane == 0)
            cta_mark(sp, 0);
        if (!fetched)
            fetch_lists(i);
        fetched = false;
        copy_parse(sp, xraw, wraw, jsrc, nullptr, misc, ready, true, true, false);
        const uint32_t nj = misc[0], nw = misc[1];
        uint32_t* wk = wrows + (k & 3) * nslot;  // publish W_k's rows for B(k+1)
        for (uint32_t t = lane; t < nw; t += 32)
            wk[1 + t] = wraw[3 + 2 * t];
        if (lane == 0)
            wk[0] = nw;
        __syncwarp();
        __threadfence_block();
        if (lane == 0)
            fl->parsed[k & 3] = k + 1;
        if (lane == 0)
            cta_mark(sp, 10);
        // W_{k-1} (the other warp's) for the hazard checks
        bool push_hz = false, w_hz = false, own_hz = false;
        // slot-set intersections: with <= 32 slots on one side, lane t holds slot t and every
        // probe is one vote (no per-lane scan of the other list)
        auto hits_any = [&](const uint32_t* list, uint32_t nl, const uint32_t* probe, uint32_t np_, bool skip_batch) {
            bool hz = false;
            if (nl <= 32) {
                const uint32_t mine = lane < nl ? list[1 + lane] : ~0u;
#pragma unroll 1
                for (uint32_t x = 0; x < np_ && !hz; ++x) {
                    const uint32_t s_ = probe[x];
                    if (!(skip_batch && (s_ >> 31)))
                        hz = __any_sync(kFull, mine == s_);
                }
            } else {
                for (uint32_t x = lane; x < np_; x += 32) {
                    const uint32_t s_ = probe[x];
                    if (!(skip_batch && (s_ >> 31)))
                        for (uint32_t t = 0; t < nl; ++t)
                            hz |= list[1 + t] == s_;
                }
                hz = __any_sync(kFull, hz);
            }
            return hz;
        };
        if (k > 1) {  // a slot pushed now that this warp's B(k-2) wrote: its stores land first
            const uint32_t* wq = wrows + ((k - 2) & 3) * nslot;
            own_hz = hits_any(wq, wq[0], jsrc, nj, true);
        }
        if (k > 0) {
            if (lane == 0)
                smem_wait_ge(&fl->parsed[(k - 1) & 3], k, rp, 2, k);
            __syncwarp();
            if (lane == 0)
                cta_mark(sp, 11);
            const uint32_t* wp = wrows + ((k - 1) & 3) * nslot;
            const uint32_t np = wp[0];
            push_hz = hits_any(wp, np, jsrc, nj, true);
            w_hz = hits_any(wp, np, wk + 1, nw, false);
        }
        const uint32_t pieces = clen ? nj + nw : 0;
        // early-ready steps: the winning batch rows come from m'_i (the A engines copied m_i
        // there): wait for every CTA's A(i), then order its stores before these TMA loads
        const bool early = __shfl_sync(kFull, cur.early ? 1 : 0, 0) != 0;
        bool from_batch = early && nw > 0;
        for (uint32_t x = lane; early && x < nj && !from_batch; x += 32)
            from_batch = (jsrc[x] >> 31) != 0;
        if (__any_sync(kFull, from_batch) && pieces) {  // every CTA's A(i) (a flat slice each)
            bool ok_a = true;
            if (lane == 0)
                ok_a = wait_seen(adone, i + 1, rp);
            if (!__shfl_sync(kFull, ok_a ? 1 : 0, 0))
                break;
            asm volatile("fence.proxy.async.global;" ::: "memory");
        }
        {
            const uint8_t* batch = early ? b.region[b.me] + b.off_aug + uint64_t(sp.aslot) * b.aug_slot_bytes +
                                               uint64_t(b.nmax - sp.n) * S  // m_i's rows inside m'_i
                                         : sp.batch;
            uint8_t* slab = reinterpret_cast<uint8_t*>(sp.slab);
            const uint32_t next_slot = (sp.aslot + 1) % b.aug_ring;
            for (uint32_t x = lane; x < pieces; x += 32) {
                const uint8_t* src;
                uint8_t* dst;
                if (x < nj) {
                    const uint32_t s_ = jsrc[x];
                    src = ((s_ >> 31) ? batch + uint64_t(s_ & 0x7fffffffu) * S : slab + uint64_t(s_) * S) + c0;
                    dst = push_dst(sp, xraw[4 + x], next_slot) + c0;
                } else {
                    src = batch + uint64_t(wraw[2 + 2 * (x - nj)]) * S + c0;
                    dst = slab + uint64_t(wraw[3 + 2 * (x - nj)]) * S + c0;
                }
                paddr[2 * x] = reinterpret_cast<uint64_t>(src);
                paddr[2 * x + 1] = reinterpret_cast<uint64_t>(dst);
            }
        }
        __syncwarp();

        if (lane == 0)
            cta_mark(sp, 12);
        bool drained = false;
        auto drain = [&]() {  // this warp's previous iteration (k-2): stores complete, arrive
            bulk_wait_all();
            __syncwarp();
            if (lane == 0 && prev_k >= 0)
                b_complete(fl, uint64_t(prev_k));
            prev_k = -1;
            drained = true;
        };
        if (k > 2) {  // the other warp's B(k-3) complete (its drain precedes every wait of B(k-1))
            if (lane == 0)
                smem_wait_ge(&fl->complete[(k - 3) & 1], k - 2, rp, 7, k);
            __syncwarp();
        }
        if (own_hz && !push_hz) {
            drain();
            asm volatile("fence.proxy.async.global;" ::: "memory");
        }
        if (push_hz) {  // B(k-1)'s W stores land before these loads read the rows. Drain own
                        // k-2 first: the other warp may be waiting for it (no wait cycle).
            drain();
            if (lane == 0)
                smem_wait_ge(&fl->complete[(k - 1) & 1], k, rp, 3, k);
            __syncwarp();
            asm volatile("fence.proxy.async.global;" ::: "memory");
        }
        for (uint32_t p0 = 0; p0 < pieces; p0 += per_win) {
            const uint32_t p1 = min(pieces, p0 + per_win);
            bulk_wait_read_all();  // arena reuse (p0 = 0: this warp's previous iteration's stores)
            __syncwarp();
            if (lane == 0)
                mbar_expect_tx(barB, (p1 - p0) * clen);
            for (uint32_t x = p0 + lane; x < p1; x += 32)
                bulk_load(arena + (x - p0) * clen, reinterpret_cast<const void*>(paddr[2 * x]), clen, barB);
            if (lane == 0)
                cta_mark(sp, 3);
            if (!drained)
                drain();
            if (!mbar_wait(barB, take_phase(phB, 0), rp.base.timeout_ns) && lane == 0)
                run_fail(rp, DRB_ERR_INTERNAL, (10u << 24) | uint32_t(k & 0xffffff));
            if (p1 == pieces && lane == 0)
                fl->landed[k & 1] = k + 1;
            if (lane == 0) {
                cta_mark(sp, 6);
                if (k > 0)  // B(k-1) finished reading the rows W_k overwrites
                    smem_wait_ge(&fl->landed[(k - 1) & 1], k, rp, 4, k);
                if (k > 0 && w_hz)  // and its own writes to them land first
                    smem_wait_ge(&fl->complete[(k - 1) & 1], k, rp, 5, k);
            }
            __syncwarp();
            for (uint32_t x = p0 + lane; x < p1; x += 32)
                bulk_store(reinterpret_cast<void*>(paddr[2 * x + 1]), arena + (x - p0) * clen, clen);
            bulk_commit();
        }
        if (!drained)
            drain();
        if (pieces == 0 && lane == 0)
            fl->landed[k & 1] = k + 1;
        // xraw / wraw are free (paddr holds this iteration's addresses): fetch this warp's next
        // lists now if sel / plan already published them, so the L2 round trip overlaps the
        // stores in flight instead of starting the next iteration
        {
            bool pre = false;
            if (lane == 0)
                pre = poll_seen(pdone, i + 3);  // (implies sel(i+2))
            if (__shfl_sync(kFull, pre ? 1 : 0, 0)) {
                fetch_lists(i + 2);
                fetched = true;
            }
        }
        prev_k = int64_t(k);
        if (lane == 0)
            cta_mark(sp, 4);
    }
    if (prev_k >= 0 && !run_failed(rp)) {
        bulk_wait_all();
        __syncwarp();
        if (lane == 0)
            b_complete(fl, uint64_t(prev_k));
    }
    asm volatile("cp.async.wait_all;" ::: "memory");  // a prefetch issued for an iteration never run
}

// CTAs 2..: copies. Warp 1 lane 0 streams m_i -> m'_i (flat slice of the batch bytes), at
// most two iterations ahead of the completed B. Warps 0 and 2 do B (even / odd iterations)
// on a fixed COLUMN of every row — bytes [c0, c1) of each slab row written (W_i) and each
// slot pushed (X_i) — so every access to a given slab byte is in this one CTA: there is no
// grid-wide hand-off between iterations. Warp 3 arrives for the CTA once A(k) and B(k) are
// complete.
// A(k) of a copy CTA is complete (its m'_i rows stored, and for CTA part 0 m_i's labels), for
// an early-ready step: arrive on the A ticket; the last arrival raises a_done to i+1.
__device__ void run_a_arrive(const RunParams& rp, uint64_t k, uint64_t i) {
    uint32_t* t = &rp.ctl->aticket[k % kTicketRing];
    uint32_t old;
    asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(old) : "l"(t) : "memory");
    if (old + 1 == rp.copy_ctas) {
        *reinterpret_cast<volatile uint32_t*>(t) = 0;  // slot reused by iteration k+32
        raise_a_done(rp, i + 1);
    }
}

// Multi-rank: pushdone[me] = b_done at every peer, one thread, in order. The system-scope fence
// that makes this rank's pushes visible to the peers before the word costs microseconds; here it
// is off the arrivals' b_done chain (the last arrival's GPU-scope release of b_done covers every
// CTA's completed B stores; this thread acquires it, fences at system scope, then stores). It
// leaves once everything this instance admitted is B-complete and announced.
__device__ void run_peer_publisher(const RunParams& rp, uint64_t i0) {
    const StepParams& b = rp.base;
    uint64_t pub = i0;
#pragma unroll 1
    for (uint32_t spin = 0;; ++spin) {
        const uint64_t bd = ld_acquire_gpu(&rp.ctl->b_done);
        if (bd > pub) {
            asm volatile("fence.acq_rel.sys;" ::: "memory");
            for (uint32_t w = 0; w < b.N; ++w)
                if (w != b.me)
                    asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(
                                     &reinterpret_cast<RegionHeader*>(b.region[w])->pushdone[b.me]),
                                 "l"(bd)
                                 : "memory");
            pub = bd;
            spin = 0;
            continue;
        }
        if (run_failed(rp))
            return;
        const uint64_t st = *reinterpret_cast<volatile const uint64_t*>(&rp.ctl->stop_at);
        if ((st >> 40) == (rp.gen & 0xffffffu) && bd >= (st & kStopMask))
            return;
        if (spin > 64)
            __nanosleep(spin < 4096 ? 32 : 256);
    }
}

// CTAs 2..: copies. The B engines work on a fixed byte COLUMN [c0, c1) of every row — so every
// slab access to a given byte happens in this one CTA, in program order, and there is no
// grid-wide hand-off between their iterations:
//   warp 1   A(k): a flat slice of m_i's bytes -> m'_i (TMA through the A ring); CTA part 0
//            also copies m_i's labels. m_i is not read after A(i): m'_i is ready without B(i).
//   warps 0, 2   B (even / odd iterations): W_i writes and X_i pushes, sourced from the slab
//            or, for winning batch rows, from m'_i's rows (after every CTA's A(i): a_done)
//   warp 3   arrival: B(k) complete -> ticket / b_done / pushdone (and descriptor retirement)
__device__ void run_copy_role(const RunParams& rp, uint32_t* sm, StepParams* sp2, uint64_t i0, uint64_t j0) {
    const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (warp >= 4) {  // the feeder and the ready publisher, when they live on this copy CTA
        if (blockIdx.x == rp.feeder_cta) {
            if (warp == 4)
                run_feeder(rp, i0, j0);  // (the whole warp)
            else if (warp == 5 && lane == 0)
                run_ready(rp, i0, j0);
        }
        if (blockIdx.x == gridDim.x - 1 && warp == 6 && lane == 0 && (rp.base.mode & kModePeers) && rp.base.N > 1)
            run_peer_publisher(rp, i0);
        return;
    }
    const StepParams& b = rp.base;
    const RunSmem R = run_smem(b.N, b.K, b.r, b.nmax);
    uint8_t* base8 = reinterpret_cast<uint8_t*>(sm);
    uint64_t* bars = reinterpret_cast<uint64_t*>(base8 + R.bars);
    uint8_t* ringA = base8 + R.ring_a;
    const uint32_t part = blockIdx.x - 2, parts = rp.copy_ctas;
    const uint64_t S = b.S;
    if (tid < sizeof(BFlags) / 8)
        reinterpret_cast<unsigned long long*>(base8 + R.flags)[tid] = 0;
    if (tid == 32) {
        for (uint32_t x = 0; x < kTmaStagesA + 2; ++x)
            mbar_init(bars + x, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    named_bar(2, 128);
    volatile BFlags* fl = reinterpret_cast<volatile BFlags*>(base8 + R.flags);
    if (warp == 0 || warp == 2) {
        run_b_warp(rp, sm, R, sp2[warp >> 1], warp >> 1, i0, j0);
        return;
    }
    if (warp == 3) {  // arrival warp (lane 0): B(k) complete -> ticket / b_done / pushdone, in
                      // order, off the B engines' own chains (the GPU-scope atomic waits on the
                      // memory system)
        if (lane != 0)
            return;
        const bool multi = (b.mode & kModePeers) && b.N > 1;
        uint64_t adm = 0;
        FeedCursor cur;
        cursor_init(cur, i0, j0);
#pragma unroll 1
        for (uint64_t k = 0;; ++k) {
            const uint64_t i = i0 + k;
            if (!wait_admit(rp, adm, i))
                return;
            cursor_seek(cur, rp, i);
            const bool a_too = !cur.early;  // this arrival also stands for the CTA's A(i)
            uint64_t t0 = 0;
            for (uint32_t spin = 0; ld_acquire_cta(&fl->complete[k & 1]) < k + 1 ||
                                    (a_too && ld_acquire_cta(&fl->a_local) < k + 1);
                 ++spin) {
                if ((spin & 63) == 63) {
                    if (run_failed(rp))
                        return;
                    const uint64_t now = globaltimer();
                    if (t0 == 0)
                        t0 = now;
                    else if (now - t0 > b.timeout_ns) {
                        run_fail(rp, DRB_ERR_INTERNAL, (8u << 24) | uint32_t(k & 0xffffff));
                        return;
                    }
                }
            }
            delay_exp(4);
            run_mark(rp, i, 8);
            run_b_arrive(rp, b, k, i, multi, a_too);
        }
    }
    // ---- A engine (warp 1): m_i -> m'_i rows (a flat slice of the batch bytes per CTA, 8 KB
    // TMA chunks), iteration after iteration ---------------------------------------------
    const uint32_t CH = kTmaChunk;
    uint32_t ph_bits = 0;  // phase of each A barrier (lane 0)
    SeenFlag bdone{&rp.ctl->b_done, 0}, adone{&rp.ctl->a_done, 0};
    uint64_t adm = 0;
    FeedCursor cur;
    cursor_init(cur, i0, j0);
    // A(i) writes m'_i's batch rows into the ring slot m'_{i-R} held: that m' was complete (its
    // pushes, B(i-R-1), done), read by B(i-R) (sourcing winners) and released (admission), so A
    // could run R-2 iterations ahead of B; DRB_A_AHEAD (default 8) bounds it: A's streaming
    // traffic far ahead delays B's loads
    const uint32_t ahead = min(b.aug_ring - 2, rp.a_ahead);
    // A(k)'s stores complete while A(k+1)'s loads are in flight: its completion (a_local, and the
    // A ticket of an early step) is signalled from the next iteration, or at once when no next
    // step is posted (lane 0's state)
    int64_t pend_k = -1;
    uint64_t pend_i = 0;
    bool pend_early = false;
    auto flush = [&]() {
        bulk_wait_all();  // A(pend)'s m'_i rows are written
        asm volatile("fence.proxy.async.global;" ::: "memory");
        st_release_cta(&fl->a_local, uint64_t(pend_k) + 1);  // for this CTA's arrival (the B ticket)
        if (pend_early)
            run_a_arrive(rp, uint64_t(pend_k), pend_i);  // m'_i's batch part is complete
        run_mark(rp, pend_i, 5);
        pend_k = -1;
    };
#pragma unroll 1
    for (uint64_t k = 0;; ++k) {
        const uint64_t i = i0 + k;
        bool ok = true;
        uint32_t n = 0;
        uint64_t bp = 0, lp = 0;
        bool early = false;
        if (lane == 0 && pend_k >= 0 && !(adm > i || (adm = ld_acquire_gpu(&rp.ctl->admitted)) > i))
            flush();  // nothing to overlap with: complete the previous step now
        if (lane == 0) {
            ok = wait_admit(rp, adm, i) && wait_seen(bdone, i0 + back(k, ahead), rp);
            if (ok) {
                cursor_seek(cur, rp, i);
                early = cur.early;
                // an early step's A ticket: within kTicketRing/2 iterations of the slowest CTA's A
                // (otherwise b_done, which the B arrivals raise only after their CTA's A, bounds it)
                if (early)
                    ok = wait_seen(adone, i0 + back(k, kTicketRing / 2), rp);
                n = cur.n;
                bp = reinterpret_cast<uint64_t>(cursor_batch(cur, i));
                lp = reinterpret_cast<uint64_t>(cursor_labels(cur, i));
            }
        }
        if (!__shfl_sync(kFull, ok ? 1 : 0, 0))
            break;
        n = __shfl_sync(kFull, n, 0);
        lp = __shfl_sync(kFull, lp, 0);
        run_mark(rp, i, 2);
        const uint32_t slot = ring_slot(i, b.aug_ring);
        const uint32_t row0 = b.nmax - n;
        if (part == 0 && lane > 0) {  // m_i's labels -> m'_i's batch rows' labels (lanes 1-31,
                                      // while lane 0 drives the TMA copy)
            const uint32_t* lab = reinterpret_cast<const uint32_t*>(lp);
            uint32_t* al = reinterpret_cast<uint32_t*>(b.region[b.me] + b.off_auglab) +
                           uint64_t(slot) * b.auglab_slot_elems + row0;
#pragma unroll 4
            for (uint32_t x = lane - 1; x < n; x += 31)
                al[x] = __ldg(lab + x);
        }
        if (lane == 0) {
            const uint64_t a16 = (uint64_t(n) * S) >> 4;
            const uint64_t alo = (a16 * part / parts) << 4, ahi = (a16 * (part + 1) / parts) << 4;
            const uint32_t nA = static_cast<uint32_t>((ahi - alo + CH - 1) / CH);
            const uint8_t* batch = reinterpret_cast<const uint8_t*>(bp);
            uint8_t* dst = b.region[b.me] + b.off_aug + uint64_t(slot) * b.aug_slot_bytes + uint64_t(row0) * S;
            for (uint32_t w0 = 0; w0 < nA; w0 += kTmaStagesA) {
                const uint32_t w1 = min(nA, w0 + kTmaStagesA);
                bulk_wait_read_all();  // the ring's previous window has been stored
                for (uint32_t x = w0; x < w1; ++x) {
                    const uint64_t off = alo + uint64_t(x) * CH;
                    const uint32_t len = static_cast<uint32_t>(min64(CH, ahi - off));
                    mbar_expect_tx(bars + (x - w0), len);
                    bulk_load(ringA + (x - w0) * CH, batch + off, len, bars + (x - w0));
                }
                if (pend_k >= 0)
                    flush();  // the previous step's stores finish under these loads
                for (uint32_t x = w0; x < w1; ++x) {
                    const uint64_t off = alo + uint64_t(x) * CH;
                    const uint32_t len = static_cast<uint32_t>(min64(CH, ahi - off));
                    if (!mbar_wait(bars + (x - w0), take_phase(ph_bits, x - w0), rp.base.timeout_ns))
                        run_fail(rp, DRB_ERR_INTERNAL, (11u << 24) | uint32_t(k & 0xffffff));
                    bulk_store(dst + off, ringA + (x - w0) * CH, len);
                }
                bulk_commit();
            }
            if (pend_k >= 0)
                flush();  // (an empty batch: no window)
            pend_k = int64_t(k);
            pend_i = i;
            pend_early = early;
        }
        __syncwarp();  // (the other lanes' label stores are ordered before lane 0's later release)
    }
    if (lane == 0) {
        if (pend_k >= 0 && !run_failed(rp))
            flush();
        bulk_wait_all();
    }
}

__global__ void __launch_bounds__(kRunThreads, 1) drb_run_kernel(const __grid_constant__ RunParams rp) {
    extern __shared__ __align__(128) uint32_t sm[];
    __shared__ StepParams sp[2];
    __shared__ __align__(8) uint32_t flag[8];  // [0..1] role flags, [2..7] the plan role's counters
    // where this instance starts (written by the previous one when it left, or by start())
    const uint64_t i0 = __ldcg(&rp.ctl->next_step[rp.gen & 1]);
    const uint64_t j0 = __ldcg(&rp.ctl->next_desc[rp.gen & 1]);
    if (blockIdx.x == 0)
        run_sel_role(rp, sm, sp[0], flag, i0, j0);
    else if (blockIdx.x == 1)
        run_plan_role(rp, sm, sp[0], flag, i0);
    else
        run_copy_role(rp, sm, sp, i0, j0);
}

// ---- global-sampling bias test (proj/src/runner/bias.cpp:104-133) -----------------------
// One warp replays rank 0's global-sampling stream plan after plan — each plan's first
// counter is where the previous one stopped, so the draws are inherently sequential — and
// counts the slots hit, indexed by flat slot (worker-major, class, slot: the order of
// size_table::view::locate). total_draw = the view's total, or rank 0's own total for the
// biased control (plan_local_only, sampler.cpp:70-83: its flats are rank 0's slots).
__global__ void bias_counts_kernel(uint64_t key, uint32_t want, uint32_t total_draw, uint64_t draws,
                                   unsigned long long* counts, uint64_t* ctr_out) {
    extern __shared__ __align__(16) uint32_t acc[];
    const uint32_t lane = threadIdx.x & 31;
    if (threadIdx.x >= 32)
        return;
    uint64_t ctr = 0;
#pragma unroll 1
    for (uint64_t d = 0; d < draws; ++d) {
        const uint32_t c = warp_plan_draw(key, ctr, want, total_draw, acc);
        for (uint32_t j = lane; j < c; j += 32)
            atomicAdd(counts + acc[j], 1ull);
        __syncwarp();
    }
    if (lane == 0)
        *ctr_out = ctr;
}

// ---- standalone kernels for the buffer-level API (tests / facade) ----------------------

__global__ void rng_draw_kernel(uint64_t key, uint64_t ctr, uint64_t bound, uint64_t n,
                                uint64_t* out, uint64_t* ctr_out) {
    // sequential semantics (bounded rejection shifts later counters): one thread
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        for (uint64_t i = 0; i < n; ++i)
            out[i] = bound ? bounded_seq(key, ctr, bound) : draw_at(key, ++ctr);
        *ctr_out = ctr;
    }
}

__global__ void swor_kernel(uint64_t key, uint64_t ctr, uint32_t n, uint32_t k, uint32_t* out,
                            uint64_t* ctr_out) {
    extern __shared__ uint32_t s[];
    if (threadIdx.x < 32) {
        warp_select(key, ctr, n, k, s, s + n);
        for (uint32_t j = threadIdx.x; j < k; j += 32)
            out[j] = s[j];
        if (threadIdx.x == 0)
            *ctr_out = ctr;
    }
}

__global__ void plan_kernel(uint64_t key, uint64_t ctr, uint32_t want, uint32_t NW, uint32_t K,
                            const uint32_t* occ, uint32_t* out, uint32_t* count,
                            uint64_t* ctr_out) {
    extern __shared__ uint32_t s[];
    const uint32_t NK = NW * K;
    uint32_t* pre = s;
    uint32_t* pfx = pre + NK;
    uint32_t* acc = pfx + NK + 1;
    for (uint32_t x = threadIdx.x; x < NK; x += blockDim.x)
        pre[x] = occ[x];
    __syncwarp();
    const uint32_t total = warp_exclusive_scan(pre, NK, pfx);
    const uint32_t c = warp_plan_draw(key, ctr, want, total, acc);
    uint32_t* pl = acc + (min(want, total) ? min(want, total) : 1);
    warp_locate(acc, c, pfx, NK, K, pl);
    for (uint32_t j = threadIdx.x; j < 3 * c; j += 32)
        out[j] = pl[j];
    if (threadIdx.x == 0) {
        *count = c;
        *ctr_out = ctr;
    }
}

// read_slots (rehearsal_buffer.cpp:88-142), single-threaded resolution + CTA copy.
__global__ void read_slots_kernel(const uint8_t* slab, const uint32_t* slab_labels,
                                  const uint32_t* occ, uint32_t K, uint32_t cap, uint64_t S,
                                  const uint32_t* req, uint32_t count, uint64_t key, uint64_t ctr,
                                  uint8_t* out, uint32_t* out_labels, uint8_t* status,
                                  uint64_t* ctr_out, int64_t* src_rows) {
    if (threadIdx.x == 0) {
        uint64_t total = 0;
        for (uint32_t c = 0; c < K; ++c)
            total += occ[c];
        for (uint32_t i = 0; i < count; ++i) {
            const uint32_t cls = req[2 * i], slot = req[2 * i + 1];
            int64_t row = -1;
            uint8_t st = DRB_READ_EMPTY;
            if (cls < K && occ[cls] > 0) {
                if (slot < occ[cls]) {
                    row = int64_t(cls) * cap + slot;
                    st = DRB_READ_EXACT;
                } else {
                    row = int64_t(cls) * cap + bounded_seq(key, ctr, occ[cls]);
                    st = DRB_READ_SUBSTITUTED;
                }
            }
            if (st == DRB_READ_EMPTY && total > 0) {  // whole-buffer fallback (:106-134)
                uint64_t flat = bounded_seq(key, ctr, total);
                for (uint32_t c = 0; c < K; ++c) {
                    if (flat < occ[c]) {
                        row = int64_t(c) * cap + flat;
                        st = DRB_READ_SUBSTITUTED;
                        break;
                    }
                    flat -= occ[c];
                }
            }
            status[i] = st;
            src_rows[i] = row;
            out_labels[i] = row >= 0 ? slab_labels[row] : 0;
        }
        *ctr_out = ctr;
    }
    __syncthreads();
    for (uint32_t i = 0; i < count; ++i) {
        const int64_t row = src_rows[i];
        for (uint64_t b = threadIdx.x; b < S; b += blockDim.x)
            out[uint64_t(i) * S + b] = row >= 0 ? slab[uint64_t(row) * S + b] : 0;
    }
}

// ---- launchers ------------------------------------------------------------------------

uint32_t sel_smem_bytes(uint32_t K, uint32_t nmax) { return sel_smem(K, nmax).words * 4; }
uint32_t plan_smem_bytes(uint32_t N, uint32_t K, uint32_t r) { return plan_smem(N, K, r).words * 4; }
uint32_t plan_threads(uint32_t N) { return 32 * (N + 1 < 3 ? 3 : N + 1); }

namespace {
constexpr int kMaxDevices = 64;
// cudaFuncSetAttribute is per device: `cache` holds kMaxDevices entries
int set_smem(const void* kern, uint32_t bytes, uint32_t* cache) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices)
        return -1;
    cache += dev;
    if (bytes > *cache) {
        if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(bytes)) != cudaSuccess)
            return -1;
        // one carveout (all shared memory) for every iteration kernel, so the residency
        // arithmetic of solo_smem_for() holds and no SM reconfigures between them
        if (cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100) != cudaSuccess)
            return -1;
        *cache = bytes;
    }
    return 0;
}
}  // namespace

namespace {
int launch_ex(const void* kern, uint32_t grid, uint32_t threads, uint32_t smem, void* stream, bool pdl,
              const StepParams& p) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(threads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = static_cast<cudaStream_t>(stream);
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
    void* args[] = {const_cast<StepParams*>(&p)};
    return cudaLaunchKernelExC(&cfg, kern, args) == cudaSuccess ? 0 : -1;
}
}  // namespace

int launch_sel(const StepParams& p, void* stream, bool pdl) {
    static uint32_t cache[kMaxDevices] = {};
    const uint32_t smem = max(sel_smem_bytes(p.K, p.nmax), p.solo_smem);
    if (set_smem(reinterpret_cast<const void*>(drb_sel_kernel), smem, cache))
        return -1;
    return launch_ex(reinterpret_cast<const void*>(drb_sel_kernel), 1, kSelThreads, smem, stream, pdl, p);
}

int launch_plan_next(const StepParams& p, void* stream, bool pdl) {
    static uint32_t cache[kMaxDevices] = {};
    const uint32_t smem = max(plan_smem_bytes(p.N, p.K, p.r), p.solo_smem);
    if (set_smem(reinterpret_cast<const void*>(drb_plan_next_kernel), smem, cache))
        return -1;
    return launch_ex(reinterpret_cast<const void*>(drb_plan_next_kernel), 1, plan_threads(p.N), smem, stream, pdl,
                     p);
}

int launch_copy(const StepParams& p, uint32_t grid, void* stream, bool pdl) {
    static uint32_t cache[3][kMaxDevices] = {};
    const bool tma = p.vec16 && !(p.dbg & 16);  // DRB_DBG bit 4: LSU kernel instead of TMA
    const int which = tma ? 2 : (p.vec16 ? 1 : 0);
    auto kern = tma ? drb_copy_tma_kernel : (p.vec16 ? drb_copy_kernel<uint4> : drb_copy_kernel<uint32_t>);
    // the TMA kernel is sized for two co-resident CTAs (copy(i) + copy(i+1) under PDL)
    const uint32_t smem = tma ? tma_smem(p.N, p.r, p.nmax).bytes : p.smem_bytes;
    if (set_smem(reinterpret_cast<const void*>(kern), smem, cache[which]))
        return -1;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(tma ? kTmaThreads : kThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = static_cast<cudaStream_t>(stream);
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kern, p) == cudaSuccess ? 0 : -1;
}

uint32_t run_smem_bytes(uint32_t N, uint32_t K, uint32_t r, uint32_t nmax) {
    return run_smem(N, K, r, nmax).bytes;
}

int launch_run(const RunParams& rp, uint32_t grid, void* stream) {
    static uint32_t cache[kMaxDevices] = {};
    // one CTA per SM (each copy CTA owns an SM's share of HBM bandwidth)
    const uint32_t smem = run_smem_bytes(rp.base.N, rp.base.K, rp.base.r, rp.base.nmax);
    if (smem > 227u * 1024u)
        return -1;
    if (set_smem(reinterpret_cast<const void*>(drb_run_kernel), smem, cache))
        return -1;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kRunThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = static_cast<cudaStream_t>(stream);
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;  // every CTA co-resident: the roles spin on each other
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, drb_run_kernel, rp) == cudaSuccess ? 0 : -1;
}

int launch_peers_wait(const StepParams& p, void* stream) {
    peers_wait_kernel<<<1, 32, 0, static_cast<cudaStream_t>(stream)>>>(p);
    return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

int copy_tma_occupancy(uint32_t smem_bytes, int* out) {
    if (cudaFuncSetAttribute(drb_copy_tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(smem_bytes)) != cudaSuccess ||
        cudaFuncSetAttribute(drb_copy_tma_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, 100) != cudaSuccess)
        return -1;
    return cudaOccupancyMaxActiveBlocksPerMultiprocessor(out, drb_copy_tma_kernel, kTmaThreads, smem_bytes) ==
                   cudaSuccess
               ? 0
               : -1;
}

int copy_kernel_max_ctas_per_sm(uint32_t smem_bytes, int* out) {
    for (auto kern : {drb_copy_kernel<uint4>, drb_copy_kernel<uint32_t>}) {
        if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(smem_bytes)) != cudaSuccess)
            return -1;
    }
    return cudaOccupancyMaxActiveBlocksPerMultiprocessor(out, drb_copy_kernel<uint4>, kThreads,
                                                         smem_bytes) == cudaSuccess
               ? 0
               : -1;
}

int launch_bias_counts(uint64_t key, uint32_t want, uint32_t total_draw, uint64_t draws,
                       unsigned long long* counts_dev, uint64_t* ctr_out_dev, void* stream) {
    const size_t smem = (size_t(want) + 32) * 4;
    if (smem > 48 * 1024 &&
        cudaFuncSetAttribute(bias_counts_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)) != cudaSuccess)
        return -1;
    bias_counts_kernel<<<1, 32, smem, static_cast<cudaStream_t>(stream)>>>(key, want, total_draw, draws, counts_dev,
                                                                            ctr_out_dev);
    return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

int launch_rng_draw(uint64_t key, uint64_t ctr, uint64_t bound, uint64_t n, uint64_t* out_dev,
                    uint64_t* ctr_out_dev, void* stream) {
    rng_draw_kernel<<<1, 32, 0, static_cast<cudaStream_t>(stream)>>>(key, ctr, bound, n, out_dev,
                                                                     ctr_out_dev);
    return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

int launch_swor(uint64_t key, uint64_t ctr, uint32_t n, uint32_t k, uint32_t* out_dev,
                uint64_t* ctr_out_dev, void* stream) {
    const size_t smem = (size_t(n) * 2 + 32) * 4;
    swor_kernel<<<1, 32, smem, static_cast<cudaStream_t>(stream)>>>(key, ctr, n, k, out_dev,
                                                                    ctr_out_dev);
    return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

int launch_plan(uint64_t key, uint64_t ctr, uint32_t want, uint32_t entries, uint32_t n_workers,
                uint32_t n_classes, const uint32_t* occ_dev, uint32_t* out_dev, uint32_t* count_dev,
                uint64_t* ctr_out_dev, void* stream) {
    // entries = min(want, total) (host-computed): the kernel never holds more draws than that
    const size_t NK = size_t(n_workers) * n_classes;
    const size_t m = entries ? entries : 1;
    const size_t smem = (2 * NK + 1 + 4 * m) * 4;
    if (smem > 200 * 1024)
        return -1;
    cudaFuncSetAttribute(plan_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(smem));
    plan_kernel<<<1, 32, smem, static_cast<cudaStream_t>(stream)>>>(
        key, ctr, want, n_workers, n_classes, occ_dev, out_dev, count_dev, ctr_out_dev);
    return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

int launch_read_slots(const uint8_t* slab, const uint32_t* slab_labels, const uint32_t* occ_dev,
                      uint32_t K, uint32_t cap, uint64_t S, const uint32_t* req_dev,
                      uint32_t count, uint64_t key, uint64_t ctr, uint8_t* out,
                      uint32_t* out_labels, uint8_t* status_dev, uint64_t* ctr_out_dev,
                      void* stream) {
    int64_t* rows = nullptr;
    if (cudaMallocAsync(&rows, (count ? count : 1) * sizeof(int64_t),
                        static_cast<cudaStream_t>(stream)) != cudaSuccess)
        return -1;
    read_slots_kernel<<<1, 256, 0, static_cast<cudaStream_t>(stream)>>>(
        slab, slab_labels, occ_dev, K, cap, S, req_dev, count, key, ctr, out, out_labels,
        status_dev, ctr_out_dev, rows);
    cudaFreeAsync(rows, static_cast<cudaStream_t>(stream));
    return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

}  // namespace drb_b200

#if DRB_INSTRUMENT
// tools/ timeline probes only: one thread stores %globaltimer when the stream reaches it.
namespace {
__global__ void dbg_stamp_kernel(unsigned long long* out) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    *out = t;
}
}  // namespace
extern "C" __attribute__((visibility("default"))) int drb_dbg_stamp(unsigned long long* out, void* stream) {
    dbg_stamp_kernel<<<1, 1, 0, static_cast<cudaStream_t>(stream)>>>(out);
    return cudaGetLastError() == cudaSuccess ? 0 : -1;
}
#endif
