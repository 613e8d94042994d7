// sm_100a kernels of the distributed rehearsal buffer (arXiv 2406.03285 hot path).
//
// One launch of drb_step_kernel is one engine iteration i on one rank:
//   * S1+S2 update_buffer(m_i)          proj/src/buffer/rehearsal_buffer.cpp:14-86
//   * publish occupancy row v=i+1       proj/src/engine/engine.cpp:108-136
//   * S4 plan(i-1) for every requester  proj/src/sampler/sampler.cpp:39-68 (+ locate,
//                                       proj/src/sampler/size_table.cpp:29-39)
//   * S5 push owned plan entries (read at version i, before this round's overwrites)
//     into each requester's m'_i rows   proj/src/sampler/sampler.cpp:111-232 (fetch) and
//                                       proj/src/engine/engine.cpp:215-251 (serve_sample)
//   * augment: m'_i = m_i ++ reps(i-1)  proj/src/sampler/sampler.cpp:234-240
// The RNG decisions are bit-identical to proj/src/core/rng.cpp:12-53 and are evaluated
// warp-parallel over consecutive counters (exact rejection semantics; see warp_* below).
// Every CTA recomputes the (tiny) control decisions redundantly so no grid-wide barrier
// is needed; the byte movement is spread evenly over all CTAs as 16-byte vectors.

#include <cuda_runtime.h>

#include <cstdint>

#include "drb_internal.cuh"

namespace drb_b200 {

namespace {

constexpr unsigned kFull = 0xffffffffu;

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

// No ordering of earlier stores (a release would wait for every store of the copy to be
// acknowledged): for flags that only announce completed LOADS.
__device__ __forceinline__ void st_relaxed_sys(uint64_t* p, uint64_t v) {
    asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
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
__device__ void warp_select(uint64_t key, uint64_t& ctr, uint32_t n, uint32_t k, uint32_t* sel,
                            uint32_t* idx) {
    const int lane = threadIdx.x & 31;
    if (k == 0)
        return;
    if (k <= 32) {
        const uint32_t j = lane;
        uint32_t s = 0xffffffffu;
        bool ok = true;
        if (j < k) {
            const uint64_t nj = n - j;
            const uint64_t thr = (0ull - nj) % nj;
            const uint64_t v = draw_at(key, ctr + 1 + j);
            ok = v >= thr;
            s = j + static_cast<uint32_t>(v % nj);
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
            ctr += k;
            __syncwarp();
            return;
        }
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
__device__ void warp_assign(uint64_t ekey, uint64_t& ectr, uint32_t cap, uint32_t k,
                            const uint32_t* sel, const uint32_t* lab, uint32_t* occ,
                            uint32_t* cand_l, uint32_t* cand_slot, uint32_t* scratch,
                            uint32_t* kind, uint32_t& appends) {
    const int lane = threadIdx.x & 31;
    const uint64_t thr = (0ull - static_cast<uint64_t>(cap)) % cap;
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
            const unsigned vmask = __ballot_sync(kFull, v >= thr);
            if (static_cast<uint32_t>(__popc(vmask)) >= R) {
                const uint32_t val = static_cast<uint32_t>(v % cap);
                const int pos = rep ? static_cast<int>(__fns(vmask, 0, e + 1)) : 0;
                const uint32_t got = __shfl_sync(kFull, val, pos);
                if (rep)
                    slot = got;
                ectr += __fns(vmask, 0, R) + 1;
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
    const uint64_t thr = (0ull - static_cast<uint64_t>(total)) % total;
    uint32_t got = 0;
    while (got < want) {
        const uint64_t v = draw_at(key, ctr + 1 + lane);
        const bool ok = v >= thr;
        const uint32_t f = static_cast<uint32_t>(v % total);
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
            ctr += __fns(nm, 0, need) + 1;
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
__device__ void warp_locate(const uint32_t* acc, uint32_t cnt, const uint32_t* pfx, uint32_t NK,
                            uint32_t K, uint32_t* plan) {
    const int lane = threadIdx.x & 31;
    for (uint32_t j = lane; j < cnt; j += 32) {
        const uint32_t f = acc[j];
        uint32_t lo = 0, hi = NK;
        while (hi - lo > 1) {
            const uint32_t mid = (lo + hi) >> 1;
            if (pfx[mid] <= f)
                lo = mid;
            else
                hi = mid;
        }
        plan[3 * j] = lo / K;
        plan[3 * j + 1] = lo % K;
        plan[3 * j + 2] = f - pfx[lo];
    }
    __syncwarp();
}

// Sum of a[0..n) by one warp.
__device__ uint32_t warp_sum(const uint32_t* a, uint32_t n) {
    const int lane = threadIdx.x & 31;
    uint32_t s = 0;
    for (uint32_t i = lane; i < n; i += 32)
        s += a[i];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
        s += __shfl_xor_sync(kFull, s, o);
    return s;
}

// Exclusive prefix of a[0..n) into out[0..n] (out[n] = total), one warp: each lane scans a
// contiguous stripe, then a warp scan of the stripe totals.
__device__ uint32_t warp_exclusive_scan(const uint32_t* a, uint32_t n, uint32_t* out) {
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t per = (n + 31) / 32;
    const uint32_t b0 = min(n, lane * per), b1 = min(n, b0 + per);
    uint32_t s = 0;
    for (uint32_t i = b0; i < b1; ++i)
        s += a[i];
    uint32_t x = s;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(kFull, x, o);
        if (lane >= static_cast<uint32_t>(o))
            x += y;
    }
    uint32_t excl = x - s;
    for (uint32_t i = b0; i < b1; ++i) {
        out[i] = excl;
        excl += a[i];
    }
    const uint32_t total = __shfl_sync(kFull, x, 31);
    if (lane == 0)
        out[n] = total;
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

// One warp copies dynamically claimed chunks of 32*U vectors out of [lo, hi) (32-bit
// vector indices). `src(gv)` gives the source address of vector gv; `store(gv, v)` writes
// it to every destination of its job (and performs the job's trailing overwrite, if any,
// after those stores — the read-before-write order of a pushed slot). All U loads of a
// lane are issued before any store (memory-level parallelism).
template <typename V, int U, typename Src, typename Store>
__device__ __forceinline__ void warp_copy(uint32_t lo, uint32_t hi, uint32_t* counter, Src src,
                                          Store store) {
    const uint32_t lane = threadIdx.x & 31;
    for (;;) {
        uint32_t c = 0;
        if (lane == 0)
            c = atomicAdd(counter, 1u);
        c = __shfl_sync(kFull, c, 0);
        const uint32_t base = lo + c * (32u * U);
        if (base >= hi)
            break;
        V r[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint32_t gv = base + u * 32 + lane;
            const V* a = gv < hi ? src(gv) : nullptr;
            if (a)
                r[u] = ld_vec(a);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint32_t gv = base + u * 32 + lane;
            if (gv < hi)
                store(gv, r[u]);
        }
    }
}

// Diagnostics: sel / plan stamp slots 0-8, copy CTA 0 slots 16-19 (DRB_TRACE=1).
// Timeline (DRB_TIMELINE=<steps>): grid-wide first start / last end of each kernel of
// each step, as globaltimer ns; works inside CUDA graphs.
__device__ __forceinline__ void tl_mark(const StepParams& p, int kind, bool end) {
    if (p.timeline && threadIdx.x == 0) {
        unsigned long long* e = p.timeline + (p.step % p.timeline_steps) * kTlStride + 2 * kind;
        if (end)
            atomicMax(e + 1, globaltimer());
        else
            atomicMin(e, globaltimer());
    }
}

// per-CTA copy stamps (timeline mode): slot s of this CTA, written by the calling thread
__device__ __forceinline__ void cta_mark(const StepParams& p, int slot) {
    if (p.timeline && blockIdx.x < kTlMaxCtas) {
        uint64_t t;  // "memory": not reordered with the surrounding loads / stores
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)::"memory");
        p.timeline[(p.step % p.timeline_steps) * kTlStride + 32 + blockIdx.x * kTlCtaSlots + slot] = t;
    }
}

__device__ __forceinline__ void trace_at(const StepParams& p, int slot) {
    if (blockIdx.x == 0 && (threadIdx.x & 31) == 0) {
        if (p.trace)
            p.trace[slot] = globaltimer();
        if (p.timeline)  // phase stamps of the pipelined run: slots 8.. of the step's record
            p.timeline[(p.step % p.timeline_steps) * kTlStride + 8 + slot] = globaltimer();
    }
}

}  // namespace

// ======================================================================================
// One engine iteration i on one rank is three kernels, pipelined across iterations
// (DESIGN.md §3):
//   sel(i)   1 CTA  : S1+S2 of round i (rehearsal_buffer.cpp:14-86), the candidate-write
//                     list W_i, round-(i+1) selection state, occupancy row v=i+1 published
//                     (engine.cpp:108-136)                        — chained only on sel(i-1)
//   plan(i)  1 CTA  : size rendezvous v=i+1 (size_table.cpp:66-100), S4 plan(i) for every
//                     requester (sampler.cpp:39-68), the push list P_{i+1}, labels of
//                     m'_{i+1}'s representatives                  — chained only on plan(i-1)
//   copy(i)  grid   : m'_i = m_i ++ reps(i-1) (sampler.cpp:234-240): m_i -> m'_i, pushes of
//                     P_i (slots read at version i into each requester's m'_i), then the
//                     writes of W_i into the slab, a pushed slot only after its push read
// so copy(i) starts with every list it needs already in memory, and sel(i+1) / plan(i)
// run concurrently with copy(i) on their own streams.
// ======================================================================================

constexpr uint32_t kSelThreads = 128;

__global__ void __launch_bounds__(kSelThreads) drb_sel_kernel(const __grid_constant__ StepParams p) {
    extern __shared__ __align__(16) uint32_t sm[];
    const SelSmem L = sel_smem(p.K, p.nmax);
    uint32_t* occ = sm + L.occ;
    uint32_t* lab = sm + L.lab;
    uint32_t* sel = sm + L.sel;
    uint32_t* cand_l = sm + L.cand_l;
    uint32_t* cand_slot = sm + L.cand_slot;
    uint32_t* kind = sm + L.kind;
    uint32_t* misc = sm + L.misc;
    SelState* st = reinterpret_cast<SelState*>(misc + 16);

    const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const unsigned lt = (1u << lane) - 1u;
    const uint32_t N = p.N, K = p.K, me = p.me, n = p.n, cap = p.cap;
    const uint32_t NK = N * K;
    const bool do_update = p.mode & kModeUpdate;
    const bool do_publish = p.mode & kModePublish;
    const bool multi = (p.mode & kModePeers) && N > 1;
    const uint32_t* tin = reinterpret_cast<const uint32_t*>(p.region[me] + p.off_table) +
                          uint64_t(p.tslot_in) * NK + uint64_t(me) * K;
    trace_at(p, 0);
    tl_mark(p, 0, false);
    // one round trip: state, own occupancy row (version i), labels of m_i
    if (tid < sizeof(SelState) / 8)
        reinterpret_cast<uint64_t*>(st)[tid] = __ldcg(reinterpret_cast<const uint64_t*>(p.sel_in) + tid);
#pragma unroll 1
    for (uint32_t x = tid; x < K; x += kSelThreads)
        occ[x] = __ldcg(tin + x);
    int any_bad = 0;
#pragma unroll 1
    for (uint32_t x = tid; x < n; x += kSelThreads) {
        const uint32_t l = __ldg(p.labels + x);
        lab[x] = l;
        any_bad |= l >= K;
    }
    const bool bad = __syncthreads_or(any_bad) != 0;  // usage_error before any draw (:44-47)
    if (warp != 0)
        return;
    trace_at(p, 1);
    const bool dead = st->error != 0;  // sticky: a failed round kills the engine
    const uint32_t k = (!dead && do_update && !bad && n > 0) ? min(p.c, n) : 0;
    uint64_t cand_ctr = (p.mode & kModeCtrParams) ? p.cand_ctr0 : st->cand_ctr;
    uint64_t evict_ctr = (p.mode & kModeCtrParams) ? p.evict_ctr0 : st->evict_ctr;
    uint32_t appends = 0;
    if (k > 0) {
        warp_select(p.cand_key, cand_ctr, n, k, sel, kind);
        trace_at(p, 2);
        warp_assign(p.evict_key, evict_ctr, cap, k, sel, lab, occ, cand_l, cand_slot, misc + 32, kind,
                    appends);
    }
    trace_at(p, 3);
    // W_i: winners = last writer of each (class, slot) in selection order, ballot-ordered
    uint32_t* wl = p.wlist;
    uint32_t n_win = 0;
#pragma unroll 1
    for (uint32_t base = 0; base < k; base += 32) {
        const uint32_t t = base + lane;
        bool w = false;
        uint32_t key = 0;
        if (t < k) {
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
    // round-(i+1) selection state
    const uint32_t err = dead ? st->error : ((bad && do_update) ? DRB_ERR_USAGE : 0u);
    if (lane == 0) {
        SelState* o = p.sel_out;
        o->cand_ctr = cand_ctr;
        o->evict_ctr = evict_ctr;
        o->version = st->version + k;  // one per mutation (rehearsal_buffer.cpp:79)
        o->total = st->total + appends;
        o->cross_class = st->cross_class;
        o->error = err;
        if (p.mailbox && err)
            reinterpret_cast<volatile uint32_t*>(p.mailbox)[2 * kAugRing] = err;
    }
#pragma unroll 1
    for (uint32_t t = lane; t < k; t += 32)  // stored label == class (class-partitioned)
        p.slab_labels[cand_l[t] * cap + cand_slot[t]] = cand_l[t];
    if (do_publish && !dead) {  // publish_row(i): version i+1 (engine.cpp:108-136)
        uint32_t* tout = reinterpret_cast<uint32_t*>(p.region[me] + p.off_table) +
                         uint64_t(p.tslot_out) * NK + uint64_t(me) * K;
#pragma unroll 1
        for (uint32_t x = lane; x < K; x += 32)
            tout[x] = occ[x];
        if (multi) {
#pragma unroll 1
            for (uint32_t w = 0; w < N; ++w) {
                if (w == me)
                    continue;
                uint32_t* pt = reinterpret_cast<uint32_t*>(p.region[w] + p.off_table) +
                               uint64_t(p.tslot_out) * NK + uint64_t(me) * K;
#pragma unroll 1
                for (uint32_t x = lane; x < K; x += 32)
                    pt[x] = occ[x];
            }
            __threadfence_system();
            __syncwarp();
            if (lane < N && lane != me) {
                RegionHeader* peer = reinterpret_cast<RegionHeader*>(p.region[lane]);
                st_release_sys(&peer->occ_flag[me], p.step + 1);
            }
        }
    }
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
    trace_at(p, 4);
    tl_mark(p, 0, true);
}

__global__ void drb_plan_next_kernel(const __grid_constant__ StepParams p) {
    extern __shared__ __align__(16) uint32_t sm[];
    const PlanSmem L = plan_smem(p.N, p.K, p.r);
    uint32_t* pre = sm + L.pre;
    uint32_t* pfx = sm + L.pfx;
    uint32_t* plan = sm + L.plan;
    uint32_t* cnt = sm + L.cnt;
    uint32_t* acc = sm + L.acc;
    uint32_t* misc = sm + L.misc;
    PlanState* st = reinterpret_cast<PlanState*>(misc + 16);
    uint32_t* maskP = misc + 64;

    const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, T = blockDim.x;
    const unsigned lt = (1u << lane) - 1u;
    const uint32_t N = p.N, K = p.K, me = p.me, cap = p.cap, r = p.r;
    const uint32_t NK = N * K;
    const uint32_t MJ = plist_mj(N, r);
    const bool multi = (p.mode & kModePeers) && N > 1;
    RegionHeader* hdr = reinterpret_cast<RegionHeader*>(p.region[me]);
    trace_at(p, 5);
    tl_mark(p, 1, false);
    if (tid < sizeof(PlanState) / 8)
        reinterpret_cast<uint64_t*>(st)[tid] = __ldcg(reinterpret_cast<const uint64_t*>(p.plan_in) + tid);
    if (tid == 0)
        misc[0] = 0;
    // size rendezvous for v = i+1 (size_table.cpp:66-100 / engine.cpp:152): every peer's
    // row of this version, bounded by timeout_ns; the own row came from sel(i)
    if (multi && tid == 0) {
        const uint64_t t0 = globaltimer();
        for (uint32_t w = 0; w < N; ++w) {
            if (w == me)
                continue;
            while (ld_acquire_sys(&hdr->occ_flag[w]) < p.step + 1) {
                if (globaltimer() - t0 > p.timeout_ns) {
                    misc[0] = DRB_ERR_TRANSPORT;
                    break;
                }
                __nanosleep(32);
            }
        }
    }
    __syncthreads();
    const uint32_t* tv1 = reinterpret_cast<const uint32_t*>(p.region[me] + p.off_table) +
                          uint64_t(p.tslot_out) * NK;
#pragma unroll 1
    for (uint32_t x = tid; x < NK; x += T)
        pre[x] = __ldcg(tv1 + x);
    __syncthreads();
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
        tl_mark(p, 1, true);
        return;
    }
    // S4 plan(i): warps 1..N draw for requester q = warp-1; warp 0 builds the prefix
    if (warp >= 1 && warp <= N) {
        const uint32_t q = warp - 1;
        uint64_t ctr = st->samp_ctr[q];
        const uint32_t total = warp_sum(pre, NK);
        const uint32_t c = warp_plan_draw(p.samp_key[q], ctr, r, total, acc + q * r);
        if (lane == 0) {
            cnt[q] = c;
            p.plan_out->samp_ctr[q] = ctr;
        }
    } else if (warp == 0) {
        warp_exclusive_scan(pre, NK, pfx);
    }
    __syncthreads();
    if (warp >= 1 && warp <= N) {
        const uint32_t q = warp - 1;
        warp_locate(acc + q * r, cnt[q], pfx, NK, K, plan + 3 * q * r);
        if (q == me && (p.mode & kModeAssemble)) {  // labels of m'_{i+1}'s reps (stored label == class)
            uint32_t* al = reinterpret_cast<uint32_t*>(p.region[me] + p.off_auglab) +
                           uint64_t((p.aslot + 1) % kAugRing) * p.auglab_slot_elems;
#pragma unroll 1
            for (uint32_t j = lane; j < cnt[q]; j += 32)
                al[p.nmax + j] = plan[3 * (q * r + j) + 1];
        }
    }
    __syncthreads();
    trace_at(p, 7);
    // Pull list for copy(i+1): (a) this rank's own plan in draw order — it reads every
    // representative itself, from the owner's slab (local or over NVLink); (b) the rows of
    // MY slab that other requesters read, deduplicated in entry order (ballots), with the
    // set of readers — a write of round i+1 to such a row must wait for those reads.
    const uint32_t R = plist_r(r);
    const uint32_t mine = cnt[me];
#pragma unroll 1
    for (uint32_t j = tid; j < mine; j += T) {
        const uint32_t* x = plan + 3 * (me * r + j);
        out[4 + j] = x[0];
        out[4 + R + j] = x[1] * cap + x[2];
    }
    const uint32_t NR = N * r;
    uint32_t* rrow = out + 4 + 2 * R;
    uint32_t* rmask = rrow + MJ;
    for (uint32_t base = warp * 32; base < NR; base += T) {
        const uint32_t e = base + lane;
        bool lead = false;
        if (e < NR) {
            const uint32_t q = e / r, j = e - q * r;
            if (q != me && j < cnt[q] && plan[3 * e] == me) {
                const uint32_t cls = plan[3 * e + 1], slot = plan[3 * e + 2];
                lead = true;
#pragma unroll 1
                for (uint32_t q2 = 0; q2 < q && lead; ++q2) {
                    if (q2 == me)
                        continue;
#pragma unroll 1
                    for (uint32_t j2 = 0; j2 < cnt[q2]; ++j2) {
                        const uint32_t* x = plan + 3 * (q2 * r + j2);
                        if (x[0] == me && x[1] == cls && x[2] == slot) {
                            lead = false;
                            break;
                        }
                    }
                }
            }
        }
        const unsigned m = __ballot_sync(kFull, lead);
        if (lane == 0)
            maskP[base >> 5] = m;
    }
    __syncthreads();
    for (uint32_t base = warp * 32; base < NR; base += T) {
        const unsigned m = maskP[base >> 5];
        if (!((m >> lane) & 1u))
            continue;
        uint32_t pos = __popc(m & lt);
#pragma unroll 1
        for (uint32_t b2 = 0; b2 < (base >> 5); ++b2)
            pos += __popc(maskP[b2]);
        const uint32_t e = base + lane, q = e / r;
        const uint32_t cls = plan[3 * e + 1], slot = plan[3 * e + 2];
        uint32_t readers = 1u << q;
#pragma unroll 1
        for (uint32_t q2 = q + 1; q2 < N; ++q2) {
            if (q2 == me)
                continue;
#pragma unroll 1
            for (uint32_t j2 = 0; j2 < cnt[q2]; ++j2) {
                const uint32_t* x = plan + 3 * (q2 * r + j2);
                if (x[0] == me && x[1] == cls && x[2] == slot) {
                    readers |= 1u << q2;
                    break;
                }
            }
        }
        rrow[pos] = cls * cap + slot;
        rmask[pos] = readers;
    }
    if (tid == 0) {
        uint32_t nrem = 0;
#pragma unroll 1
        for (uint32_t b2 = 0; b2 < (NR + 31) / 32; ++b2)
            nrem += __popc(maskP[b2]);
        out[0] = mine;
        out[1] = nrem;
        p.plan_out->error = misc[0];
        if (misc[0] && p.mailbox)  // rendezvous failure: the engine is dead from here
            reinterpret_cast<volatile uint32_t*>(p.mailbox)[2 * kAugRing] = misc[0];
    }
    trace_at(p, 8);
    tl_mark(p, 1, true);
}

__device__ __forceinline__ uint4 ld_cg16(const uint4* p) {
    uint4 v;
    asm volatile("ld.global.cg.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p));
    return v;
}

template <typename V>
__device__ __forceinline__ V ld_pull(const V* p) {  // possibly a peer's memory (NVLink)
    if constexpr (sizeof(V) == 16) {
        const uint4 v = ld_cg16(reinterpret_cast<const uint4*>(p));
        return *reinterpret_cast<const V*>(&v);
    } else {
        return __ldcg(p);
    }
}

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

// Copy CTA, warp 0: wait for the staged lists (cp.async), classify W_i's writes — safe
// (rowmap when fused into A, else `win` jobs), local hazard C (`post`), remote-read D
// (`defer`) — wait for the owners of remote pulls (done >= i), publish misc[0..2] and the
// ready flag; CTA 0 also writes m'_i's batch labels and row count.
struct CopyLists {
    uint32_t *praw, *wraw, *win, *defer, *misc;
    int *post, *rowmap;
    volatile uint32_t* ready;
};
__device__ void copy_parse_lists(const StepParams& p, const CopyLists& cl, bool do_pull, bool do_update,
                                 bool multi, bool fuse) {
    const uint32_t lane = threadIdx.x & 31;
    const unsigned lt = (1u << lane) - 1u;
    const uint32_t N = p.N, me = p.me, n = p.n;
    const uint32_t R = plist_r(p.r), MJ = plist_mj(N, p.r);
    RegionHeader* hdr = reinterpret_cast<RegionHeader*>(p.region[me]);
    const uint32_t row0 = p.nmax - n;
    uint32_t* praw = cl.praw;
    uint32_t* wraw = cl.wraw;
    uint32_t* win = cl.win;
    uint32_t* defer = cl.defer;
    uint32_t* misc = cl.misc;
    int* post = cl.post;
    int* rowmap = cl.rowmap;
    volatile uint32_t* ready = cl.ready;
    const uint32_t* owner = praw + 4;
    const uint32_t* prow = praw + 4 + R;
    const uint32_t* rrow = praw + 4 + 2 * R;
    const uint32_t* rmask = rrow + MJ;
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncwarp();
    const uint32_t cnt = do_pull ? praw[0] : 0;
    const uint32_t nrem = (do_pull && multi) ? praw[1] : 0;
    const uint32_t n_win = do_update ? wraw[0] : 0;
    // round-i writes: to a row this rank pulls -> post on that pull (C); to a row a
    // remote requester pulls -> deferred (D); otherwise a plain write (B)
#pragma unroll 1
    for (uint32_t j = lane; j < cnt; j += 32)
        post[j] = -1;
    __syncwarp();
    uint32_t n_safe = 0, n_def = 0;
#pragma unroll 1
    for (uint32_t base = 0; base < n_win; base += 32) {
        const uint32_t t = base + lane;
        uint32_t row = 0, key = 0, readers = 0;
        bool local_hz = false;
        if (t < n_win) {
            row = wraw[2 + 2 * t];
            key = wraw[3 + 2 * t];
#pragma unroll 1
            for (uint32_t j = 0; j < cnt; ++j)
                if (owner[j] == me && prow[j] == key) {
                    post[j] = static_cast<int>(row);
                    local_hz = true;
                    break;
                }
#pragma unroll 1
            for (uint32_t x = 0; x < nrem; ++x)
                if (rrow[x] == key) {
                    readers = rmask[x];
                    break;
                }
        }
        const bool safe = t < n_win && !local_hz && readers == 0;
        const bool def = t < n_win && readers != 0;
        const unsigned ms = __ballot_sync(kFull, safe);
        const unsigned md = __ballot_sync(kFull, def);
        if (safe) {
            const uint32_t pos = n_safe + __popc(ms & lt);
            win[2 * pos] = row;
            win[2 * pos + 1] = key;
        }
        if (def) {  // (a local hazard that is also remote-read: D after the local read
                    //  — D runs after this CTA's barrier anyway)
            const uint32_t pos = n_def + __popc(md & lt);
            defer[3 * pos] = row;
            defer[3 * pos + 1] = key;
            defer[3 * pos + 2] = readers;
        }
        n_safe += __popc(ms);
        n_def += __popc(md);
    }
    // a local-hazard row that is also remote-read is written in D only
    if (n_def) {
#pragma unroll 1
        for (uint32_t j = lane; j < cnt; j += 32)
            if (post[j] >= 0)
#pragma unroll 1
                for (uint32_t x = 0; x < n_def; ++x)
                    if (defer[3 * x + 1] == prow[j] && owner[j] == me)
                        post[j] = -1;
    }
    // pulls from a peer need that owner's copy(i-1) complete (its slab at version i)
    if (multi && cnt) {
        uint32_t need = 0;
        for (uint32_t j = lane; j < cnt; j += 32)
            if (owner[j] != me)
                need |= 1u << owner[j];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1)
            need |= __shfl_xor_sync(kFull, need, o);
        bool ok = true;
        if (lane < N && ((need >> lane) & 1u))
            ok = wait_flag(&hdr->done[lane], p.step, p.timeout_ns);
        if (__any_sync(kFull, !ok) && lane == 0 && p.mailbox) {
            volatile uint32_t* mb = p.mailbox;
            mb[kAugRing + p.aslot] = DRB_ERR_TRANSPORT;
            mb[2 * kAugRing] = DRB_ERR_TRANSPORT;
        }
    }
    if (fuse) {
#pragma unroll 1
        for (uint32_t x = lane; x < n; x += 32)
            rowmap[x] = -1;
        __syncwarp();
#pragma unroll 1
        for (uint32_t x = lane; x < n_safe; x += 32)
            rowmap[win[2 * x]] = static_cast<int>(win[2 * x + 1]);
    }
    if (lane == 0) {
        misc[0] = cnt;
        misc[1] = fuse ? 0u : n_safe;
        misc[2] = n_def;
    }
    __syncwarp();
    __threadfence_block();
    if (lane == 0) {
        *ready = 1;
        cta_mark(p, 1);
    }
    trace_at(p, 20);
    if (blockIdx.x == 0 && (p.mode & kModeAssemble)) {
        // m'_i labels of rows [row0, row0+n) and its row count n + |reps(i-1)|
        uint32_t* al = reinterpret_cast<uint32_t*>(p.region[me] + p.off_auglab) +
                       uint64_t(p.aslot) * p.auglab_slot_elems;
#pragma unroll 1
        for (uint32_t x = lane; x < n; x += 32)
            al[row0 + x] = __ldg(p.labels + x);
        if (lane == 0) {
            hdr->aug_count[p.aslot] = n + cnt;
            if (p.mailbox) {
                volatile uint32_t* mb = p.mailbox;
                mb[p.aslot] = n + cnt;
                mb[kAugRing + p.aslot] = 0;
            }
        }
    }
}

// copy(i): m'_i = m_i ++ reps(i-1) and the slab writes of round i. Every CTA owns fixed
// slices of the vector spaces below; warps claim 32*U-vector chunks of a slice dynamically.
//   A  m_i -> m'_i rows [nmax-n, nmax)                                   (n rows)
//   B  pulls: rep j of this rank <- owner's slab row (local or a peer's over NVLink, read
//      at version i: the owner finished copy(i-1)) into m'_i row nmax+j; plus the
//      candidate writes of W_i nobody reads this round
//   C  a write to a row this rank itself pulled: by the same CTA, after the pull (barrier)
//   D  a write to a row a remote requester pulls: after that requester's pulls completed
// Multi-rank signals (peer headers, release/acquire .sys): readdone[me] after the last
// CTA's B phase, done[me] after the last CTA's writes — the only cross-rank waits are
// "owner finished copy(i-1)" before pulling from it and the rare D case.
template <typename V>
__global__ void __launch_bounds__(kThreads, 1) drb_copy_kernel(const __grid_constant__ StepParams p) {
    extern __shared__ __align__(16) uint32_t sm[];
    const CopySmem L = copy_smem(p.N, p.r, p.nmax);
    uint32_t* praw = sm + L.praw;
    uint32_t* wraw = sm + L.wraw;
    int* post = reinterpret_cast<int*>(sm + L.post);
    uint32_t* win = sm + L.win;
    uint32_t* defer = sm + L.defer;
    int* rowmap = reinterpret_cast<int*>(sm + L.rowmap);
    uint32_t* misc = sm + L.misc;

    const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const unsigned lt = (1u << lane) - 1u;
    const uint32_t N = p.N, me = p.me, n = p.n;
    const uint32_t R = plist_r(p.r), MJ = plist_mj(N, p.r);
    const uint64_t S = p.S;
    const uint32_t nvec = static_cast<uint32_t>(S / sizeof(V));
    RegionHeader* hdr = reinterpret_cast<RegionHeader*>(p.region[me]);
    const bool do_assemble = p.mode & kModeAssemble;
    const bool do_pull = (p.mode & kModePlan) && p.step > 0 && p.plist_in;
    const bool do_update = p.mode & kModeUpdate;
    const bool multi = (p.mode & kModePeers) && N > 1;
    const uint32_t part = blockIdx.x, parts = gridDim.x;
    const V* batch = reinterpret_cast<const V*>(p.batch);
    V* slab = reinterpret_cast<V*>(p.slab);
    const uint64_t aug_off = p.off_aug + uint64_t(p.aslot) * p.aug_slot_bytes;
    V* my_aug = reinterpret_cast<V*>(p.region[me] + aug_off);
    const uint32_t row0 = p.nmax - n;
    const uint32_t* owner = praw + 4;
    const uint32_t* prow = praw + 4 + R;
    const uint32_t* rrow = praw + 4 + 2 * R;
    const uint32_t* rmask = rrow + MJ;

    trace_at(p, 16);
    tl_mark(p, 2, false);
    if (threadIdx.x == 0)
        cta_mark(p, 0);
    asm volatile("griddepcontrol.launch_dependents;");
    if (p.trace && tid == 0)
        atomicMin(p.trace + 14, globaltimer());
    volatile uint32_t* ready = misc + 6;
    if (tid < 16)
        misc[tid] = 0;
    const uint32_t pw = do_pull ? plist_words(N, p.r) : 0;
    const uint32_t ww = do_update ? wlist_words(p.nmax) : 0;
    if (warp == 0) {
        // list loads first (async into shared memory), before any bulk traffic of this CTA
        asm volatile("griddepcontrol.wait;" ::: "memory");
        // copy(i-1) of this rank is complete (kernel boundary: its slab writes are visible),
        // so peers may pull round-i representatives from our slab: done[me] = i everywhere
        if (multi && blockIdx.x == 0 && lane < N)
            st_release_sys(&reinterpret_cast<RegionHeader*>(p.region[lane])->done[me], p.step);
#pragma unroll 1
        for (uint32_t x = lane; x < pw; x += 32)
            asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(praw + x))),
                         "l"(p.plist_in + x)
                         : "memory");
#pragma unroll 1
        for (uint32_t x = lane; x < ww; x += 32)
            asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(wraw + x))),
                         "l"(p.wlist + x)
                         : "memory");
        asm volatile("cp.async.commit_group;" ::: "memory");
    }
    __syncthreads();  // chunk counters / ready flag zeroed; list loads issued

    // ---- A + B with a static per-thread schedule: every thread (warp 0 included) issues
    //      its A loads at once, then (lists ready) its B loads, and only then stores — both
    //      memory latencies overlap. Thread t handles vectors lo + t + k*512 of each slice.
    //      A's stores also perform the safe candidate writes of W_i (batch row -> slab row,
    //      rowmap) from the same registers; B is then the pulls only.
    constexpr int KA = sizeof(V) == 16 ? 8 : 16;  // A vectors in flight per thread
    constexpr int KB = sizeof(V) == 16 ? 4 : 8;   // B vectors in flight per thread
    const uint32_t T = kThreads;
    const uint32_t tva = do_assemble ? n * nvec : 0;
    const uint32_t alo = static_cast<uint32_t>(uint64_t(tva) * part / parts);
    const uint32_t ahi = static_cast<uint32_t>(uint64_t(tva) * (part + 1) / parts);
    const V* batch_v = batch;
    V ra[KA];
    uint32_t a_next = alo + tid;
    const bool lists_first = p.dbg & 4;  // every warp waits for the lists before its A loads
    const bool late0 = ((p.dbg & 2) && warp == 0) || lists_first;
    if ((p.dbg >> 8) && warp != 0)
        __nanosleep(p.dbg >> 8);
    if (!late0) {
#pragma unroll
        for (int k = 0; k < KA; ++k) {
            const uint32_t gv = a_next + k * T;
            if (gv < ahi)
                ra[k] = ld_vec(batch_v + gv);
        }
    }
    const bool fuse = do_assemble && !(p.dbg & 1);  // safe writes ride on A (else: B jobs)
    if (warp == 0)
        copy_parse_lists(p, CopyLists{praw, wraw, win, defer, misc, post, rowmap, ready}, do_pull, do_update,
                         multi, fuse);
    V* asm_dst = my_aug + uint64_t(row0) * nvec;
    auto a_store = [&](uint32_t gv, const V& v) {
        asm_dst[gv] = v;
        if (fuse) {
            const uint32_t row = gv / nvec;
            const int key = rowmap[row];
            if (key >= 0)
                slab[uint64_t(key) * nvec + (gv - row * nvec)] = v;
        }
    };
    auto b_src = [&](uint32_t gv, uint32_t pv_tot) -> const V* {
        if (gv < pv_tot) {
            const uint32_t j = gv / nvec, off = gv - j * nvec;
            return reinterpret_cast<const V*>(p.slab_peer[praw[4 + j]]) + uint64_t(praw[4 + R + j]) * nvec + off;
        }
        const uint32_t wv = gv - pv_tot, job = wv / nvec, off = wv - job * nvec;
        return batch + uint64_t(win[2 * job]) * nvec + off;
    };
    auto b_store = [&](uint32_t gv, uint32_t pv_tot, const V& v) {
        if (gv < pv_tot) {
            const uint32_t j = gv / nvec, off = gv - j * nvec;
            my_aug[uint64_t(p.nmax + j) * nvec + off] = v;
        } else {
            const uint32_t wv = gv - pv_tot, job = wv / nvec, off = wv - job * nvec;
            slab[uint64_t(win[2 * job + 1]) * nvec + off] = v;
        }
    };
    if (tid == 32)
        cta_mark(p, 2);  // warp 1: A loads issued
    if (lists_first) {
        while (*ready == 0)
            __nanosleep(20);
    }
    if (late0) {
#pragma unroll
        for (int k = 0; k < KA; ++k) {
            const uint32_t gv = a_next + k * T;
            if (gv < ahi)
                ra[k] = ld_vec(batch_v + gv);
        }
    }
    // lists staged (warp 0) -> B bounds
    if (p.trace && blockIdx.x == 0 && lane == 0)
        atomicMin(p.trace + 21, globaltimer());
    while (*ready == 0)
        __nanosleep(20);
    __threadfence_block();
    if (tid == 32)
        cta_mark(p, 3);  // warp 1 past the lists-ready wait
    const uint32_t cnt = misc[0];
    const uint32_t pv_tot = cnt * nvec;
    const uint32_t tvb = pv_tot + misc[1] * nvec;
    const uint32_t blo = static_cast<uint32_t>(uint64_t(tvb) * part / parts);
    const uint32_t bhi = static_cast<uint32_t>(uint64_t(tvb) * (part + 1) / parts);
    V rb[KB];
    uint32_t b_next = blo + tid;
#pragma unroll
    for (int k = 0; k < KB; ++k) {
        const uint32_t gv = b_next + k * T;
        if (gv < bhi)
            rb[k] = ld_pull(b_src(gv, pv_tot));
    }
    if (tid == 32)
        cta_mark(p, 4);  // B loads issued
#pragma unroll
    for (int k = 0; k < KA; ++k) {
        const uint32_t gv = a_next + k * T;
        if (gv < ahi)
            a_store(gv, ra[k]);
    }
    if (tid == 32)
        cta_mark(p, 5);  // A data in, stores issued
#pragma unroll
    for (int k = 0; k < KB; ++k) {
        const uint32_t gv = b_next + k * T;
        if (gv < bhi)
            b_store(gv, pv_tot, rb[k]);
    }
    if (tid == 32)
        cta_mark(p, 6);  // B data in, stores issued
    // larger slices: further rounds
    for (a_next += KA * T; a_next < ahi; a_next += KA * T) {
#pragma unroll
        for (int k = 0; k < KA; ++k) {
            const uint32_t gv = a_next + k * T;
            if (gv < ahi)
                ra[k] = ld_vec(batch + gv);
        }
#pragma unroll
        for (int k = 0; k < KA; ++k) {
            const uint32_t gv = a_next + k * T;
            if (gv < ahi)
                a_store(gv, ra[k]);
        }
    }
    for (b_next += KB * T; b_next < bhi; b_next += KB * T) {
#pragma unroll
        for (int k = 0; k < KB; ++k) {
            const uint32_t gv = b_next + k * T;
            if (gv < bhi)
                rb[k] = ld_pull(b_src(gv, pv_tot));
        }
#pragma unroll
        for (int k = 0; k < KB; ++k) {
            const uint32_t gv = b_next + k * T;
            if (gv < bhi)
                b_store(gv, pv_tot, rb[k]);
        }
    }
    if (p.trace && blockIdx.x == 0 && lane == 0) {
        atomicMin(p.trace + 22, globaltimer());  // first warp out of the chunk loop
        atomicMax(p.trace + 18, globaltimer());  // last warp out
    }
    // ---- C: writes to rows this CTA pulled, after ALL its pulls (barrier only when this
    //      CTA has one; the condition is uniform: it reads staged lists) ------------------
    const uint32_t clo = blo, chi = min(bhi, pv_tot);
    bool any_post = false;
    if (clo < chi) {
        const uint32_t j0 = clo / nvec, j1 = (chi - 1) / nvec;
        for (uint32_t j = j0; j <= j1; ++j)
            any_post |= post[j] >= 0;
    }
    if (any_post) {
        __syncthreads();
#pragma unroll 1
        for (uint32_t gv = clo + tid; gv < chi; gv += kThreads) {
            const uint32_t j = gv / nvec, off = gv - j * nvec;
            const int pr = post[j];
            if (pr >= 0)
                slab[uint64_t(prow[j]) * nvec + off] = ld_vec(batch + uint64_t(pr) * nvec + off);
        }
    }
    trace_at(p, 19);
    if (multi) {
        const uint32_t n_def = misc[2];
        // ---- pulls of this rank done -> readdone[me] at every peer (last CTA). The pulled
        //      values were consumed before the barrier, so a relaxed ticket suffices; the
        //      flag itself is a release store (no bulk fence on the stores of the copy).
        __syncthreads();
        if (tid == 0) {
            const uint64_t t = atomicAdd(reinterpret_cast<unsigned long long*>(&hdr->rticket), 1ull);
            if ((t + 1) % gridDim.x == 0) {
                if (p.trace)
                    p.trace[23] = globaltimer();
                for (uint32_t w = 0; w < N; ++w)
                    st_relaxed_sys(&reinterpret_cast<RegionHeader*>(p.region[w])->readdone[me], p.step + 1);
            }
        }
        // ---- D: writes to rows remote requesters pull, after their pulls ------------------
        if (n_def) {
            if (tid == 0) {
                uint32_t readers = 1u << me;  // own pulls of the row too (other CTAs)
                for (uint32_t x = 0; x < n_def; ++x)
                    readers |= defer[3 * x + 2];
                for (uint32_t w = 0; w < N; ++w)
                    if (((readers >> w) & 1u) && !wait_flag(&hdr->readdone[w], p.step + 1, p.timeout_ns) &&
                        p.mailbox) {
                        volatile uint32_t* mb = p.mailbox;
                        mb[kAugRing + p.aslot] = DRB_ERR_TRANSPORT;
                        mb[2 * kAugRing] = DRB_ERR_TRANSPORT;
                    }
            }
            __syncthreads();
            const uint32_t tvd = n_def * nvec;
            const uint32_t dlo = static_cast<uint32_t>(uint64_t(tvd) * part / parts);
            const uint32_t dhi = static_cast<uint32_t>(uint64_t(tvd) * (part + 1) / parts);
#pragma unroll 1
            for (uint32_t gv = dlo + tid; gv < dhi; gv += kThreads) {
                const uint32_t x = gv / nvec, off = gv - x * nvec;
                slab[uint64_t(defer[3 * x + 1]) * nvec + off] = ld_vec(batch + uint64_t(defer[3 * x]) * nvec + off);
            }
        }
        // (done[me] = i+1 is published by copy(i+1) at its start)
    }
    if (p.trace && tid == 0)
        atomicMax(p.trace + 15, globaltimer());
    if (p.timeline) {
        __syncthreads();
        tl_mark(p, 2, true);
        if (tid == 0)
            cta_mark(p, 7);
    }
}

// ---- TMA bulk-copy path (S % 16 == 0) ---------------------------------------------------
// The same copy(i) as drb_copy_kernel, moved with the SM's TMA engine instead of LSU
// loads/stores: 1-D cp.async.bulk global->shared (mbarrier completion) and
// shared->global (bulk groups). Bytes in flight per SM are bounded by the shared-memory
// ring (kTmaStages x kTmaChunk), not by the L1 miss-tracking capacity that throttles
// 16-byte vector loads; two elected threads issue everything:
//   warp 1 lane 0  A: batch slice -> ring -> m'_i rows, then (lists parsed) the same ring
//                  bytes -> slab rows of the safe W_i winners (rowmap)
//   warp 0         staged lists (copy_parse_lists), then lane 0: B pulls owner slab ->
//                  ring -> m'_i rep rows; C: a round-i write to a pulled row is loaded
//                  alongside and stored only after the pull's load completed;
//                  non-fused safe writes (update_buffer without assembly)
//   all            D (remote-read rows, multi-GPU) after the readers' readdone, LSU path
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
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
    uint32_t ok = 0;
    while (!ok)
        asm volatile(
            "{\n .reg .pred q;\n mbarrier.try_wait.parity.shared::cta.b64 q, [%1], %2;\n selp.u32 %0, 1, 0, q;\n}"
            : "=r"(ok)
            : "r"(smem_u32(b)), "r"(parity)
            : "memory");
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

__global__ void __launch_bounds__(kTmaThreads, 1) drb_copy_tma_kernel(const __grid_constant__ StepParams p) {
    extern __shared__ __align__(128) uint32_t sm[];
    const CopySmem L = copy_smem(p.N, p.r, p.nmax);
    uint32_t* praw = sm + L.praw;
    uint32_t* wraw = sm + L.wraw;
    int* post = reinterpret_cast<int*>(sm + L.post);
    uint32_t* win = sm + L.win;
    uint32_t* defer = sm + L.defer;
    int* rowmap = reinterpret_cast<int*>(sm + L.rowmap);
    uint32_t* misc = sm + L.misc;
    const TmaSmem T = tma_smem(p.N, p.r, p.nmax);
    uint64_t* bars = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(sm) + T.bars);
    uint8_t* ring = reinterpret_cast<uint8_t*>(sm) + T.ring;

    const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t N = p.N, me = p.me, n = p.n;
    const uint32_t R = plist_r(p.r);
    const uint64_t S = p.S;
    RegionHeader* hdr = reinterpret_cast<RegionHeader*>(p.region[me]);
    const bool do_assemble = p.mode & kModeAssemble;
    const bool do_pull = (p.mode & kModePlan) && p.step > 0 && p.plist_in;
    const bool do_update = p.mode & kModeUpdate;
    const bool multi = (p.mode & kModePeers) && N > 1;
    const uint32_t part = blockIdx.x, parts = gridDim.x;
    const uint8_t* batch = reinterpret_cast<const uint8_t*>(p.batch);
    uint8_t* slab = reinterpret_cast<uint8_t*>(p.slab);
    uint8_t* my_aug = p.region[me] + p.off_aug + uint64_t(p.aslot) * p.aug_slot_bytes;
    const uint32_t row0 = p.nmax - n;
    const uint32_t* owner = praw + 4;
    const uint32_t* prow = praw + 4 + R;
    volatile uint32_t* ready = misc + 6;

    tl_mark(p, 2, false);
    if (tid == 0)
        cta_mark(p, 0);
    asm volatile("griddepcontrol.launch_dependents;");
    if (tid < 16)
        misc[tid] = 0;
    if (tid == 0 || tid == 32) {  // each engine thread owns its barriers
        const uint32_t b0 = tid == 0 ? kTmaStagesA : 0, b1 = tid == 0 ? kTmaStages + kTmaStagesB : kTmaStagesA;
        for (uint32_t b = b0; b < b1; ++b)
            mbar_init(bars + b, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    const uint32_t pw = do_pull ? plist_words(N, p.r) : 0;
    const uint32_t ww = do_update ? wlist_words(p.nmax) : 0;
    if (warp == 0) {
        asm volatile("griddepcontrol.wait;" ::: "memory");
        if (multi && blockIdx.x == 0 && lane < N)
            st_release_sys(&reinterpret_cast<RegionHeader*>(p.region[lane])->done[me], p.step);
#pragma unroll 1
        for (uint32_t x = lane; x < pw; x += 32)
            asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(praw + x)), "l"(p.plist_in + x)
                         : "memory");
#pragma unroll 1
        for (uint32_t x = lane; x < ww; x += 32)
            asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(wraw + x)), "l"(p.wlist + x)
                         : "memory");
        asm volatile("cp.async.commit_group;" ::: "memory");
    }
    __syncthreads();  // misc / ready zeroed, barriers initialised, list loads issued

    const uint32_t CH = kTmaChunk;
    if (warp == 1) {
        // ---- A engine: batch bytes [alo, ahi) of this CTA -> m'_i (+ safe slab rows) ----
        if (lane == 0) {
            const uint64_t a16 = do_assemble ? (uint64_t(n) * S) >> 4 : 0;
            const uint64_t alo = (a16 * part / parts) << 4, ahi = (a16 * (part + 1) / parts) << 4;
            const uint32_t nA = static_cast<uint32_t>((ahi - alo + CH - 1) / CH);
            uint8_t* dst = my_aug + uint64_t(row0) * S;
            uint32_t ph_base = 0;  // uses of each A barrier so far (parity)
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
                if (w0 == 0 && tid == 32)
                    cta_mark(p, 2);
                for (uint32_t k = w0; k < w1; ++k) {  // m'_i rows as soon as each piece lands
                    const uint64_t off = alo + uint64_t(k) * CH;
                    const uint32_t len = static_cast<uint32_t>(min64(CH, ahi - off));
                    mbar_wait(bars + (k - w0), ph_base & 1);
                    bulk_store(dst + off, ring + (k - w0) * CH, len);
                }
                bulk_commit();
                if (w0 == 0)
                    cta_mark(p, 5);
                if (!lists) {
                    while (*ready == 0)
                        __nanosleep(20);
                    __threadfence_block();
                    lists = true;
                    cta_mark(p, 3);
                }
                for (uint32_t k = w0; k < w1; ++k) {  // safe W_i winners among these rows
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
                ++ph_base;
            }
            bulk_wait_read_all();
            cta_mark(p, 6);
        }
    } else if (warp == 0) {
        copy_parse_lists(p, CopyLists{praw, wraw, win, defer, misc, post, rowmap, ready}, do_pull, do_update,
                         multi, do_assemble);
        if (tid == 0)
            cta_mark(p, 1);
        if (lane == 0) {
            // ---- B engine: pulls (+ C after each pull's read) and non-fused safe writes ----
            uint8_t* ringB = ring + kTmaStagesA * CH;
            uint8_t* ringC = ring + kTmaStages * CH;
            uint64_t* barB = bars + kTmaStagesA;
            uint64_t* barC = bars + kTmaStages;
            const uint32_t cnt = misc[0];
            const uint64_t pv = uint64_t(cnt) * S;
            const uint64_t sv = do_assemble ? 0 : uint64_t(misc[1]) * S;
            const uint64_t b16 = (pv + sv) >> 4;
            const uint64_t blo = (b16 * part / parts) << 4, bhi = (b16 * (part + 1) / parts) << 4;
            uint32_t use = 0;   // window count (B barrier parity)
            uint32_t cpar = 0;  // C barrier parities (bit x), armed only with a hazard
            uint64_t off = blo;
            while (off < bhi) {
                // one window: up to kTmaStagesB pieces, each inside one row and <= CH
                uint64_t poff[kTmaStagesB];
                uint32_t plen[kTmaStagesB], m = 0;
                while (m < kTmaStagesB && off < bhi) {
                    const bool is_pull = off < pv;
                    const uint64_t base = is_pull ? 0 : pv;
                    const uint32_t j = static_cast<uint32_t>((off - base) / S);
                    const uint64_t rend = min64(min64(bhi, is_pull ? pv : pv + sv), base + uint64_t(j + 1) * S);
                    const uint32_t len = static_cast<uint32_t>(min64(CH, rend - off));
                    poff[m] = off;
                    plen[m] = len;
                    const uint64_t o = off - base - uint64_t(j) * S;
                    const uint8_t* src = is_pull ? p.slab_peer[owner[j]] + uint64_t(prow[j]) * S + o
                                                 : batch + uint64_t(win[2 * j]) * S + o;
                    mbar_expect_tx(barB + m, len);
                    bulk_load(ringB + m * CH, src, len, barB + m);
                    if (is_pull && post[j] >= 0) {  // C: the new round-i bytes of the pulled row
                        mbar_expect_tx(barC + m, len);
                        bulk_load(ringC + m * CH, batch + uint64_t(post[j]) * S + o, len, barC + m);
                    }
                    off += len;
                    ++m;
                }
                if (use == 0 && tid == 0)
                    cta_mark(p, 4);
                for (uint32_t x = 0; x < m; ++x) {
                    const bool is_pull = poff[x] < pv;
                    const uint64_t base = is_pull ? 0 : pv;
                    const uint32_t j = static_cast<uint32_t>((poff[x] - base) / S);
                    const uint64_t o = poff[x] - base - uint64_t(j) * S;
                    mbar_wait(barB + x, use & 1);  // the pull's read of the slab row is complete
                    if (is_pull) {
                        bulk_store(my_aug + uint64_t(p.nmax + j) * S + o, ringB + x * CH, plen[x]);
                        if (post[j] >= 0) {
                            mbar_wait(barC + x, (cpar >> x) & 1u);
                            cpar ^= 1u << x;
                            bulk_store(slab + uint64_t(prow[j]) * S + o, ringC + x * CH, plen[x]);
                        }
                    } else {
                        bulk_store(slab + uint64_t(win[2 * j + 1]) * S + o, ringB + x * CH, plen[x]);
                    }
                }
                bulk_commit();
                bulk_wait_read_all();  // the ring is reused by the next window
                ++use;
            }
        }
    }
    __syncthreads();  // all pulls of this CTA read, all bulk stores issued and sourced
    if (multi) {
        const uint32_t n_def = misc[2];
        if (tid == 0) {
            const uint64_t t = atomicAdd(reinterpret_cast<unsigned long long*>(&hdr->rticket), 1ull);
            if ((t + 1) % gridDim.x == 0)
                for (uint32_t w = 0; w < N; ++w)
                    st_relaxed_sys(&reinterpret_cast<RegionHeader*>(p.region[w])->readdone[me], p.step + 1);
        }
        if (n_def) {  // D: rows remote requesters pull, after their pulls (LSU path, rare)
            if (tid == 0) {
                uint32_t readers = 1u << me;
                for (uint32_t x = 0; x < n_def; ++x)
                    readers |= defer[3 * x + 2];
                for (uint32_t w = 0; w < N; ++w)
                    if (((readers >> w) & 1u) && !wait_flag(&hdr->readdone[w], p.step + 1, p.timeout_ns) &&
                        p.mailbox) {
                        volatile uint32_t* mb = p.mailbox;
                        mb[kAugRing + p.aslot] = DRB_ERR_TRANSPORT;
                        mb[2 * kAugRing] = DRB_ERR_TRANSPORT;
                    }
            }
            __syncthreads();
            const uint32_t nvec = static_cast<uint32_t>(S / 16);
            const uint32_t tvd = n_def * nvec;
            const uint32_t dlo = static_cast<uint32_t>(uint64_t(tvd) * part / parts);
            const uint32_t dhi = static_cast<uint32_t>(uint64_t(tvd) * (part + 1) / parts);
            const uint4* bv = reinterpret_cast<const uint4*>(batch);
            uint4* sv = reinterpret_cast<uint4*>(slab);
#pragma unroll 1
            for (uint32_t gv = dlo + tid; gv < dhi; gv += blockDim.x) {
                const uint32_t x = gv / nvec, o = gv - x * nvec;
                sv[uint64_t(defer[3 * x + 1]) * nvec + o] = ld_vec(bv + uint64_t(defer[3 * x]) * nvec + o);
            }
        }
    }
    if (p.timeline) {
        __syncthreads();
        tl_mark(p, 2, true);
        if (tid == 0)
            cta_mark(p, 7);
    }
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
        *cache = bytes;
    }
    return 0;
}
}  // namespace

int launch_sel(const StepParams& p, void* stream) {
    static uint32_t cache[kMaxDevices] = {};
    const uint32_t smem = max(sel_smem_bytes(p.K, p.nmax), p.solo_smem);
    if (set_smem(reinterpret_cast<const void*>(drb_sel_kernel), smem, cache))
        return -1;
    drb_sel_kernel<<<1, kSelThreads, smem, static_cast<cudaStream_t>(stream)>>>(p);
    return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

int launch_plan_next(const StepParams& p, void* stream) {
    static uint32_t cache[kMaxDevices] = {};
    const uint32_t smem = max(plan_smem_bytes(p.N, p.K, p.r), p.solo_smem);
    if (set_smem(reinterpret_cast<const void*>(drb_plan_next_kernel), smem, cache))
        return -1;
    drb_plan_next_kernel<<<1, plan_threads(p.N), smem, static_cast<cudaStream_t>(stream)>>>(p);
    return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

int launch_copy(const StepParams& p, uint32_t grid, void* stream, bool pdl) {
    static uint32_t cache[3][kMaxDevices] = {};
    const bool tma = p.vec16 && !(p.dbg & 16);  // DRB_DBG bit 4: LSU kernel instead of TMA
    const int which = tma ? 2 : (p.vec16 ? 1 : 0);
    auto kern = tma ? drb_copy_tma_kernel : (p.vec16 ? drb_copy_kernel<uint4> : drb_copy_kernel<uint32_t>);
    const uint32_t smem = tma ? max(p.smem_bytes, tma_smem(p.N, p.r, p.nmax).bytes) : p.smem_bytes;
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

int launch_plan(uint64_t key, uint64_t ctr, uint32_t want, uint32_t n_workers, uint32_t n_classes,
                const uint32_t* occ_dev, uint32_t* out_dev, uint32_t* count_dev,
                uint64_t* ctr_out_dev, void* stream) {
    const uint32_t NK = n_workers * n_classes;
    const size_t smem = (2 * size_t(NK) + 1 + size_t(want + 1) * 4) * 4;
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
