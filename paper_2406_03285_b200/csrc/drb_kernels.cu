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
            int pa = -1, q = -1;
#pragma unroll
            for (int m = 0; m < 32; ++m) {
                const uint32_t sm = __shfl_sync(kFull, s, m);
                if (m < lane && j < k) {
                    if (sm == j)
                        pa = m;
                    if (sm == s)
                        q = m;
                }
            }
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
        uint32_t rho = 0;
        bool last_of_class = true;
#pragma unroll
        for (int m = 0; m < 32; ++m) {
            const uint32_t lm = __shfl_sync(kFull, L, m);
            if (act && lm == L) {
                if (m < lane)
                    ++rho;
                if (m > lane)
                    last_of_class = false;
            }
        }
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

// S4 — plan(want, view) (sampler.cpp:39-68) for one requester, one full warp.
// pre: exclusive prefix of the view's occupancy [N*K] with pre[NK] = total.
// Draws are bounded(total) on consecutive counters; lane l holds counter ctr+1+l.
// Rejected draws are skipped, duplicates (of accepted flats or of earlier lanes in the
// same batch) consume their counter without producing an entry — exactly the
// `while (|out| < want) { f = bounded(total); if (insert(f)) out.push(locate(f)); }`
// loop. The counter advances to the draw that completed the plan.
// Exhaustion (want >= total) lists every slot in flat order with no draws.
// locate (size_table.cpp:29-39) is a binary search over pre (largest i with pre[i] <= f).
__device__ uint32_t warp_plan(uint64_t key, uint64_t& ctr, uint32_t want, const uint32_t* pre,
                              uint32_t NK, uint32_t K, uint32_t* acc, uint32_t* plan) {
    const int lane = threadIdx.x & 31;
    const unsigned lt = (1u << lane) - 1u;
    const uint32_t total = pre[NK];
    if (want == 0 || total == 0)
        return 0;
    uint32_t cnt;
    if (want >= total) {
        cnt = total;
        for (uint32_t j = lane; j < total; j += 32)
            acc[j] = j;
    } else {
        const uint64_t thr = (0ull - static_cast<uint64_t>(total)) % total;
        uint32_t got = 0;
        while (got < want) {
            const uint64_t v = draw_at(key, ctr + 1 + lane);
            const bool ok = v >= thr;
            const uint32_t f = static_cast<uint32_t>(v % total);
            bool dup = !ok;
#pragma unroll
            for (int m = 0; m < 32; ++m) {
                const uint32_t fm = __shfl_sync(kFull, f, m);
                const int okm = __shfl_sync(kFull, static_cast<int>(ok), m);
                if (m < lane && okm && fm == f)
                    dup = true;
            }
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
        cnt = want;
    }
    __syncwarp();
    for (uint32_t j = lane; j < cnt; j += 32) {
        const uint32_t f = acc[j];
        uint32_t lo = 0, hi = NK;
        while (hi - lo > 1) {
            const uint32_t mid = (lo + hi) >> 1;
            if (pre[mid] <= f)
                lo = mid;
            else
                hi = mid;
        }
        plan[3 * j] = lo / K;
        plan[3 * j + 1] = lo % K;
        plan[3 * j + 2] = f - pre[lo];
    }
    __syncwarp();
    return cnt;
}

// Block-wide exclusive scan of a[0..n) in place, a[n] = total. All threads participate.
__device__ uint32_t block_exclusive_scan(uint32_t* a, uint32_t n, uint32_t* wtot) {
    const uint32_t T = blockDim.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t nw = T >> 5;
    const uint32_t per = (n + T - 1) / T;
    const uint32_t b0 = min(n, tid * per), b1 = min(n, b0 + per);
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
    if (lane == 31)
        wtot[warp] = x;
    __syncthreads();
    if (warp == 0) {
        uint32_t w = lane < nw ? wtot[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(kFull, w, o);
            if (lane >= static_cast<uint32_t>(o))
                w += y;
        }
        if (lane < nw)
            wtot[lane] = w;
    }
    __syncthreads();
    uint32_t excl = x - s + (warp ? wtot[warp - 1] : 0);
    for (uint32_t i = b0; i < b1; ++i) {
        const uint32_t v = a[i];
        a[i] = excl;
        excl += v;
    }
    const uint32_t total = wtot[nw - 1];
    __syncthreads();
    if (tid == 0)
        a[n] = total;
    __syncthreads();
    return total;
}

// Copy `len` vectors (16 B, or 4 B when !vec16) from src to up to 1+kMaxWorld dsts, then
// optionally overwrite post_dst with post_src — in that order per vector and per thread,
// which is what lets a slot be read for a push and overwritten by this round's candidate
// in the same launch (exact-horizon semantics).
template <typename V, int U>
__device__ __forceinline__ void copy_run(const V* src, V* const* dsts, int nd, const V* post_src,
                                         V* post_dst, uint64_t len, uint32_t first,
                                         uint32_t stride) {
    for (uint64_t i = first; i < len; i += uint64_t(stride) * U) {
        V r[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint64_t x = i + uint64_t(u) * stride;
            if (x < len) {
                if constexpr (sizeof(V) == 16)
                    r[u] = ld_stream(reinterpret_cast<const uint4*>(src + x));
                else
                    r[u] = __ldg(src + x);
            }
        }
        for (int d = 0; d < nd; ++d) {
            V* dst = dsts[d];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const uint64_t x = i + uint64_t(u) * stride;
                if (x < len)
                    dst[x] = r[u];
            }
        }
        if (post_dst) {
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const uint64_t x = i + uint64_t(u) * stride;
                if (x < len) {
                    if constexpr (sizeof(V) == 16)
                        r[u] = ld_stream(reinterpret_cast<const uint4*>(post_src + x));
                    else
                        r[u] = __ldg(post_src + x);
                }
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const uint64_t x = i + uint64_t(u) * stride;
                if (x < len)
                    post_dst[x] = r[u];
            }
        }
    }
}

// Even split of a virtual vector space [0, jobs*nvec) over the grid; `resolve(job, ...)`
// yields the byte pointers of one job.
template <typename V, int U, typename Resolve>
__device__ __forceinline__ void copy_space(uint32_t jobs, uint64_t nvec, uint32_t first,
                                           uint32_t stride, uint32_t part, uint32_t parts,
                                           Resolve resolve) {
    const uint64_t tv = uint64_t(jobs) * nvec;
    if (tv == 0)
        return;
    uint64_t lo = tv * part / parts, hi = tv * (part + 1) / parts;
    while (lo < hi) {
        const uint32_t job = static_cast<uint32_t>(lo / nvec);
        const uint64_t in_row = lo - uint64_t(job) * nvec;
        const uint64_t end = min(hi, uint64_t(job + 1) * nvec);
        const uint8_t* src = nullptr;
        uint8_t* dst8[1 + kMaxWorld];
        int nd = 0;
        const uint8_t* psrc = nullptr;
        uint8_t* pdst = nullptr;
        resolve(job, src, dst8, nd, psrc, pdst);
        V* dsts[1 + kMaxWorld];
        for (int d = 0; d < nd; ++d)
            dsts[d] = reinterpret_cast<V*>(dst8[d]) + in_row;
        copy_run<V, U>(reinterpret_cast<const V*>(src) + in_row, dsts, nd,
                       psrc ? reinterpret_cast<const V*>(psrc) + in_row : nullptr,
                       pdst ? reinterpret_cast<V*>(pdst) + in_row : nullptr, end - lo, first,
                       stride);
        lo = end;
    }
}

}  // namespace

// misc[] words (shared)
enum : uint32_t {
    kMiscErr = 0,       // error detected this launch
    kMiscBad = 1,       // a label >= K
    kMiscJobs = 2,      // push-job counter
    kMiscWin = 3,       // winner (candidate-write) job counter
    kMiscCtr = 4,       // 4 words: cand_ctr, evict_ctr (u64 each)
    kMiscApp = 8,       // appends
    kMiscWtot = 12,     // 16 words: scan warp totals
    kMiscScratch = 12,  // aliases wtot (eviction fallback scratch, used after the scan)
};

__global__ void __launch_bounds__(kThreads, 1) drb_step_kernel(const __grid_constant__ StepParams p) {
    extern __shared__ __align__(16) uint32_t sm[];
    const SmemLayout L = smem_layout(p.N, p.K, p.nmax, p.r);
    uint32_t* pre = sm + L.pre;
    uint32_t* occ = sm + L.occ;
    uint32_t* lab = sm + L.lab;
    uint32_t* sel = sm + L.sel;
    uint32_t* cand_l = sm + L.cand_l;
    uint32_t* cand_slot = sm + L.cand_slot;
    uint32_t* win = sm + L.win;  // candidate-write jobs: (batch row, slab row) pairs
    uint32_t* kind = sm + L.idx; // per candidate: 1 = append (after selection, idx is free)
    uint32_t* plan = sm + L.plan;
    uint32_t* cnt = sm + L.cnt;
    uint32_t* acc = sm + L.acc;
    uint32_t* hkey = sm + L.hkey;
    uint32_t* hfirst = sm + L.hfirst;
    uint32_t* hjob = sm + L.hjob;
    uint32_t* pj_src = sm + L.pj_src;
    int* pj_post = reinterpret_cast<int*>(sm + L.pj_post);
    uint32_t* pj_ndst = sm + L.pj_ndst;
    uint32_t* pj_dst = sm + L.pj_dst;
    uint32_t* misc = sm + L.misc;

    const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t T = blockDim.x;
    const bool leader = blockIdx.x == 0;
    const uint32_t N = p.N, K = p.K, me = p.me, n = p.n, cap = p.cap, r = p.r;
    const uint32_t NK = N * K;
    const uint64_t S = p.S;
    RegionHeader* hdr = reinterpret_cast<RegionHeader*>(p.region[me]);
    const bool do_update = p.mode & kModeUpdate;
    const bool do_assemble = p.mode & kModeAssemble;
    const bool do_plan = (p.mode & kModePlan) && p.step > 0;
    const bool do_publish = p.mode & kModePublish;
    const bool multi = (p.mode & kModePeers) && N > 1;
    constexpr uint32_t kEmpty = 0xffffffffu;

    if (tid < 32)
        misc[tid] = 0;
    for (uint32_t x = tid; x <= L.hmask; x += T) {
        hkey[x] = kEmpty;
        hfirst[x] = kEmpty;
    }
    const uint32_t dead = __ldcg(&p.st_in->error);
    if (dead) {  // sticky: a failed round kills the engine (engine.cpp:67-68,188-198)
        if (leader && tid == 0) {
            *p.st_out = *p.st_in;
            if (p.mailbox) {
                volatile uint32_t* mb = p.mailbox;
                mb[p.aslot] = 0;
                mb[kAugRing + p.aslot] = dead;
                mb[2 * kAugRing] = dead;
            }
        }
        return;
    }

    uint8_t* my_aug = p.region[me] + p.off_aug + uint64_t(p.aslot) * p.aug_slot_bytes;
    uint32_t* my_auglab = reinterpret_cast<uint32_t*>(p.region[me] + p.off_auglab) +
                          uint64_t(p.aslot) * p.auglab_slot_elems;
    const uint32_t row0 = p.nmax - n;  // m'_i occupies rows [nmax-n, nmax+|reps|)

    // Phase A0: loads that need no peer (own occupancy at version i, batch labels).
    const uint32_t* table = reinterpret_cast<const uint32_t*>(p.region[me] + p.off_table);
    const uint32_t* tin = table + uint64_t(p.tslot_in) * NK;
    __syncthreads();
    for (uint32_t x = tid; x < K; x += T)
        occ[x] = __ldcg(tin + uint64_t(me) * K + x);
    for (uint32_t x = tid; x < n; x += T) {
        const uint32_t l = __ldg(p.labels + x);
        lab[x] = l;
        if (l >= K)
            misc[kMiscBad] = 1;
    }

    // Phase A1: wait for every peer's occupancy row of version i (the size rendezvous,
    // size_table.cpp:66-100 / engine.cpp:152), bounded by timeout_ns.
    if (do_plan && multi && tid == 0) {
        const uint64_t t0 = globaltimer();
        for (uint32_t w = 0; w < N; ++w) {
            if (w == me)
                continue;
            while (ld_acquire_sys(&hdr->occ_flag[w]) < p.step) {
                if (globaltimer() - t0 > p.timeout_ns) {
                    misc[kMiscErr] = DRB_ERR_TRANSPORT;
                    break;
                }
                __nanosleep(64);
            }
        }
    }
    __syncthreads();
    if (do_plan) {
        for (uint32_t x = tid; x < NK; x += T)
            pre[x] = __ldcg(tin + x);
        __syncthreads();
        block_exclusive_scan(pre, NK, misc + kMiscWtot);
    }
    const bool bad = misc[kMiscBad] != 0;  // label >= K: usage_error before any draw (:44-47)
    const uint32_t k = (do_update && !bad && n > 0) ? min(p.c, n) : 0;

    // Phase B: control decisions, redundantly in every CTA.
    //   warp 0      : S1 selection + S2 slot assignment of this rank's candidates
    //   warps 1..N  : S4 plan(i-1) of requester q = warp-1 (each rank replicates every
    //                 requester's global-sampling stream, so owners know what to push)
    if (warp == 0) {
        uint64_t cand_ctr = (p.mode & kModeCtrParams) ? p.cand_ctr0 : p.st_in->cand_ctr;
        uint64_t evict_ctr = (p.mode & kModeCtrParams) ? p.evict_ctr0 : p.st_in->evict_ctr;
        uint32_t appends = 0;
        if (k > 0) {
            warp_select(p.cand_key, cand_ctr, n, k, sel, kind);
            warp_assign(p.evict_key, evict_ctr, cap, k, sel, lab, occ, cand_l, cand_slot,
                        misc + kMiscScratch, kind, appends);
        }
        if (lane == 0) {
            reinterpret_cast<uint64_t*>(misc + kMiscCtr)[0] = cand_ctr;
            reinterpret_cast<uint64_t*>(misc + kMiscCtr)[1] = evict_ctr;
            misc[kMiscApp] = appends;
        }
    } else if (do_plan && warp <= N) {
        const uint32_t q = warp - 1;
        uint64_t ctr = p.st_in->samp_ctr[q];
        const uint32_t c = warp_plan(p.samp_key[q], ctr, r, pre, NK, K, acc + q * r,
                                     plan + 3 * q * r);
        if (lane == 0) {
            cnt[q] = c;
            if (leader)
                p.st_out->samp_ctr[q] = ctr;
        }
    }
    __syncthreads();

    // Phase C: job construction.
    //  C1: owned plan entries (any requester) insert their slab row into a shared hash
    //      table keeping the first entry index -> one push job per distinct slot.
    const uint32_t NR = do_plan ? N * r : 0;
    for (uint32_t e = tid; e < NR; e += T) {
        const uint32_t q = e / r, j = e - q * r;
        if (j < cnt[q] && plan[3 * e] == me) {
            const uint32_t key = plan[3 * e + 1] * cap + plan[3 * e + 2];
            uint32_t h = (key * 0x9e3779b1u) & L.hmask;
            for (;;) {
                const uint32_t prev = atomicCAS(&hkey[h], kEmpty, key);
                if (prev == kEmpty || prev == key) {
                    atomicMin(&hfirst[h], e);
                    break;
                }
                h = (h + 1) & L.hmask;
            }
        }
    }
    __syncthreads();
    //  C2: the first entry of each slot allocates the push job.
    for (uint32_t e = tid; e < NR; e += T) {
        const uint32_t q = e / r, j = e - q * r;
        if (j < cnt[q] && plan[3 * e] == me) {
            const uint32_t key = plan[3 * e + 1] * cap + plan[3 * e + 2];
            uint32_t h = (key * 0x9e3779b1u) & L.hmask;
            while (hkey[h] != key)
                h = (h + 1) & L.hmask;
            if (hfirst[h] == e) {
                const uint32_t pj = atomicAdd(&misc[kMiscJobs], 1u);
                hjob[h] = pj;
                pj_src[pj] = key;
                pj_ndst[pj] = 0;
                pj_post[pj] = -1;
            }
        }
    }
    __syncthreads();
    //  C3: every owned entry registers its destination row (requester q, rep j);
    //      every winning candidate (last writer of its (class, slot) in selection order)
    //      becomes either a candidate-write job or, if its slot is also read by a push
    //      this round, the push job's trailing overwrite (read-before-write hazard).
    for (uint32_t e = tid; e < NR; e += T) {
        const uint32_t q = e / r, j = e - q * r;
        if (j < cnt[q] && plan[3 * e] == me) {
            const uint32_t key = plan[3 * e + 1] * cap + plan[3 * e + 2];
            uint32_t h = (key * 0x9e3779b1u) & L.hmask;
            while (hkey[h] != key)
                h = (h + 1) & L.hmask;
            const uint32_t pj = hjob[h];
            const uint32_t slotpos = atomicAdd(&pj_ndst[pj], 1u);
            pj_dst[pj * N + slotpos] = (q << 16) | j;
        }
    }
    for (uint32_t t = tid; t < k; t += T) {
        bool winner = true;
        for (uint32_t u = t + 1; u < k; ++u)
            if (cand_l[u] == cand_l[t] && cand_slot[u] == cand_slot[t])
                winner = false;
        if (!winner)
            continue;
        const uint32_t key = cand_l[t] * cap + cand_slot[t];
        int hazard_job = -1;
        if (NR) {
            uint32_t h = (key * 0x9e3779b1u) & L.hmask;
            while (hkey[h] != kEmpty) {
                if (hkey[h] == key) {
                    hazard_job = static_cast<int>(hjob[h]);
                    break;
                }
                h = (h + 1) & L.hmask;
            }
        }
        if (hazard_job >= 0) {
            pj_post[hazard_job] = static_cast<int>(sel[t]);
        } else {
            const uint32_t w = atomicAdd(&misc[kMiscWin], 1u);
            win[2 * w] = sel[t];
            win[2 * w + 1] = key;
        }
    }
    __syncthreads();
    const uint32_t n_win = misc[kMiscWin];
    const uint32_t n_push = misc[kMiscJobs];

    // Phase D (leader CTA): state for round i+1, occupancy publish, m' labels, report.
    if (leader) {
        const uint64_t cctr = reinterpret_cast<uint64_t*>(misc + kMiscCtr)[0];
        const uint64_t ectr = reinterpret_cast<uint64_t*>(misc + kMiscCtr)[1];
        const uint32_t appends = misc[kMiscApp];
        const uint32_t err = misc[kMiscErr] | ((bad && do_update) ? DRB_ERR_USAGE : 0u);
        if (tid == 0) {
            DevState* o = p.st_out;
            o->cand_ctr = cctr;
            o->evict_ctr = ectr;
            o->version = p.st_in->version + k;  // one per mutation (rehearsal_buffer.cpp:79)
            o->total = p.st_in->total + appends;
            o->cross_class = p.st_in->cross_class;
            o->error = err;
            if (!do_plan)
                for (uint32_t q = 0; q < N; ++q)
                    o->samp_ctr[q] = p.st_in->samp_ctr[q];
        }
        for (uint32_t t = tid; t < k; t += T)  // stored label == class (class-partitioned)
            p.slab_labels[cand_l[t] * cap + cand_slot[t]] = cand_l[t];
        if (do_publish) {  // publish_row(i): version i+1 (engine.cpp:108-136)
            uint32_t* tout_local = reinterpret_cast<uint32_t*>(p.region[me] + p.off_table) +
                                   uint64_t(p.tslot_out) * NK + uint64_t(me) * K;
            for (uint32_t x = tid; x < K; x += T)
                tout_local[x] = occ[x];
            if (multi) {
                for (uint32_t w = 0; w < N; ++w) {
                    if (w == me)
                        continue;
                    uint32_t* tout = reinterpret_cast<uint32_t*>(p.region[w] + p.off_table) +
                                     uint64_t(p.tslot_out) * NK + uint64_t(me) * K;
                    for (uint32_t x = tid; x < K; x += T)
                        tout[x] = occ[x];
                }
                __threadfence_system();
                __syncthreads();
                if (tid < N && tid != me) {
                    RegionHeader* peer = reinterpret_cast<RegionHeader*>(p.region[tid]);
                    st_release_sys(&peer->occ_flag[me], p.step + 1);
                }
            }
        }
        if (do_assemble) {
            for (uint32_t x = tid; x < n; x += T)
                my_auglab[row0 + x] = lab[x];
            const uint32_t mine = do_plan ? cnt[me] : 0;
            for (uint32_t j = tid; j < mine; j += T)
                my_auglab[p.nmax + j] = plan[3 * (me * r + j) + 1];
            if (tid == 0) {
                hdr->aug_count[p.aslot] = n + mine;
                if (p.mailbox) {
                    // m'_i itself is only invalid on a rendezvous failure; a bad label kills
                    // the engine for the NEXT update (engine.cpp:188-198 then :67-68).
                    volatile uint32_t* mb = p.mailbox;
                    mb[p.aslot] = n + mine;
                    mb[kAugRing + p.aslot] = misc[kMiscErr];
                    if (err)
                        mb[2 * kAugRing] = err;
                }
            }
        }
        if (p.mode & kModeReport) {  // insertion_report (rehearsal_buffer.hpp:17-26)
            for (uint32_t x = tid; x < 2 * K + 2; x += T)
                p.report[x] = 0;
            __syncthreads();
            for (uint32_t t = tid; t < k; t += T) {
                const bool app = kind[t] != 0;
                atomicAdd(&p.report[(app ? 0 : K) + cand_l[t]], 1u);
                atomicAdd(&p.report[2 * K + (app ? 0 : 1)], 1u);
            }
        }
    }

    // Phase E: byte movement. Three job spaces, each split evenly over the grid:
    //   assemble : m_i row x            -> m'_i row row0+x                 (n jobs)
    //   write    : m_i row x (winner)   -> slab[L][slot]                   (n_win jobs)
    //   push     : slab[cls][slot]      -> m'_i(q) row nmax+j for each requester entry
    //              that drew it, then (hazard) m_i row -> slab[cls][slot]  (n_push jobs)
    const uint32_t part = blockIdx.x, parts = gridDim.x;
    auto run = [&](auto vec_tag) {
        using V = decltype(vec_tag);
        const uint64_t nvec = S / sizeof(V);
        constexpr int U = sizeof(V) == 16 ? 4 : 8;
        if (do_assemble)
            copy_space<V, U>(n, nvec, tid, T, part, parts,
                             [&](uint32_t job, const uint8_t*& src, uint8_t** d, int& nd,
                                 const uint8_t*&, uint8_t*&) {
                                 src = p.batch + uint64_t(job) * S;
                                 d[0] = my_aug + uint64_t(row0 + job) * S;
                                 nd = 1;
                             });
        copy_space<V, U>(n_win, nvec, tid, T, part, parts,
                         [&](uint32_t job, const uint8_t*& src, uint8_t** d, int& nd,
                             const uint8_t*&, uint8_t*&) {
                             src = p.batch + uint64_t(win[2 * job]) * S;
                             d[0] = p.slab + uint64_t(win[2 * job + 1]) * S;
                             nd = 1;
                         });
        copy_space<V, U>(n_push, nvec, tid, T, part, parts,
                         [&](uint32_t job, const uint8_t*& src, uint8_t** d, int& nd,
                             const uint8_t*& psrc, uint8_t*& pdst) {
                             src = p.slab + uint64_t(pj_src[job]) * S;
                             nd = static_cast<int>(pj_ndst[job]);
                             for (int x = 0; x < nd; ++x) {
                                 const uint32_t e = pj_dst[job * N + x];
                                 const uint32_t q = e >> 16, j = e & 0xffffu;
                                 d[x] = p.region[q] + p.off_aug +
                                        uint64_t(p.aslot) * p.aug_slot_bytes +
                                        uint64_t(p.nmax + j) * S;
                             }
                             if (pj_post[job] >= 0) {
                                 psrc = p.batch + uint64_t(pj_post[job]) * S;
                                 pdst = p.slab + uint64_t(pj_src[job]) * S;
                             }
                         });
    };
    if (p.vec16)
        run(uint4{});
    else
        run(uint32_t{});

    // Phase F (multi-rank): completion handshake. The last CTA of this rank to finish
    // tells every requester that all pushes of step i into it have landed, then waits
    // until every owner has done the same for us — so this launch's completion implies
    // m'_i is complete (the promise resolution of engine.cpp:169).
    if (do_plan && multi) {
        __threadfence_system();
        __syncthreads();
        if (tid == 0) {
            const uint64_t t = atomicAdd(reinterpret_cast<unsigned long long*>(&hdr->ticket), 1ull);
            if ((t + 1) % gridDim.x == 0) {
                __threadfence_system();
                for (uint32_t w = 0; w < N; ++w) {
                    if (w == me)
                        continue;
                    RegionHeader* peer = reinterpret_cast<RegionHeader*>(p.region[w]);
                    st_release_sys(&peer->arrive[me], p.step + 1);
                }
                const uint64_t t0 = globaltimer();
                bool to = false;
                for (uint32_t w = 0; w < N && !to; ++w) {
                    if (w == me)
                        continue;
                    while (ld_acquire_sys(&hdr->arrive[w]) < p.step + 1) {
                        if (globaltimer() - t0 > p.timeout_ns) {
                            to = true;
                            break;
                        }
                        __nanosleep(64);
                    }
                }
                if (to) {
                    atomicOr(&p.st_out->error, static_cast<uint32_t>(DRB_ERR_TRANSPORT));
                    if (p.mailbox) {
                        volatile uint32_t* mb = p.mailbox;
                        mb[kAugRing + p.aslot] = DRB_ERR_TRANSPORT;
                        mb[2 * kAugRing] = DRB_ERR_TRANSPORT;
                    }
                }
            }
        }
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
    uint32_t* wtot = s + NK + 1;
    uint32_t* acc = wtot + 32;
    for (uint32_t x = threadIdx.x; x < NK; x += blockDim.x)
        pre[x] = occ[x];
    __syncthreads();
    const uint32_t total = block_exclusive_scan(pre, NK, wtot);
    const uint32_t cap_entries = min(want, total);
    uint32_t* pl = acc + (cap_entries ? cap_entries : 1);
    if (threadIdx.x < 32) {
        const uint32_t c = warp_plan(key, ctr, want, pre, NK, K, acc, pl);
        for (uint32_t j = threadIdx.x; j < 3 * c; j += 32)
            out[j] = pl[j];
        if (threadIdx.x == 0) {
            *count = c;
            *ctr_out = ctr;
        }
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

int launch_step(const StepParams& p, uint32_t grid, void* stream) {
    static bool attr_set = false;
    static uint32_t attr_bytes = 0;
    if (!attr_set || p.smem_bytes > attr_bytes) {
        if (cudaFuncSetAttribute(drb_step_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(p.smem_bytes)) != cudaSuccess)
            return -1;
        attr_set = true;
        attr_bytes = p.smem_bytes;
    }
    drb_step_kernel<<<grid, kThreads, p.smem_bytes, static_cast<cudaStream_t>(stream)>>>(p);
    return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

int step_kernel_max_ctas_per_sm(uint32_t smem_bytes, int* out) {
    if (cudaFuncSetAttribute(drb_step_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(smem_bytes)) != cudaSuccess)
        return -1;
    return cudaOccupancyMaxActiveBlocksPerMultiprocessor(out, drb_step_kernel, kThreads,
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
    const size_t smem = (size_t(NK) + 1 + 32 + size_t(want + 1) * 4) * 4;
    if (smem > 200 * 1024)
        return -1;
    cudaFuncSetAttribute(plan_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(smem));
    plan_kernel<<<1, 256, smem, static_cast<cudaStream_t>(stream)>>>(
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
