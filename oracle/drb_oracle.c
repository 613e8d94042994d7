/*
 * drb_oracle.c — TEST INFRASTRUCTURE (see drb_oracle.h). Clean-room restatement of
 * SURVEY.md Appendix A, S0–S6; every function cites the reference lines it follows.
 * Deliberately simple and sequential: it is the checker, never the thing measured.
 */
#include "drb_oracle.h"

#include <stdlib.h>
#include <string.h>

#define PHI 0x9e3779b97f4a7c15ULL

/* proj/src/core/rng.cpp:12-17 */
uint64_t or_mix64(uint64_t z) {
    z += PHI;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

/* proj/src/core/rng.cpp:19-27 (derive_key), :33-39 (ctor / keyed adds +1 to k1,k2) */
or_stream or_stream_make(uint64_t seed, uint32_t worker, uint32_t purpose, int keyed,
                         uint64_t k1, uint64_t k2) {
    if (keyed) {
        k1 += 1;
        k2 += 1;
    } else {
        k1 = 0;
        k2 = 0;
    }
    uint64_t key = or_mix64(seed);
    key = or_mix64(key ^ ((uint64_t)worker * 0xd1342543de82ef95ULL));
    key = or_mix64(key ^ ((uint64_t)purpose * 0xaf251af3b0f025b5ULL));
    key = or_mix64(key ^ k1);
    key = or_mix64(key ^ k2);
    or_stream s = {key, 0};
    return s;
}

/* proj/src/core/rng.cpp:41-43 */
uint64_t or_next_u64(or_stream* s) {
    s->ctr += 1;
    return or_mix64(s->key ^ (s->ctr * PHI));
}

/* proj/src/core/rng.cpp:45-53 */
uint64_t or_bounded(or_stream* s, uint64_t n) {
    const uint64_t thr = (0 - n) % n;
    for (;;) {
        const uint64_t v = or_next_u64(s);
        if (v >= thr)
            return v % n;
    }
}

int or_rng_next(uint64_t seed, uint32_t worker, uint32_t purpose, int keyed, uint64_t k1,
                uint64_t k2, uint64_t n, uint64_t* out) {
    or_stream s = or_stream_make(seed, worker, purpose, keyed, k1, k2);
    for (uint64_t i = 0; i < n; ++i)
        out[i] = or_next_u64(&s);
    return 0;
}

int or_rng_bounded(uint64_t seed, uint32_t worker, uint32_t purpose, int keyed, uint64_t k1,
                   uint64_t k2, uint64_t bound, uint64_t n, uint64_t* out) {
    or_stream s = or_stream_make(seed, worker, purpose, keyed, k1, k2);
    for (uint64_t i = 0; i < n; ++i)
        out[i] = or_bounded(&s, bound);
    return 0;
}

/* S1 — proj/src/buffer/rehearsal_buffer.cpp:14-26: k=min(k,n); iota; for j<k swap(j, j+bounded(n-j)). */
static uint64_t swor_stream(uint64_t n, uint64_t k, or_stream* s, uint64_t* out) {
    if (k > n)
        k = n;
    uint64_t* idx = (uint64_t*)malloc((n ? n : 1) * sizeof(uint64_t));
    for (uint64_t i = 0; i < n; ++i)
        idx[i] = i;
    for (uint64_t j = 0; j < k; ++j) {
        const uint64_t w = j + or_bounded(s, n - j);
        const uint64_t t = idx[j];
        idx[j] = idx[w];
        idx[w] = t;
    }
    memcpy(out, idx, k * sizeof(uint64_t));
    free(idx);
    return k;
}

int or_swor(uint64_t n, uint64_t k, uint64_t seed, uint32_t worker, uint32_t purpose,
            uint64_t* out, uint64_t* out_k) {
    or_stream s = or_stream_make(seed, worker, purpose, 0, 0, 0);
    *out_k = swor_stream(n, k, &s, out);
    return 0;
}

/* S3 locate — proj/src/sampler/size_table.cpp:29-39: worker-major, then class, then slot. */
static void locate(uint64_t flat, uint32_t N, uint32_t K, const uint32_t* occ, uint32_t* ref) {
    for (uint32_t w = 0; w < N; ++w)
        for (uint32_t k = 0; k < K; ++k) {
            const uint64_t o = occ[(size_t)w * K + k];
            if (flat < o) {
                ref[0] = w;
                ref[1] = k;
                ref[2] = (uint32_t)flat;
                return;
            }
            flat -= o;
        }
    ref[0] = ref[1] = ref[2] = 0xffffffffu; /* unreachable for flat < total */
}

/* S4 — proj/src/sampler/sampler.cpp:39-61 (plan_over_flat) via :65-68 (plan). */
static uint32_t plan_stream(uint64_t want, uint32_t N, uint32_t K, const uint32_t* occ,
                            or_stream* s, uint32_t* out) {
    uint64_t total = 0;
    for (size_t i = 0; i < (size_t)N * K; ++i)
        total += occ[i];
    if (total == 0 || want == 0)
        return 0;
    if (want >= total) { /* exhaustion: every slot in flat order, no draws */
        for (uint64_t f = 0; f < total; ++f)
            locate(f, N, K, occ, out + 3 * f);
        return (uint32_t)total;
    }
    uint64_t* chosen = (uint64_t*)malloc(want * sizeof(uint64_t));
    uint32_t got = 0;
    while (got < want) {
        const uint64_t f = or_bounded(s, total);
        int seen = 0;
        for (uint32_t i = 0; i < got; ++i)
            if (chosen[i] == f) {
                seen = 1;
                break;
            }
        if (!seen) {
            chosen[got] = f;
            locate(f, N, K, occ, out + 3 * got);
            ++got;
        }
    }
    free(chosen);
    return got;
}

int or_plan(uint64_t want, uint32_t n_workers, uint32_t n_classes, const uint32_t* occ,
            uint64_t seed, uint32_t worker, uint32_t purpose, uint32_t rounds, uint32_t* out,
            uint64_t* out_counts) {
    or_stream s = or_stream_make(seed, worker, purpose, 0, 0, 0);
    size_t pos = 0;
    for (uint32_t rd = 0; rd < rounds; ++rd) {
        const uint32_t got = plan_stream(want, n_workers, n_classes, occ, &s, out + pos);
        out_counts[rd] = got;
        pos += 3 * (size_t)got;
    }
    return 0;
}

/* S1+S2 — proj/src/buffer/rehearsal_buffer.cpp:37-86. */
int or_update_buffer(uint8_t* slab, uint32_t* slab_labels, uint32_t* occ, uint64_t* version,
                     uint32_t K, uint32_t cap, uint64_t S, const uint8_t* batch,
                     const uint32_t* labels, uint32_t n, uint32_t c, or_stream* cand,
                     or_stream* evict, uint32_t* report_appends, uint32_t* report_repl) {
    if (report_appends)
        memset(report_appends, 0, K * sizeof(uint32_t));
    if (report_repl)
        memset(report_repl, 0, K * sizeof(uint32_t));
    if (n == 0) /* :42-43 empty batch: no draws */
        return 0;
    for (uint32_t i = 0; i < n; ++i) /* :44-47 label check before any draw */
        if (labels[i] >= K)
            return 7;
    uint64_t* chosen = (uint64_t*)malloc(n * sizeof(uint64_t));
    const uint64_t k = swor_stream(n, c, cand, chosen);
    for (uint64_t t = 0; t < k; ++t) { /* selection order */
        const uint32_t L = labels[chosen[t]];
        uint32_t slot;
        if (occ[L] < cap) { /* append :61-70 */
            slot = occ[L]++;
            if (report_appends)
                report_appends[L]++;
        } else { /* uniform replacement :71-78, n = occupancy == cap */
            slot = (uint32_t)or_bounded(evict, occ[L]);
            if (report_repl)
                report_repl[L]++;
        }
        memcpy(slab + ((size_t)L * cap + slot) * S, batch + chosen[t] * S, S);
        slab_labels[(size_t)L * cap + slot] = L;
        *version += 1; /* :79 */
    }
    free(chosen);
    return 0;
}

/* read_slots (rehearsal_buffer.cpp:88-142) */
int or_read_slots(const uint8_t* slab, const uint32_t* slab_labels, const uint32_t* occ, uint32_t K,
                  uint32_t cap, uint64_t S, const uint32_t* req, uint32_t count, or_stream* sub,
                  uint8_t* out, uint32_t* out_labels, uint8_t* status) {
    uint64_t total = 0; /* m_total (rehearsal_buffer.hpp:89) = sum of occupancies */
    for (uint32_t c = 0; c < K; ++c)
        total += occ[c];
    for (uint32_t i = 0; i < count; ++i) {
        const uint32_t cls = req[2 * i], slot = req[2 * i + 1];
        int64_t row = -1;
        uint8_t st = 2;
        if (cls < K && occ[cls] > 0) { /* :96-103 */
            if (slot < occ[cls]) {
                st = 0;
                row = (int64_t)cls * cap + slot;
            } else {
                st = 1;
                row = (int64_t)cls * cap + (int64_t)or_bounded(sub, occ[cls]);
            }
        }
        if (st == 2 && total > 0) { /* :106-121 flat fallback over the whole buffer */
            uint64_t flat = or_bounded(sub, total);
            for (uint32_t c = 0; c < K; ++c) {
                if (flat < occ[c]) {
                    st = 1;
                    row = (int64_t)c * cap + (int64_t)flat;
                    break;
                }
                flat -= occ[c];
            }
        }
        status[i] = st;
        if (row >= 0) {
            memcpy(out + (size_t)i * S, slab + (size_t)row * S, S);
            out_labels[i] = slab_labels[row];
        } else {
            memset(out + (size_t)i * S, 0, S);
            out_labels[i] = 0;
        }
    }
    return 0;
}

/* ---- S5 synchronous replay --------------------------------------------------------- */

typedef struct replay {
    uint32_t N, K, cap, c, r;
    uint64_t S;
    uint8_t** slab;
    uint32_t** slab_labels;
    uint32_t* occ;      /* N x K */
    uint64_t* version;  /* N */
    or_stream *cand, *evict, *samp;
    uint8_t* pending;   /* N x r x S : reps(i-1) bytes */
    uint32_t* pending_labels;
    uint32_t* pending_count;
    uint32_t* plan;     /* N x r x 3 */
    uint32_t* plan_count;
    uint32_t* rep_app;  /* N x K */
    uint32_t* rep_rep;  /* N x K */
    uint64_t step;
} replay;

void* or_replay_create(uint32_t N, uint32_t K, uint32_t cap, uint64_t S, uint32_t c, uint32_t r,
                       uint64_t seed) {
    replay* h = (replay*)calloc(1, sizeof(replay));
    h->N = N; h->K = K; h->cap = cap; h->S = S; h->c = c; h->r = r;
    h->slab = (uint8_t**)calloc(N, sizeof(uint8_t*));
    h->slab_labels = (uint32_t**)calloc(N, sizeof(uint32_t*));
    for (uint32_t w = 0; w < N; ++w) {
        h->slab[w] = (uint8_t*)calloc((size_t)K * cap, S);
        h->slab_labels[w] = (uint32_t*)calloc((size_t)K * cap, 4);
    }
    h->occ = (uint32_t*)calloc((size_t)N * K, 4);
    h->version = (uint64_t*)calloc(N, 8);
    h->cand = (or_stream*)calloc(N, sizeof(or_stream));
    h->evict = (or_stream*)calloc(N, sizeof(or_stream));
    h->samp = (or_stream*)calloc(N, sizeof(or_stream));
    for (uint32_t w = 0; w < N; ++w) { /* proj/src/engine/engine.cpp:27-35 */
        h->cand[w] = or_stream_make(seed, w, 1, 0, 0, 0);
        h->evict[w] = or_stream_make(seed, w, 2, 0, 0, 0);
        h->samp[w] = or_stream_make(seed, w, 3, 0, 0, 0);
    }
    h->pending = (uint8_t*)calloc((size_t)N * (r ? r : 1), S);
    h->pending_labels = (uint32_t*)calloc((size_t)N * (r ? r : 1), 4);
    h->pending_count = (uint32_t*)calloc(N, 4);
    h->plan = (uint32_t*)calloc((size_t)N * (r ? r : 1) * 3, 4);
    h->plan_count = (uint32_t*)calloc(N, 4);
    h->rep_app = (uint32_t*)calloc((size_t)N * K, 4);
    h->rep_rep = (uint32_t*)calloc((size_t)N * K, 4);
    return h;
}

void or_replay_destroy(void* p) {
    replay* h = (replay*)p;
    if (!h)
        return;
    for (uint32_t w = 0; w < h->N; ++w) {
        free(h->slab[w]);
        free(h->slab_labels[w]);
    }
    free(h->slab); free(h->slab_labels); free(h->occ); free(h->version);
    free(h->cand); free(h->evict); free(h->samp);
    free(h->pending); free(h->pending_labels); free(h->pending_count);
    free(h->plan); free(h->plan_count); free(h->rep_app); free(h->rep_rep);
    free(h);
}

int or_replay_step(void* p, const uint8_t* batches, const uint32_t* labels, uint32_t n,
                   uint8_t* out, uint32_t* out_labels, uint32_t* out_counts) {
    replay* h = (replay*)p;
    const uint64_t S = h->S;
    const uint32_t N = h->N, K = h->K, r = h->r;
    /* round i: every rank inserts its candidates (engine.cpp:138-146) */
    for (uint32_t w = 0; w < N; ++w) {
        const int rc = or_update_buffer(h->slab[w], h->slab_labels[w], h->occ + (size_t)w * K,
                                        &h->version[w], K, h->cap, S,
                                        batches + (size_t)w * n * S, labels + (size_t)w * n, n,
                                        h->c, &h->cand[w], &h->evict[w],
                                        h->rep_app + (size_t)w * K, h->rep_rep + (size_t)w * K);
        if (rc)
            return rc;
    }
    /* m'_i = m_i ++ reps(i-1) (sampler.cpp:234-240; engine timeline engine.cpp:62-106) */
    for (uint32_t w = 0; w < N; ++w) {
        uint8_t* o = out + (size_t)w * (n + r) * S;
        uint32_t* ol = out_labels + (size_t)w * (n + r);
        memcpy(o, batches + (size_t)w * n * S, (size_t)n * S);
        memcpy(ol, labels + (size_t)w * n, (size_t)n * 4);
        const uint32_t cnt = h->pending_count[w];
        memcpy(o + (size_t)n * S, h->pending + (size_t)w * r * S, (size_t)cnt * S);
        memcpy(ol + n, h->pending_labels + (size_t)w * r, (size_t)cnt * 4);
        out_counts[w] = n + cnt;
    }
    /* plan(i) on the view at version i+1 = all ranks' occ now; exact reads now (S3-S5) */
    for (uint32_t w = 0; w < N; ++w) {
        uint32_t* pl = h->plan + (size_t)w * r * 3;
        const uint32_t got = plan_stream(r, N, K, h->occ, &h->samp[w], pl);
        h->plan_count[w] = got;
        for (uint32_t j = 0; j < got; ++j) {
            const uint32_t o = pl[3 * j], k = pl[3 * j + 1], s = pl[3 * j + 2];
            memcpy(h->pending + ((size_t)w * r + j) * S, h->slab[o] + ((size_t)k * h->cap + s) * S, S);
            h->pending_labels[(size_t)w * r + j] = h->slab_labels[o][(size_t)k * h->cap + s];
        }
        h->pending_count[w] = got;
    }
    h->step++;
    return 0;
}

uint32_t or_replay_last_plan(void* p, uint32_t w, uint32_t* out) {
    replay* h = (replay*)p;
    memcpy(out, h->plan + (size_t)w * h->r * 3, (size_t)h->plan_count[w] * 3 * 4);
    return h->plan_count[w];
}

int or_replay_last_report(void* p, uint32_t w, uint32_t* appends, uint32_t* replacements,
                          uint32_t* totals) {
    replay* h = (replay*)p;
    memcpy(appends, h->rep_app + (size_t)w * h->K, h->K * 4);
    memcpy(replacements, h->rep_rep + (size_t)w * h->K, h->K * 4);
    totals[0] = totals[1] = 0;
    for (uint32_t k = 0; k < h->K; ++k) {
        totals[0] += appends[k];
        totals[1] += replacements[k];
    }
    return 0;
}

int or_replay_dump(void* p, uint32_t w, uint32_t* occ, uint64_t* version, uint8_t* slab,
                   uint32_t* slab_labels) {
    replay* h = (replay*)p;
    memcpy(occ, h->occ + (size_t)w * h->K, h->K * 4);
    *version = h->version[w];
    if (!slab || !slab_labels)  /* occupancy and version only */
        return 0;
    for (uint32_t k = 0; k < h->K; ++k)
        for (uint32_t s = 0; s < h->cap; ++s) {
            const size_t i = (size_t)k * h->cap + s;
            if (s < occ[k]) {
                memcpy(slab + i * h->S, h->slab[w] + i * h->S, h->S);
                slab_labels[i] = h->slab_labels[w][i];
            } else {
                memset(slab + i * h->S, 0, h->S);
                slab_labels[i] = 0;
            }
        }
    return 0;
}

int or_replay_counters(void* p, uint32_t w, uint64_t* out3) {
    replay* h = (replay*)p;
    out3[0] = h->cand[w].ctr;
    out3[1] = h->evict[w].ctr;
    out3[2] = h->samp[w].ctr;
    return 0;
}
