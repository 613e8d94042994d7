/*
 * drb_oracle — TEST INFRASTRUCTURE, not product code.
 *
 * A clean-room CPU restatement (plain C11) of the reference's rehearsal-buffer hot
 * path, semantics S0–S6 of SURVEY.md Appendix A. Used only by tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg, and only as the checker.
 *
 * Parity is PINNED: tests/test_oracle.py checks this restatement against
 *   (1) the golden vectors in tests/golden/ generated from the reference itself
 *       (oracle/gen_golden.py driving oracle/_ref/libdrb_ref.so), and
 *   (2) the reference library directly on randomised configs when oracle/_ref is built.
 */
#ifndef DRB_ORACLE_H
#define DRB_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* S0: counter-based splitmix64 stream (proj/src/core/rng.cpp:12-53). */
typedef struct or_stream {
    uint64_t key;
    uint64_t ctr;
} or_stream;

uint64_t or_mix64(uint64_t z);
or_stream or_stream_make(uint64_t seed, uint32_t worker, uint32_t purpose, int keyed,
                         uint64_t k1, uint64_t k2);
uint64_t or_next_u64(or_stream* s);
uint64_t or_bounded(or_stream* s, uint64_t n);

int or_rng_next(uint64_t seed, uint32_t worker, uint32_t purpose, int keyed, uint64_t k1,
                uint64_t k2, uint64_t n, uint64_t* out);
int or_rng_bounded(uint64_t seed, uint32_t worker, uint32_t purpose, int keyed, uint64_t k1,
                   uint64_t k2, uint64_t bound, uint64_t n, uint64_t* out);

/* S1: partial Fisher–Yates (proj/src/buffer/rehearsal_buffer.cpp:14-26). */
int or_swor(uint64_t n, uint64_t k, uint64_t seed, uint32_t worker, uint32_t purpose,
            uint64_t* out, uint64_t* out_k);

/* S3+S4: plan over a view occ[n_workers][n_classes] (sampler.cpp:39-68, size_table.cpp:29-39). */
int or_plan(uint64_t want, uint32_t n_workers, uint32_t n_classes, const uint32_t* occ,
            uint64_t seed, uint32_t worker, uint32_t purpose, uint32_t rounds, uint32_t* out,
            uint64_t* out_counts);

/* S1+S2 on one rank's byte slab (rehearsal_buffer.cpp:37-86). Returns 0, or 7 on a
 * label >= K (before any draw). report_*: per-class appends / replacements (K each). */
int or_update_buffer(uint8_t* slab, uint32_t* slab_labels, uint32_t* occ, uint64_t* version,
                     uint32_t K, uint32_t cap, uint64_t S, const uint8_t* batch,
                     const uint32_t* labels, uint32_t n, uint32_t c, or_stream* cand,
                     or_stream* evict, uint32_t* report_appends, uint32_t* report_repl);

/* read_slots on one rank's slab (rehearsal_buffer.cpp:88-142): req = (cls, slot) pairs.
 * Exact read if slot < occ[cls]; a stale index draws a substitute slot of the class
 * (sub.bounded(occ)); an empty (or out-of-range) class falls back to a uniform draw over every
 * stored slot (sub.bounded(total), class-major flat order); nothing stored -> empty (zero
 * bytes, label 0, as serve_sample sends it, engine.cpp:239-244). status: 0 exact,
 * 1 substituted, 2 empty. (The reference's retry after a concurrent append cannot occur in a
 * single-threaded replay.) */
int or_read_slots(const uint8_t* slab, const uint32_t* slab_labels, const uint32_t* occ, uint32_t K,
                  uint32_t cap, uint64_t S, const uint32_t* req, uint32_t count, or_stream* sub,
                  uint8_t* out, uint32_t* out_labels, uint8_t* status);

/* Synchronous multi-rank replay (S5): the bit-exact oracle of SURVEY.md §8c.
 * Same signatures as oracle/ref_capi.cpp's ref_replay_*. */
void* or_replay_create(uint32_t N, uint32_t K, uint32_t cap, uint64_t S, uint32_t c, uint32_t r,
                       uint64_t seed);
void or_replay_destroy(void* h);
int or_replay_step(void* h, const uint8_t* batches, const uint32_t* labels, uint32_t n,
                   uint8_t* out, uint32_t* out_labels, uint32_t* out_counts);
uint32_t or_replay_last_plan(void* h, uint32_t w, uint32_t* out);
int or_replay_last_report(void* h, uint32_t w, uint32_t* appends, uint32_t* replacements,
                          uint32_t* totals);
int or_replay_dump(void* h, uint32_t w, uint32_t* occ, uint64_t* version, uint8_t* slab,
                   uint32_t* slab_labels);
/* Stream counters of rank w after the last step: cand, evict, samp. */
int or_replay_counters(void* h, uint32_t w, uint64_t* out3);

#ifdef __cplusplus
}
#endif
#endif
