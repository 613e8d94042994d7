#ifndef DRB_RB_H
#define DRB_RB_H

/*
 * drb_rb — C ABI of the B200-native distributed rehearsal buffer (arXiv 2406.03285).
 *
 * This is the drop-in boundary for the reference's hot path. The
 * reference exposes that path only through its C++ API:
 *   rehearsal_buffer(K, cap) / update_buffer / read_slots / snapshot / total_stored /
 *   cross_class_evictions          proj/src/buffer/rehearsal_buffer.hpp:60-95
 *   engine(cfg, rank, ...) / start / update / shutdown / total_wait_ms / drain_timings
 *                                  proj/src/engine/engine.hpp:53-93
 *   plan / augment                 proj/src/sampler/sampler.hpp:33-61
 *   rng_stream                     proj/src/core/rng.hpp:16-51
 * and its own C ABI (proj/include/drb.h) only has run-level entry points. Every function
 * below replaces one of those C++ calls (cited per function) and follows the reference C
 * ABI's conventions: opaque handles, drb_status codes (proj/include/drb.h:33-43), a
 * thread-local drb_last_error() (proj/src/capi/drb_capi.cpp:15,69-71), NULL arguments ->
 * DRB_ERR_INVALID_ARGUMENT, exception taxonomy -> status (drb_capi.cpp:29-46).
 *
 * No torch types: device buffers are plain device pointers, streams are cudaStream_t
 * passed as void* (NULL = the handle's own stream, which is not ordered with the caller's
 * work; pass cudaStreamLegacy for the legacy default stream).
 *
 * Payloads are opaque fixed-size samples of `sample_bytes` bytes (S); labels are uint32.
 * The reference stores float features; any S that is a multiple of 4 is bit-compatible
 * with it (bytes packed into floats).
 */

#include <stddef.h>
#include <stdint.h>

#if defined(_WIN32)
#define DRB_RB_API __declspec(dllexport)
#else
#define DRB_RB_API __attribute__((visibility("default")))
#endif

#ifdef __cplusplus
extern "C" {
#endif

#ifndef DRB_STATUS_DEFINED
#define DRB_STATUS_DEFINED
/* Identical numbering to proj/include/drb.h:33-43. */
typedef enum drb_status {
    DRB_OK = 0,
    DRB_ERR_INVALID_ARGUMENT = 1,
    DRB_ERR_CONFIG = 2,
    DRB_ERR_IO = 3,
    DRB_ERR_TRANSPORT = 4,
    DRB_ERR_PROTOCOL = 5,
    DRB_ERR_TRAINING = 6, /* also engine_error, as drb_capi.cpp:40-41 maps it */
    DRB_ERR_USAGE = 7,
    DRB_ERR_INTERNAL = 8
} drb_status;
#endif

#define DRB_RB_MAX_WORLD 8

/* rng purposes, proj/src/core/rng.hpp:18-26 */
enum {
    DRB_PURPOSE_CANDIDATE_SELECTION = 1,
    DRB_PURPOSE_EVICTION = 2,
    DRB_PURPOSE_GLOBAL_SAMPLING = 3,
    DRB_PURPOSE_DATA_SHUFFLE = 4,
    DRB_PURPOSE_MODEL_INIT = 5,
    DRB_PURPOSE_SLOT_SUBSTITUTE = 6,
    DRB_PURPOSE_SYNTH = 7
};

/* Counter-based stream state: replaces rng_stream (proj/src/core/rng.hpp:16-51).
 * key = derive_key(...), ctr = number of draws consumed so far. Plain data, host side;
 * device kernels consume draws and write the advanced counter back. */
typedef struct drb_rng {
    uint64_t key;
    uint64_t ctr;
} drb_rng;

typedef struct drb_rb drb_rb; /* one rank: HBM slab + occupancy + engine state */

/* drb_rb_config.flags: record per-round timings on the device (drb_rb_drain_timings) */
#define DRB_RB_FLAG_TIMINGS 1u

typedef struct drb_rb_config {
    uint32_t n_classes;       /* K                                   (config.hpp:37) */
    uint32_t per_class_cap;   /* floor(S_max / K)                    (capacity.cpp:10-18) */
    uint64_t sample_bytes;    /* S, multiple of 4                                        */
    uint32_t max_batch;       /* largest |m| ever passed to step/update_buffer (b)       */
    uint32_t candidate_count; /* c                                   (config.hpp:41)     */
    uint32_t rep_count;       /* r                                   (config.hpp:40)     */
    uint32_t rank;            /* worker id                                               */
    uint32_t world;           /* N <= DRB_RB_MAX_WORLD                                   */
    uint64_t seed;            /* rng_seed                            (config.hpp:49)     */
    int32_t device;           /* CUDA device ordinal                                     */
    uint32_t flags;           /* DRB_RB_FLAG_* bits, 0 by default                         */
    uint32_t aug_ring;        /* m' ring depth: m'_i's slot is rewritten by step i+aug_ring;
                                 0 = 32 (the default), else >= 6. A deep ring keeps every m'
                                 of a multi-step run readable (drb_rb_aug_slot)            */
    uint32_t engine_ctas;     /* CTAs (one per SM) of the resident engine while busy; 0 = half
                                 the SMs, leaving the rest to a co-running training step  */
} drb_rb_config;

/* Per-class insertion report of one update, replaces insertion_report
 * (proj/src/buffer/rehearsal_buffer.hpp:17-26). Arrays are caller-owned, K entries. */
typedef struct drb_insertion_report {
    uint32_t* per_class_appends;
    uint32_t* per_class_replacements;
    uint32_t appends;
    uint32_t replacements;
} drb_insertion_report;

/* Read request / status, replaces read_request / read_status (rehearsal_buffer.hpp:28-37). */
typedef struct drb_read_request {
    uint32_t cls;
    uint32_t slot;
} drb_read_request;
enum { DRB_READ_EXACT = 0, DRB_READ_SUBSTITUTED = 1, DRB_READ_EMPTY = 2 };

/* Global slot reference (owner, cls, slot), replaces slot_ref (proj/src/core/types.hpp:26-32). */
typedef struct drb_slot_ref {
    uint32_t owner;
    uint32_t cls;
    uint32_t slot;
} drb_slot_ref;

/* Augmented mini-batch m'_i = m_i ++ reps(i-1), engine-owned device memory.
 * rows [0, n) are m_i, rows [n, count) the representatives in plan order
 * (sampler.cpp:234-240). `count` is valid once the step's work on the stream completes
 * (drb_rb_aug_count). Valid until work enqueued before the next-but-one step call. */
typedef struct drb_aug {
    void* data;            /* count x S bytes, contiguous          */
    uint32_t* labels;      /* count labels                          */
    uint32_t n;            /* |m_i|                                 */
    uint32_t ring_slot;    /* pass to drb_rb_aug_count              */
    uint64_t step;         /* iteration index i                     */
} drb_aug;

/* ---- library ------------------------------------------------------------------------- */
DRB_RB_API const char* drb_rb_version(void);
/* Last error message of the calling thread; never NULL (drb_capi.cpp:69-71). */
DRB_RB_API const char* drb_rb_last_error(void);

/* ---- rng_stream (proj/src/core/rng.cpp:33-53) ------------------------------------------ */
/* rng_stream(seed, worker, purpose)                       rng.cpp:33-34 */
DRB_RB_API drb_status drb_rng_init(drb_rng* s, uint64_t seed, uint32_t worker, uint32_t purpose);
/* rng_stream::keyed(seed, worker, purpose, k1, k2)        rng.cpp:36-39 */
DRB_RB_API drb_status drb_rng_keyed(drb_rng* s, uint64_t seed, uint32_t worker, uint32_t purpose,
                                    uint64_t k1, uint64_t k2);
/* n draws on the GPU: next_u64 (bound == 0) or bounded(bound) (rng.cpp:41-53); out is host
 * memory; s->ctr advances exactly as n sequential calls would. */
DRB_RB_API drb_status drb_rng_draw(drb_rng* s, uint64_t bound, uint64_t n, uint64_t* out,
                                   int32_t device);
/* sample_without_replacement(n, k, rng) on the GPU (rehearsal_buffer.cpp:14-26). out: min(n,k). */
DRB_RB_API drb_status drb_sample_without_replacement(uint32_t n, uint32_t k, drb_rng* s,
                                                     uint32_t* out, uint32_t* out_k,
                                                     int32_t device);
/* plan(want, view, rng) on the GPU (sampler.cpp:65-68). occ: host [n_workers][n_classes].
 * out: host, capacity min(want, total) refs; *out_count = entries written. */
DRB_RB_API drb_status drb_plan(uint32_t want, uint32_t n_workers, uint32_t n_classes,
                               const uint32_t* occ, drb_rng* s, drb_slot_ref* out,
                               uint32_t* out_count, int32_t device);

/* Global-sampling bias test (drb_bias_test, proj/include/drb.h:91-97; the procedure of
 * proj/src/runner/bias.cpp:35-154): every rank of an n_workers mesh freezes its share of
 * `fill` samples (labels i % K, all inserted), rank 0 draws `draws` plans of rep_count from
 * its global-sampling stream of `seed` — on the GPU — and the per-slot hit counts are tested
 * against uniform with Pearson's chi-square (make_bias_report, metrics.cpp:90-107; p-value
 * = Q(df/2, stat/2), stats.cpp:54-96). biased_control != 0 plans over rank 0's own slots only
 * (plan_local_only, sampler.cpp:70-83), the negative control. counts: NULL or `fill`
 * entries (one per slot, flat worker-major order). config_error when fill < n_workers,
 * usage_error when draws == 0 (zero expected count). */
DRB_RB_API drb_status drb_rb_bias_test(uint32_t n_workers, uint32_t n_classes, uint32_t rep_count,
                                       uint64_t seed, uint64_t draws, uint64_t fill, int biased_control,
                                       uint64_t* counts, double* statistic, double* p_value,
                                       int32_t device);

/* ---- rehearsal_buffer (proj/src/buffer/rehearsal_buffer.hpp:60-95) --------------------- */
/* rehearsal_buffer(K, cap) + engine(cfg, rank, ...) storage. config_error on K==0 / cap==0
 * (rehearsal_buffer.cpp:30-31). */
DRB_RB_API drb_status drb_rb_create(const drb_rb_config* cfg, drb_rb** out);
DRB_RB_API drb_status drb_rb_destroy(drb_rb* h);

/* update_buffer(m, c, cand, evict) (rehearsal_buffer.cpp:37-86). batch/labels: DEVICE
 * pointers, n samples. Synchronous. usage_error (DRB_ERR_USAGE) on any label >= K, before
 * any draw. report may be NULL. Not allowed while the engine is started with world > 1. */
DRB_RB_API drb_status drb_rb_update_buffer(drb_rb* h, const void* batch, const uint32_t* labels,
                                           uint32_t n, uint32_t c, drb_rng* cand,
                                           drb_rng* evict, drb_insertion_report* report);
/* read_slots(requests, substitute_rng) (rehearsal_buffer.cpp:88-142). requests/status: host;
 * out/out_labels: DEVICE, count rows of S bytes. Synchronous. */
DRB_RB_API drb_status drb_rb_read_slots(drb_rb* h, const drb_read_request* requests,
                                        uint32_t count, drb_rng* substitute, void* out,
                                        uint32_t* out_labels, uint8_t* status);
/* snapshot() (rehearsal_buffer.cpp:144-152): per_class[K] host, version. */
DRB_RB_API drb_status drb_rb_snapshot(drb_rb* h, uint32_t* per_class, uint64_t* version);
DRB_RB_API drb_status drb_rb_total_stored(drb_rb* h, uint64_t* out);
DRB_RB_API drb_status drb_rb_cross_class_evictions(drb_rb* h, uint64_t* out);
/* Raw device views for zero-copy consumers: slab [K][cap][S], slab labels [K][cap]. */
DRB_RB_API drb_status drb_rb_device_views(drb_rb* h, void** slab, uint32_t** slab_labels);

/* ---- multi-rank wiring (replaces worker_mesh + rpc transport, proj/src/runner/mesh.cpp) -- */
/* Export this rank's peer-shareable region (CUDA IPC handle + metadata) into blob. */
DRB_RB_API drb_status drb_rb_export_handle(drb_rb* h, void* blob, size_t* len);
DRB_RB_API size_t drb_rb_handle_size(void);
/* Map every rank's region; blobs = world blobs of drb_rb_handle_size() bytes in rank order
 * (the caller does the all-gather, e.g. torch.distributed). */
DRB_RB_API drb_status drb_rb_connect(drb_rb* h, const void* blobs, size_t blob_len);

/* ---- engine (proj/src/engine/engine.hpp:53-93) ------------------------------------------ */
DRB_RB_API drb_status drb_rb_start(drb_rb* h);    /* usage_error on double start (engine.cpp:50-52) */
DRB_RB_API drb_status drb_rb_shutdown(drb_rb* h); /* usage_error before start / twice (:203-206) */
/* One iteration: `reps = engine.update(m_i); m' = augment(m_i, reps)` fused
 * (trainer.cpp:109-113). Enqueues on `stream` (device batch/labels): insert candidates of
 * m_i (round i), publish occupancy version i+1, and materialise m'_i = m_i ++ reps(i-1)
 * where reps(i-1) = plan(r, view at version i) read at version i — the exact-horizon
 * semantics of engine.cpp:138-170. out describes m'_i. usage_error before start / after
 * shutdown; engine_error (DRB_ERR_TRAINING) once a previous round failed. */
DRB_RB_API drb_status drb_rb_step(drb_rb* h, const void* batch, const uint32_t* labels,
                                  uint32_t n, void* stream, drb_aug* out);
/* Same, with HOST (ideally pinned) buffers: copies m_i in, runs the step, copies m'_i out
 * into out/out_labels (capacity n + r rows). Asynchronous on the handle's streams;
 * call drb_rb_synchronize before reading out or *out_count.
 * In place (out == batch and out_labels == labels, capacity n + r rows): m_i's rows are
 * already where m'_i keeps them, so only reps(i-1) (rows [n, n+|reps|)) and their labels
 * come back — `augment(m, reps)` (sampler.cpp:234-240) without the host-side copy of m. */
/* drb_rb_step with the producer / consumer split of the reference's asynchronous engine
 * (engine.cpp:62-106: the loader hands m_i over, the trainer consumes m'_i): m_i is posted in
 * `producer`'s order (after the work that produced it), and `consumer` first releases every
 * m' it was handed before this call (everything already enqueued on it has used them), then
 * waits for m'_i. Steps posted back to back on the producer run pipelined in the engine;
 * the engine refills an m' ring slot only after its consumer released it. */
DRB_RB_API drb_status drb_rb_step_split(drb_rb* h, const void* batch, const uint32_t* labels, uint32_t n,
                                        void* producer, void* consumer, drb_aug* out);
DRB_RB_API drb_status drb_rb_step_host(drb_rb* h, const void* batch, const uint32_t* labels,
                                       uint32_t n, void* out, uint32_t* out_labels,
                                       uint32_t* out_count);
/* `steps` consecutive iterations over a device-resident ring of `ring` input batches
 * (batch j at batches + j*batch_stride bytes, labels + j*label_stride elements), issued
 * back to back from native code on `stream`. The throughput-harness analogue of
 * drb_overlap_bench (proj/include/drb.h:107-114, proj/src/runner/overlap.cpp:83-89, zero
 * train cost). If step_events is non-NULL it must hold 2*steps cudaEvent_t created by the
 * caller; iteration i's copy kernel (the dominant one) is bracketed by events 2i and 2i+1,
 * recorded after its dependencies resolved (per-launch device timing). */
DRB_RB_API drb_status drb_rb_run(drb_rb* h, const void* batches, uint64_t batch_stride,
                                 const uint32_t* labels, uint64_t label_stride, uint32_t ring,
                                 uint32_t n, uint64_t steps, uint64_t first, void* stream,
                                 void* const* step_events);
/* The same `steps` iterations captured into a CUDA graph without running them (host
 * launch cost paid here, once). The handle's iteration state advances as if the steps had
 * been enqueued: launch the graph exactly once with drb_rb_graph_launch, before any
 * further step on this handle. */
typedef struct drb_rb_graph drb_rb_graph;
DRB_RB_API drb_status drb_rb_graph_prepare(drb_rb* h, const void* batches, uint64_t batch_stride,
                                           const uint32_t* labels, uint64_t label_stride,
                                           uint32_t ring, uint32_t n, uint64_t steps,
                                           uint64_t first, void* const* step_events,
                                           drb_rb_graph** out);
DRB_RB_API drb_status drb_rb_graph_launch(drb_rb_graph* g, void* stream);
DRB_RB_API drb_status drb_rb_graph_destroy(drb_rb_graph* g);
/* Rows of m' for a completed step (blocks on that step's completion). */
/* Per-round timings, replaces engine::timings / drain_timings() (proj/src/engine/engine.hpp:43-50,
 * :93; recorded at engine.cpp:139-168). Device timestamps of the resident engine (config flag
 * DRB_RB_FLAG_TIMINGS; the three-kernel path records none):
 *   populate_ms  sel(i): update_buffer + publish_row           (engine.cpp:141-144)
 *   augment_ms   plan(i) start -> round i's pushes complete   (view_at + plan + fetch, :146-163)
 *   latency_ms   round i admitted -> its pushes complete      (enqueue -> promise, :139,168)
 *   wait_ms      0: no engine thread blocks (the consumer's stream waits on the device)
 *   degraded     0: a stalled peer fails the engine instead */
typedef struct drb_timing {
    uint64_t iteration;
    double populate_ms;
    double augment_ms;
    double latency_ms;
    double wait_ms;
    uint32_t degraded;
    uint32_t pad;
} drb_timing;
/* Moves the timings of the rounds completed since the last drain (at most the last 4096) into
 * out[0..capacity); *count = records written. Waits for the engine's posted work first. */
DRB_RB_API drb_status drb_rb_drain_timings(drb_rb* h, drb_timing* out, uint32_t capacity, uint32_t* count);

/* m'_step still held by the engine's ring (one of the last aug_ring enqueued steps), for a
 * step whose batch had n rows: the same views drb_rb_step returned for it. With a deep ring
 * (drb_rb_config.aug_ring >= steps) every m' of a drb_rb_run stays readable after the run
 * (step-by-step parity of the benchmarked path). Engine-internal; no reference counterpart. */
/* Resident-engine bookkeeping (no reference counterpart): whether the engine runs as a
 * resident kernel, how many instances have been launched so far (one per busy period; a
 * step itself launches nothing), descriptors posted, CTAs per instance. */
DRB_RB_API drb_status drb_rb_engine_info(drb_rb* h, uint32_t* resident, uint64_t* instances,
                                         uint64_t* posted, uint32_t* grid);
DRB_RB_API drb_status drb_rb_aug_slot(drb_rb* h, uint64_t step, uint32_t n, drb_aug* out);
DRB_RB_API drb_status drb_rb_aug_count(drb_rb* h, const drb_aug* aug, uint32_t* count);
DRB_RB_API drb_status drb_rb_synchronize(drb_rb* h);
/* total_wait_ms (engine.hpp:88): host time blocked waiting for round results. */
DRB_RB_API drb_status drb_rb_total_wait_ms(drb_rb* h, double* out);
/* engine::iterations / queue_depth / degraded_rounds / replanned_entries (engine.hpp:87-92), any
 * pointer may be NULL. iterations = steps enqueued; queue_depth = enqueued steps whose m' is not
 * ready yet (the reference holds at most one queued job; here several rounds may be in flight);
 * degraded_rounds and replanned_entries are always 0: a stalled peer fails the engine
 * (DRB_ERR_TRANSPORT) instead of degrading to stale rows. */
DRB_RB_API drb_status drb_rb_engine_counters(drb_rb* h, uint64_t* iterations, uint64_t* queue_depth,
                                             uint64_t* degraded_rounds, uint64_t* replanned_entries);
/* engine::broadcast_sizes (engine.hpp:82, engine.cpp:256-265): re-publish the freshest occupancy
 * row at a task boundary. A no-op here: every round already stores the row into every peer's
 * table. */
DRB_RB_API drb_status drb_rb_broadcast_sizes(drb_rb* h);
/* Device-side error word of the last completed step (0 = none). */
DRB_RB_API drb_status drb_rb_device_error(drb_rb* h, uint32_t* out);
/* Diagnostics (DRB_TRACE=1 at create): globaltimer stamps of the last step's phases in
 * CTA 0 (slots 0-9), CTA 1 (slots 16-25) and the grid-wide first start / last end
 * (slots 14, 15). out must hold 32 values. */
DRB_RB_API drb_status drb_rb_trace_read(drb_rb* h, uint64_t* out32);
/* Diagnostics (DRB_TIMELINE=<steps> at create): per step s (ring of `steps`), per kernel
 * kind (0 sel, 1 plan, 2 copy) the grid-wide [first start, last end] globaltimer stamps at
 * out[(s*3 + kind)*2 + {0,1}]. out = NULL queries *steps only. */
DRB_RB_API drb_status drb_rb_timeline_read(drb_rb* h, uint64_t* out, uint32_t* steps);
/* Launch configuration of the step kernel: grid CTAs, threads, dynamic smem. */
DRB_RB_API drb_status drb_rb_launch_info(drb_rb* h, uint32_t* grid, uint32_t* threads,
                                         uint32_t* smem);

/* ---- Input side: the producer of m ----------------------------
 * A DRDS dataset file (proj/src/scenario/dataset.hpp:10-17: "DRDS", u16 version 1,
 * u64 count, u32 feature_dim, u32 n_classes, count x {feature_dim f32, u32 label}, all LE;
 * optional "<path>.split" sidecar) resident in HBM as SoA features [count][feature_dim*4 B]
 * + u32 labels[count]. Sample bytes S = feature_dim*4 match a rehearsal buffer whose
 * sample_bytes is S, so drb_ds_gather output feeds drb_rb_step / drb_rb_run directly. */
typedef struct drb_ds drb_ds;
/* load_dataset (proj/src/scenario/dataset.cpp:102-143): same checks, same order, same
 * messages; every failure is DRB_ERR_IO (io_error). */
DRB_RB_API drb_status drb_ds_load(const char* path, int32_t device, drb_ds** out);
/* synth_dataset (proj/src/scenario/dataset.cpp:145-205): the reference's Gaussian-blob
 * dataset, bit-identical (same stream, same double arithmetic), placed in HBM.
 * separation <= 0 -> DRB_ERR_CONFIG. */
DRB_RB_API drb_status drb_ds_synth(uint32_t n_classes, uint32_t per_class, uint32_t feature_dim,
                                   double separation, uint64_t seed, int32_t device, drb_ds** out);
DRB_RB_API drb_status drb_ds_destroy(drb_ds* ds);
/* dataset::size / feature_dim / n_classes / train_count / eval_count (dataset.hpp:19-27). */
DRB_RB_API drb_status drb_ds_info(const drb_ds* ds, uint64_t* count, uint32_t* feature_dim,
                                  uint32_t* n_classes, uint64_t* train_count,
                                  uint64_t* eval_count);
DRB_RB_API drb_status drb_ds_device_views(const drb_ds* ds, void** features, uint32_t** labels);
/* train_indices_of (eval = 0) / eval_indices_of (eval = 1) (dataset.cpp:48-64): ascending
 * dataset indices whose label is in classes[0..n_classes). *n_out = the full count; at most
 * cap are written (out = NULL, cap = 0 queries the count). */
DRB_RB_API drb_status drb_ds_indices_of(const drb_ds* ds, const uint32_t* classes,
                                        uint32_t n_classes, int32_t eval, uint64_t* out,
                                        uint64_t cap, uint64_t* n_out);
/* dataset::gather (dataset.cpp:66-72) on the device, ordered on `stream`: out_batch row j
 * (S bytes) and out_labels[j] (may be NULL) = record indices[j]. indices is a DEVICE array
 * of n u64. An index >= count leaves row j untouched and sets bit 0 of the device error
 * word (drb_ds_device_error). */
DRB_RB_API drb_status drb_ds_gather(const drb_ds* ds, const uint64_t* indices, uint32_t n,
                                    void* out_batch, uint32_t* out_labels, void* stream);
/* Synchronizes the device, returns and clears the gather error word. */
DRB_RB_API drb_status drb_ds_device_error(const drb_ds* ds, uint32_t* out);
/* make_schedule (proj/src/scenario/schedule.cpp:10-35): classes[K] = the seeded class
 * permutation, task t = the next task_sizes[t] entries. T == 0 or T > K -> DRB_ERR_CONFIG. */
DRB_RB_API drb_status drb_make_schedule(uint32_t n_classes, uint32_t n_tasks, uint64_t seed,
                                        uint32_t* classes, uint32_t* task_sizes);
/* shard_batches (schedule.cpp:37-62), flattened: this worker's shard in order; batch b is
 * entries [b*batch_size, (b+1)*batch_size). *n_out = shard size; at most cap written.
 * worker >= n_workers -> DRB_ERR_USAGE (usage_error); batch_size 0 -> DRB_ERR_USAGE. */
DRB_RB_API drb_status drb_shard_batches(const uint64_t* task_data, uint64_t n, uint32_t worker,
                                        uint32_t n_workers, uint32_t batch_size, uint64_t seed,
                                        uint64_t task_index, uint64_t epoch, uint64_t* out,
                                        uint64_t cap, uint64_t* n_out);
/* lockstep_batches (schedule.cpp:64-69). */
DRB_RB_API drb_status drb_lockstep_batches(uint64_t task_size, uint32_t n_workers,
                                           uint32_t batch_size, uint64_t* out);

#ifdef __cplusplus
} /* extern "C" */
#endif

#endif /* DRB_RB_H */
