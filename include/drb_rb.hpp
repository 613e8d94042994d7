// drb_rb.hpp — header-only C++ facade over the C ABI (drb_rb.h), mirroring the reference's
// hot-path C++ API so call sites port one-to-one:
//
//   reference (proj/src/...)                          this facade (namespace drb::b200)
//   rng_stream(seed, worker, purpose)  core/rng.hpp   rng_stream(seed, worker, purpose)
//   rng_stream::keyed(...)                            rng_stream::keyed(...)
//   sample_without_replacement(n, k, rng)             sample_without_replacement(n, k, rng)
//   rehearsal_buffer(K, cap)   buffer/rehearsal_buffer.hpp:62
//                                                     rehearsal_buffer(config)  (S, max batch,
//                                                     c, r, rank, world, device fixed at creation)
//   update_buffer(m, c, cand, evict)                  update_buffer(device_batch, c, cand, evict)
//   read_slots(requests, substitute_rng)              read_slots(requests, substitute_rng, out...)
//   snapshot() / total_stored() / cross_class_evictions()   same
//   plan(want, view, rng)      sampler/sampler.hpp:33 plan(want, view, rng)
//   engine(cfg, rank, buffer, table, client)  engine/engine.hpp:53
//                                                     engine(rehearsal_buffer&)
//   engine::start / update / shutdown / total_wait_ms        same; update() returns the fused
//                                                     augmented batch m'_i = m_i ++ reps(i-1)
//   augment(m, reps)           sampler/sampler.hpp:61 augmented_batch (already m ++ reps)
//
// Errors are thrown as the reference's exception taxonomy (proj/src/core/errors.hpp):
// config_error, usage_error, transport_error, engine_error; anything else drb_error.
// Device memory is plain device pointers: the caller owns batches, the engine owns m'.
#pragma once

#include <algorithm>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "drb_rb.h"

namespace drb::b200 {

struct drb_error : std::runtime_error {
    drb_status status;
    drb_error(drb_status s, const std::string& w) : std::runtime_error(w), status(s) {}
};
struct config_error : drb_error {
    using drb_error::drb_error;
};
struct usage_error : drb_error {
    using drb_error::drb_error;
};
struct transport_error : drb_error {
    using drb_error::drb_error;
};
struct engine_error : drb_error {
    using drb_error::drb_error;
};
struct io_error : drb_error {
    using drb_error::drb_error;
};

inline void check(drb_status s) {
    if (s == DRB_OK)
        return;
    const std::string msg = drb_rb_last_error();
    switch (s) {
    case DRB_ERR_CONFIG: throw config_error(s, msg);
    case DRB_ERR_USAGE: throw usage_error(s, msg);
    case DRB_ERR_TRANSPORT: throw transport_error(s, msg);
    case DRB_ERR_TRAINING: throw engine_error(s, msg);
    case DRB_ERR_IO: throw io_error(s, msg);
    default: throw drb_error(s, msg);
    }
}

class rng_stream {
public:
    enum class purpose : std::uint32_t {
        candidate_selection = 1,
        eviction = 2,
        global_sampling = 3,
        data_shuffle = 4,
        model_init = 5,
        slot_substitute = 6,
        synth = 7,
    };
    rng_stream(std::uint64_t seed, std::uint32_t worker, purpose p, int device = 0) : device_(device) {
        check(drb_rng_init(&s_, seed, worker, static_cast<std::uint32_t>(p)));
    }
    static rng_stream keyed(std::uint64_t seed, std::uint32_t worker, purpose p, std::uint64_t k1,
                            std::uint64_t k2 = 0, int device = 0) {
        rng_stream r(seed, worker, p, device);
        check(drb_rng_keyed(&r.s_, seed, worker, static_cast<std::uint32_t>(p), k1, k2));
        return r;
    }
    std::uint64_t next_u64() {
        std::uint64_t v = 0;
        check(drb_rng_draw(&s_, 0, 1, &v, device_));
        return v;
    }
    std::uint64_t bounded(std::uint64_t n) {
        if (n == 0)
            throw usage_error(DRB_ERR_USAGE, "bounded: n must be nonzero");
        std::uint64_t v = 0;
        check(drb_rng_draw(&s_, n, 1, &v, device_));
        return v;
    }
    std::uint64_t counter() const { return s_.ctr; }
    drb_rng* raw() { return &s_; }
    int device() const { return device_; }

private:
    drb_rng s_{};
    int device_ = 0;
};

inline std::vector<std::uint32_t> sample_without_replacement(std::uint32_t n, std::uint32_t k, rng_stream& rng) {
    std::vector<std::uint32_t> out(k < n ? k : n);
    std::uint32_t got = 0;
    check(drb_sample_without_replacement(n, k, rng.raw(), out.data(), &got, rng.device()));
    out.resize(got);
    return out;
}

struct slot_ref {
    std::uint32_t owner = 0, cls = 0, slot = 0;
    bool operator==(const slot_ref&) const = default;
};

struct sampling_plan {
    std::vector<slot_ref> entries;
};

// plan(want, view, rng): view = occupancy[n_workers][n_classes] (sampler.cpp:65-68)
inline sampling_plan plan(std::uint32_t want, const std::vector<std::vector<std::uint32_t>>& view, rng_stream& rng) {
    const std::uint32_t nw = static_cast<std::uint32_t>(view.size());
    const std::uint32_t nk = nw ? static_cast<std::uint32_t>(view[0].size()) : 0;
    std::vector<std::uint32_t> flat;
    std::uint64_t total = 0;
    for (const auto& row : view)
        for (auto o : row) {
            flat.push_back(o);
            total += o;
        }
    sampling_plan p;
    p.entries.resize(want < total ? want : total);
    std::uint32_t got = 0;
    check(drb_plan(want, nw, nk, flat.data(), rng.raw(), reinterpret_cast<drb_slot_ref*>(p.entries.data()), &got,
                   rng.device()));
    p.entries.resize(got);
    return p;
}

struct device_batch {  // a mini-batch resident in device memory
    const void* data = nullptr;        // n x S bytes
    const std::uint32_t* labels = nullptr;
    std::uint32_t n = 0;
};

struct insertion_report {
    std::vector<std::uint32_t> per_class_appends, per_class_replacements;
    std::uint32_t appends = 0, replacements = 0;
};

struct occupancy_snapshot {
    std::vector<std::uint32_t> per_class;
    std::uint64_t version = 0;
    std::uint64_t total() const {
        std::uint64_t t = 0;
        for (auto o : per_class)
            t += o;
        return t;
    }
};

class rehearsal_buffer {
public:
    explicit rehearsal_buffer(const drb_rb_config& cfg) : cfg_(cfg) { check(drb_rb_create(&cfg_, &h_)); }
    rehearsal_buffer(std::uint32_t n_classes, std::uint32_t per_class_cap, std::uint64_t sample_bytes,
                     std::uint32_t max_batch = 64, std::uint32_t c = 14, std::uint32_t r = 7, std::uint64_t seed = 1,
                     int device = 0)
        : rehearsal_buffer(drb_rb_config{n_classes, per_class_cap, sample_bytes, max_batch, c, r, 0, 1, seed, device, 0}) {}
    ~rehearsal_buffer() {
        if (h_)
            drb_rb_destroy(h_);
    }
    rehearsal_buffer(const rehearsal_buffer&) = delete;
    rehearsal_buffer& operator=(const rehearsal_buffer&) = delete;

    insertion_report update_buffer(const device_batch& m, std::uint32_t candidate_count, rng_stream& cand,
                                   rng_stream& evict) {
        insertion_report rep;
        rep.per_class_appends.assign(cfg_.n_classes, 0);
        rep.per_class_replacements.assign(cfg_.n_classes, 0);
        drb_insertion_report r{rep.per_class_appends.data(), rep.per_class_replacements.data(), 0, 0};
        check(drb_rb_update_buffer(h_, m.data, m.labels, m.n, candidate_count, cand.raw(), evict.raw(), &r));
        rep.appends = r.appends;
        rep.replacements = r.replacements;
        return rep;
    }
    occupancy_snapshot snapshot() const {
        occupancy_snapshot s;
        s.per_class.assign(cfg_.n_classes, 0);
        check(drb_rb_snapshot(h_, s.per_class.data(), &s.version));
        return s;
    }
    std::uint64_t total_stored() const {
        std::uint64_t v = 0;
        check(drb_rb_total_stored(h_, &v));
        return v;
    }
    std::uint64_t cross_class_evictions() const {
        std::uint64_t v = 0;
        check(drb_rb_cross_class_evictions(h_, &v));
        return v;
    }
    // read_slots: out / out_labels are device buffers of requests.size() rows
    std::vector<std::uint8_t> read_slots(const std::vector<drb_read_request>& requests, rng_stream& substitute,
                                         void* out, std::uint32_t* out_labels) {
        std::vector<std::uint8_t> status(requests.size());
        check(drb_rb_read_slots(h_, requests.data(), static_cast<std::uint32_t>(requests.size()), substitute.raw(),
                                out, out_labels, status.data()));
        return status;
    }
    std::vector<std::uint8_t> export_handle() const {
        std::vector<std::uint8_t> blob(drb_rb_handle_size());
        std::size_t len = blob.size();
        check(drb_rb_export_handle(h_, blob.data(), &len));
        return blob;
    }
    void connect(const std::vector<std::uint8_t>& all_blobs) { check(drb_rb_connect(h_, all_blobs.data(), all_blobs.size())); }
    std::uint32_t n_classes() const { return cfg_.n_classes; }
    std::uint32_t per_class_cap() const { return cfg_.per_class_cap; }
    drb_rb* raw() const { return h_; }

private:
    drb_rb_config cfg_{};
    drb_rb* h_ = nullptr;
};

// m'_i = m_i ++ reps(i-1), engine-owned; valid until work enqueued before update(i+2).
class augmented_batch {
public:
    augmented_batch(drb_rb* h, const drb_aug& a) : h_(h), a_(a) {}
    const void* data() const { return a_.data; }
    const std::uint32_t* labels() const { return a_.labels; }
    std::uint32_t batch_rows() const { return a_.n; }
    std::uint32_t count() const {  // blocks until this iteration's m' is complete
        std::uint32_t c = 0;
        check(drb_rb_aug_count(h_, &a_, &c));
        return c;
    }
    std::uint32_t reps() const { return count() - a_.n; }

private:
    drb_rb* h_;
    drb_aug a_;
};

class engine {
public:
    explicit engine(rehearsal_buffer& b) : b_(b) {}
    ~engine() {
        if (started_ && !shut_)
            drb_rb_shutdown(b_.raw());
    }
    void start() {
        check(drb_rb_start(b_.raw()));
        started_ = true;
    }
    // engine.update(m) fused with augment(m, reps) (trainer.cpp:109-113); stream: cudaStream_t
    augmented_batch update(const device_batch& m, void* stream = nullptr) {
        drb_aug a{};
        check(drb_rb_step(b_.raw(), m.data, m.labels, m.n, stream, &a));
        return augmented_batch(b_.raw(), a);
    }
    // the loader / trainer split: m posted in `producer` order, `consumer` releases the m'
    // it used and waits for m'_i (drb_rb_step_split)
    augmented_batch update(const device_batch& m, void* producer, void* consumer) {
        drb_aug a{};
        check(drb_rb_step_split(b_.raw(), m.data, m.labels, m.n, producer, consumer, &a));
        return augmented_batch(b_.raw(), a);
    }
    void shutdown() {
        check(drb_rb_shutdown(b_.raw()));
        shut_ = true;
    }
    double total_wait_ms() const {
        double v = 0;
        check(drb_rb_total_wait_ms(b_.raw(), &v));
        return v;
    }
    void synchronize() { check(drb_rb_synchronize(b_.raw())); }
    // engine::iterations / queue_depth / degraded_rounds / replanned_entries (engine.hpp:87-92)
    std::uint64_t iterations() const { return counter(0); }
    std::size_t queue_depth() const { return std::size_t(counter(1)); }
    std::uint64_t degraded_rounds() const { return counter(2); }
    std::uint64_t replanned_entries() const { return counter(3); }
    // engine::broadcast_sizes (engine.hpp:82): a no-op, rows are published every round
    void broadcast_sizes() { check(drb_rb_broadcast_sizes(b_.raw())); }
    // engine::drain_timings (engine.hpp:93); needs DRB_RB_FLAG_TIMINGS in the buffer's config
    std::vector<drb_timing> drain_timings() {
        std::vector<drb_timing> out(4096);
        std::uint32_t n = 0;
        check(drb_rb_drain_timings(b_.raw(), out.data(), std::uint32_t(out.size()), &n));
        out.resize(n);
        return out;
    }

private:
    std::uint64_t counter(int which) const {
        std::uint64_t v[4] = {0, 0, 0, 0};
        check(drb_rb_engine_counters(b_.raw(), &v[0], &v[1], &v[2], &v[3]));
        return v[which];
    }
    rehearsal_buffer& b_;
    bool started_ = false, shut_ = false;
};

// ---- input side: the producer of m (proj/src/scenario/dataset.hpp, schedule.hpp) ----

/// dataset (dataset.hpp:19-40), resident in HBM; load_dataset throws io_error like
/// dataset.cpp:102-143. gather() is dataset::gather on the device: indices is a device array.
class dataset {
public:
    explicit dataset(const std::string& path, int device = 0) {
        check(drb_ds_load(path.c_str(), device, &h_));
        check(drb_ds_info(h_, &count_, &feature_dim, &n_classes, &train_count, &eval_count));
    }
    /// synth_dataset (dataset.cpp:145-205), bit-identical to the reference's, in HBM.
    static dataset synth(std::uint32_t n_classes, std::uint32_t per_class, std::uint32_t feature_dim,
                         double separation, std::uint64_t seed, int device = 0) {
        drb_ds* h = nullptr;
        check(drb_ds_synth(n_classes, per_class, feature_dim, separation, seed, device, &h));
        return dataset(h);
    }
    dataset(dataset&& o) noexcept
        : feature_dim(o.feature_dim), n_classes(o.n_classes), train_count(o.train_count),
          eval_count(o.eval_count), h_(o.h_), count_(o.count_) {
        o.h_ = nullptr;
    }
    ~dataset() {
        if (h_)
            drb_ds_destroy(h_);
    }
    dataset(const dataset&) = delete;
    dataset& operator=(const dataset&) = delete;

    std::size_t size() const { return count_; }
    std::vector<std::size_t> train_indices_of(const std::vector<std::uint32_t>& classes) const {
        return indices_of(classes, 0);
    }
    std::vector<std::size_t> eval_indices_of(const std::vector<std::uint32_t>& classes) const {
        return indices_of(classes, 1);
    }
    /// rows -> out (n x feature_dim*4 bytes) and labels, ordered on `stream`.
    device_batch gather(const std::uint64_t* indices, std::uint32_t n, void* out, std::uint32_t* out_labels,
                        void* stream = nullptr) const {
        check(drb_ds_gather(h_, indices, n, out, out_labels, stream));
        return device_batch{out, out_labels, n};
    }
    std::uint32_t device_error() const {
        std::uint32_t e = 0;
        check(drb_ds_device_error(h_, &e));
        return e;
    }
    drb_ds* raw() const { return h_; }

    std::uint32_t feature_dim = 0, n_classes = 0;
    std::uint64_t train_count = 0, eval_count = 0;

private:
    explicit dataset(drb_ds* h) : h_(h) {
        check(drb_ds_info(h_, &count_, &feature_dim, &n_classes, &train_count, &eval_count));
    }
    std::vector<std::size_t> indices_of(const std::vector<std::uint32_t>& classes, int eval) const {
        std::uint64_t n = 0;
        check(drb_ds_indices_of(h_, classes.data(), std::uint32_t(classes.size()), eval, nullptr, 0, &n));
        std::vector<std::uint64_t> v(n);
        check(drb_ds_indices_of(h_, classes.data(), std::uint32_t(classes.size()), eval, v.data(), n, &n));
        return std::vector<std::size_t>(v.begin(), v.end());
    }
    drb_ds* h_ = nullptr;
    std::uint64_t count_ = 0;
};

/// task_schedule / make_schedule (schedule.hpp:10-25, schedule.cpp:10-35).
struct task_schedule {
    std::vector<std::vector<std::uint32_t>> tasks;
    unsigned epochs_per_task = 1;
};
inline task_schedule make_schedule(std::uint32_t n_classes, std::uint32_t n_tasks, std::uint64_t seed,
                                   unsigned epochs_per_task = 1) {
    std::vector<std::uint32_t> cls(n_classes), sizes(n_tasks);
    check(drb_make_schedule(n_classes, n_tasks, seed, cls.data(), sizes.data()));
    task_schedule s;
    s.epochs_per_task = epochs_per_task;
    std::size_t cur = 0;
    for (std::uint32_t t = 0; t < n_tasks; ++t) {
        s.tasks.emplace_back(cls.begin() + cur, cls.begin() + cur + sizes[t]);
        cur += sizes[t];
    }
    return s;
}

/// shard_batches (schedule.cpp:37-62): this worker's batches for (task, epoch).
inline std::vector<std::vector<std::size_t>> shard_batches(const std::vector<std::size_t>& task_data,
                                                           std::uint32_t worker, std::uint32_t n_workers,
                                                           unsigned batch_size, std::uint64_t seed,
                                                           std::uint64_t task_index, std::uint64_t epoch) {
    const std::vector<std::uint64_t> td(task_data.begin(), task_data.end());
    std::vector<std::uint64_t> out(n_workers ? (td.size() + n_workers - 1) / n_workers : 0);
    std::uint64_t n = 0;
    check(drb_shard_batches(td.data(), td.size(), worker, n_workers, batch_size, seed, task_index, epoch,
                            out.data(), out.size(), &n));
    std::vector<std::vector<std::size_t>> batches;
    for (std::uint64_t s = 0; s < n; s += batch_size)
        batches.emplace_back(out.begin() + s, out.begin() + std::min<std::uint64_t>(n, s + batch_size));
    return batches;
}

inline std::size_t lockstep_batches(std::size_t task_size, std::uint32_t n_workers, unsigned batch_size) {
    std::uint64_t out = 0;
    check(drb_lockstep_batches(task_size, n_workers, batch_size, &out));
    return out;
}

}  // namespace drb::b200
