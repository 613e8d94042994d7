// Test-infrastructure harness over the UNMODIFIED reference (compiled from
// /root/reference/proj/src by oracle/Makefile into oracle/_ref/). Not product
// code: only tests/, __graft_entry__.smoke() and bench.py's reference arm use it.
//
// It exposes, as extern "C", exactly the reference calls the parity oracle needs:
//   * rng_stream draws            (proj/src/core/rng.cpp:33-53)
//   * sample_without_replacement  (proj/src/buffer/rehearsal_buffer.cpp:14-26)
//   * plan over a given view      (proj/src/sampler/sampler.cpp:65-68)
//   * a synchronous multi-rank replay built from rehearsal_buffer::update_buffer,
//     rehearsal_buffer::snapshot, size_table::store_row/view_at, plan and
//     rehearsal_buffer::read_slots — the "synchronous replay" oracle of SURVEY.md §8c
//   * the real asynchronous engine (engine::update + augment), N in-process workers
//     over loopback TCP (the engine_pair wiring of proj/tests/test_engine.cpp:57-107
//     generalised to N), timed for the CPU baseline.
// Byte payloads ride in the reference's float features bit-exactly (S/4 floats;
// copies are memmove so bits survive).

#include "buffer/rehearsal_buffer.hpp"
#include "core/config.hpp"
#include "core/errors.hpp"
#include "core/rng.hpp"
#include "engine/engine.hpp"
#include "metrics/metrics.hpp"
#include "runner/mesh.hpp"
#include "scenario/dataset.hpp"
#include "scenario/schedule.hpp"
#include "sampler/sampler.hpp"
#include "sampler/size_table.hpp"
#include "transport/socket.hpp"

#include <chrono>
#include <cstring>
#include <memory>
#include <thread>
#include <vector>

using namespace drb;

namespace {

rng_stream make_stream(std::uint64_t seed, std::uint32_t worker, std::uint32_t purpose,
                       int keyed, std::uint64_t k1, std::uint64_t k2) {
    const auto p = static_cast<rng_stream::purpose>(purpose);
    return keyed ? rng_stream::keyed(seed, worker, p, k1, k2) : rng_stream(seed, worker, p);
}

sample to_sample(const std::uint8_t* bytes, std::size_t S, std::uint32_t label) {
    sample s;
    s.features.resize(S / 4);
    std::memcpy(s.features.data(), bytes, S);
    s.label = label;
    return s;
}

mini_batch to_batch(const std::uint8_t* bytes, const std::uint32_t* labels, std::size_t n,
                    std::size_t S) {
    mini_batch m(n);
    for (std::size_t i = 0; i < n; ++i)
        m[i] = to_sample(bytes + i * S, S, labels[i]);
    return m;
}

struct replay {
    std::uint32_t N, K, cap, c, r;
    std::size_t S;
    std::uint64_t seed;
    std::vector<std::unique_ptr<rehearsal_buffer>> buffers;
    std::vector<std::unique_ptr<size_table>> tables;
    std::vector<rng_stream> cand, evict, samp, subst;
    std::vector<std::vector<sample>> pending;          // reps(i-1) per rank
    std::vector<std::vector<slot_ref>> last_plan;      // plan(i) per rank
    std::vector<insertion_report> last_report;
    std::uint64_t step = 0;
};

} // namespace

extern "C" {

int ref_rng_next(std::uint64_t seed, std::uint32_t worker, std::uint32_t purpose, int keyed,
                 std::uint64_t k1, std::uint64_t k2, std::uint64_t n, std::uint64_t* out) {
    auto s = make_stream(seed, worker, purpose, keyed, k1, k2);
    for (std::uint64_t i = 0; i < n; ++i)
        out[i] = s.next_u64();
    return 0;
}

int ref_rng_bounded(std::uint64_t seed, std::uint32_t worker, std::uint32_t purpose, int keyed,
                    std::uint64_t k1, std::uint64_t k2, std::uint64_t bound, std::uint64_t n,
                    std::uint64_t* out) {
    auto s = make_stream(seed, worker, purpose, keyed, k1, k2);
    for (std::uint64_t i = 0; i < n; ++i)
        out[i] = s.bounded(bound);
    return 0;
}

int ref_swor(std::uint64_t n, std::uint64_t k, std::uint64_t seed, std::uint32_t worker,
             std::uint32_t purpose, std::uint64_t* out, std::uint64_t* out_k) {
    auto s = make_stream(seed, worker, purpose, 0, 0, 0);
    const auto idx = sample_without_replacement(n, k, s);
    for (std::size_t i = 0; i < idx.size(); ++i)
        out[i] = idx[i];
    *out_k = idx.size();
    return 0;
}

// plan(want, view{occ[n_workers][n_classes]}, rng(seed, worker, purpose)) repeated
// `rounds` times on one stream; entries written as (owner, cls, slot) triples.
int ref_plan(std::uint64_t want, std::uint32_t n_workers, std::uint32_t n_classes,
             const std::uint32_t* occ, std::uint64_t seed, std::uint32_t worker,
             std::uint32_t purpose, std::uint32_t rounds, std::uint32_t* out,
             std::uint64_t* out_counts) {
    size_table::view v;
    v.n_workers = n_workers;
    v.n_classes = n_classes;
    v.occupancy.resize(n_workers);
    for (std::uint32_t w = 0; w < n_workers; ++w) {
        v.occupancy[w].assign(occ + w * n_classes, occ + (w + 1) * n_classes);
        for (auto o : v.occupancy[w])
            v.total += o;
    }
    auto s = make_stream(seed, worker, purpose, 0, 0, 0);
    std::size_t pos = 0;
    for (std::uint32_t rd = 0; rd < rounds; ++rd) {
        const auto p = plan(want, v, s);
        out_counts[rd] = p.entries.size();
        for (const auto& e : p.entries) {
            out[pos++] = e.owner;
            out[pos++] = e.cls;
            out[pos++] = e.slot;
        }
    }
    return 0;
}

void* ref_replay_create(std::uint32_t N, std::uint32_t K, std::uint32_t cap, std::uint64_t S,
                        std::uint32_t c, std::uint32_t r, std::uint64_t seed) {
    auto* h = new replay{};
    h->N = N; h->K = K; h->cap = cap; h->c = c; h->r = r; h->S = S; h->seed = seed;
    for (std::uint32_t w = 0; w < N; ++w) {
        h->buffers.push_back(std::make_unique<rehearsal_buffer>(K, cap));
        h->tables.push_back(std::make_unique<size_table>(N, K, w));
        // Per-rank streams exactly as the engine wires them (proj/src/engine/engine.cpp:27-35).
        h->cand.emplace_back(seed, w, rng_stream::purpose::candidate_selection);
        h->evict.emplace_back(seed, w, rng_stream::purpose::eviction);
        h->samp.emplace_back(seed, w, rng_stream::purpose::global_sampling);
        h->subst.emplace_back(seed, w, rng_stream::purpose::slot_substitute);
    }
    h->pending.resize(N);
    h->last_plan.resize(N);
    h->last_report.resize(N);
    return h;
}

void ref_replay_destroy(void* p) { delete static_cast<replay*>(p); }

// One synchronous round i on every rank. batches: N x n x S bytes, labels N x n.
// Writes m'_i = m_i ++ reps(i-1) into out (N x (n+r) x S) / out_labels, out_counts[N].
int ref_replay_step(void* p, const std::uint8_t* batches, const std::uint32_t* labels,
                    std::uint32_t n, std::uint8_t* out, std::uint32_t* out_labels,
                    std::uint32_t* out_counts) {
    auto* h = static_cast<replay*>(p);
    const std::size_t S = h->S;
    try {
        for (std::uint32_t w = 0; w < h->N; ++w) {
            const auto m = to_batch(batches + std::size_t(w) * n * S, labels + std::size_t(w) * n, n, S);
            h->last_report[w] = h->buffers[w]->update_buffer(m, h->c, h->cand[w], h->evict[w]);
        }
    } catch (const usage_error&) {
        return 7;
    }
    // publish_row (engine.cpp:108-136): version = round+1, every table gets every row.
    for (std::uint32_t w = 0; w < h->N; ++w) {
        const auto snap = h->buffers[w]->snapshot();
        for (std::uint32_t t = 0; t < h->N; ++t)
            h->tables[t]->store_row(w, h->step + 1, snap.per_class);
    }
    // assemble m'_i from the previous round's reps.
    for (std::uint32_t w = 0; w < h->N; ++w) {
        std::uint8_t* o = out + std::size_t(w) * (n + h->r) * S;
        std::uint32_t* ol = out_labels + std::size_t(w) * (n + h->r);
        std::memcpy(o, batches + std::size_t(w) * n * S, std::size_t(n) * S);
        std::memcpy(ol, labels + std::size_t(w) * n, n * 4);
        const auto& reps = h->pending[w];
        for (std::size_t j = 0; j < reps.size(); ++j) {
            std::memcpy(o + (n + j) * S, reps[j].features.data(), S);
            ol[n + j] = reps[j].label;
        }
        out_counts[w] = n + static_cast<std::uint32_t>(reps.size());
    }
    // plan(i) + exact reads at version i+1 (engine.cpp:152-160; serve path engine.cpp:215-251).
    for (std::uint32_t w = 0; w < h->N; ++w) {
        const auto view = h->tables[w]->view_at(h->step + 1, std::chrono::milliseconds(0));
        const auto pl = plan(h->r, view, h->samp[w]);
        h->last_plan[w] = pl.entries;
        std::vector<sample> reps;
        for (const auto& e : pl.entries) {
            const std::vector<read_request> req{{e.cls, e.slot}};
            auto got = h->buffers[e.owner]->read_slots(req, h->subst[e.owner]);
            if (got[0].status != read_status::exact)
                return 8; // cannot happen under exact horizons
            reps.push_back(std::move(got[0].value));
        }
        h->pending[w] = std::move(reps);
        h->tables[w]->prune_below(h->step + 1);
    }
    ++h->step;
    return 0;
}

// Plan drawn at the last step for rank w: (owner, cls, slot) triples; returns count.
std::uint32_t ref_replay_last_plan(void* p, std::uint32_t w, std::uint32_t* out) {
    auto* h = static_cast<replay*>(p);
    const auto& pl = h->last_plan[w];
    for (std::size_t j = 0; j < pl.size(); ++j) {
        out[3 * j] = pl[j].owner;
        out[3 * j + 1] = pl[j].cls;
        out[3 * j + 2] = pl[j].slot;
    }
    return static_cast<std::uint32_t>(pl.size());
}

// Last insertion report of rank w: per-class appends/replacements (K each) + totals.
int ref_replay_last_report(void* p, std::uint32_t w, std::uint32_t* appends,
                           std::uint32_t* replacements, std::uint32_t* totals) {
    auto* h = static_cast<replay*>(p);
    const auto& rep = h->last_report[w];
    std::memset(appends, 0, h->K * 4);
    std::memset(replacements, 0, h->K * 4);
    for (const auto& [cls, cnt] : rep.per_class) {
        appends[cls] = cnt.appends;
        replacements[cls] = cnt.replacements;
    }
    totals[0] = rep.appends;
    totals[1] = rep.replacements;
    return 0;
}

// Snapshot + full slab dump of rank w (slab: K x cap x S, unoccupied slots zeroed).
int ref_replay_dump(void* p, std::uint32_t w, std::uint32_t* occ, std::uint64_t* version,
                    std::uint8_t* slab, std::uint32_t* slab_labels) {
    auto* h = static_cast<replay*>(p);
    const auto snap = h->buffers[w]->snapshot();
    *version = snap.version;
    rng_stream sub(0, 0, rng_stream::purpose::slot_substitute);
    for (std::uint32_t k = 0; k < h->K; ++k) {
        occ[k] = snap.per_class[k];
        for (std::uint32_t s = 0; s < h->cap; ++s) {
            std::uint8_t* dst = slab + (std::size_t(k) * h->cap + s) * h->S;
            if (s < snap.per_class[k]) {
                const std::vector<read_request> req{{k, s}};
                const auto got = h->buffers[w]->read_slots(req, sub);
                std::memcpy(dst, got[0].value.features.data(), h->S);
                slab_labels[k * h->cap + s] = got[0].value.label;
            } else {
                std::memset(dst, 0, h->S);
                slab_labels[k * h->cap + s] = 0;
            }
        }
    }
    return 0;
}

// The reference's real asynchronous engine, timed: N in-process workers (own buffer,
// size_table, worker_mesh over loopback TCP, engine), one driver thread each doing
// `reps = engine.update(m); m' = augment(m, reps)` (proj/src/trainer/trainer.cpp:109-113,
// proj/src/runner/overlap.cpp:83-89 with zero train cost). batches: per rank a ring of
// n_batches batches (N x n_batches x n x S bytes). Runs `warmup` untimed then `iters`
// timed iterations per worker; returns the slowest worker's timed seconds in *seconds
// and the total augmented samples produced in *samples.
int ref_engine_bench(std::uint32_t N, std::uint32_t K, std::uint32_t cap, std::uint64_t S,
                     std::uint32_t n, std::uint32_t c, std::uint32_t r, std::uint64_t seed,
                     const std::uint8_t* batches, const std::uint32_t* labels,
                     std::uint32_t n_batches, std::uint32_t warmup, std::uint32_t iters,
                     double* seconds, std::uint64_t* samples) {
    try {
        run_config cfg;
        cfg.n_workers = N;
        cfg.n_classes = K;
        cfg.batch_size = n;
        cfg.rep_count = r;
        cfg.candidate_count = c;
        cfg.feature_dim = static_cast<unsigned>(S / 4);
        cfg.rng_seed = seed;
        std::vector<roster_entry> roster;
        for (std::uint32_t w = 0; w < N; ++w)
            roster.push_back({w, "127.0.0.1", N > 1 ? find_free_port() : std::uint16_t(0)});

        // Pre-convert the input rings into reference mini_batches (not timed).
        std::vector<std::vector<mini_batch>> rings(N);
        for (std::uint32_t w = 0; w < N; ++w)
            for (std::uint32_t i = 0; i < n_batches; ++i) {
                const std::size_t off = (std::size_t(w) * n_batches + i) * n;
                rings[w].push_back(to_batch(batches + off * S, labels + off, n, S));
            }

        std::vector<std::unique_ptr<rehearsal_buffer>> bufs;
        std::vector<std::unique_ptr<size_table>> tables;
        std::vector<std::unique_ptr<worker_mesh>> meshes;
        std::vector<std::unique_ptr<engine>> engines;
        for (std::uint32_t w = 0; w < N; ++w) {
            bufs.push_back(std::make_unique<rehearsal_buffer>(K, cap));
            tables.push_back(std::make_unique<size_table>(N, K, w));
            meshes.push_back(std::make_unique<worker_mesh>(cfg, w, roster));
            engines.push_back(std::make_unique<engine>(cfg, w, *bufs[w], *tables[w],
                                                       meshes[w]->client()));
            meshes[w]->wire_engine(*engines[w]);
            meshes[w]->start();
        }
        for (auto& e : engines)
            e->start();

        std::vector<double> secs(N, 0.0);
        std::vector<std::uint64_t> produced(N, 0);
        std::vector<std::thread> threads;
        for (std::uint32_t w = 0; w < N; ++w) {
            threads.emplace_back([&, w] {
                std::size_t next = 0;
                for (std::uint32_t i = 0; i < warmup; ++i) {
                    const auto& m = rings[w][next++ % n_batches];
                    auto reps = engines[w]->update(m);
                    auto aug = augment(m, reps);
                    (void)aug;
                }
                const auto t0 = std::chrono::steady_clock::now();
                std::uint64_t got = 0;
                for (std::uint32_t i = 0; i < iters; ++i) {
                    const auto& m = rings[w][next++ % n_batches];
                    auto reps = engines[w]->update(m);
                    auto aug = augment(m, reps);
                    got += aug.size();
                }
                secs[w] = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
                produced[w] = got;
            });
        }
        for (auto& t : threads)
            t.join();
        for (auto& e : engines)
            e->shutdown();
        for (auto& m : meshes)
            m->stop();
        double worst = 0.0;
        std::uint64_t total = 0;
        for (std::uint32_t w = 0; w < N; ++w) {
            worst = std::max(worst, secs[w]);
            total += produced[w];
        }
        *seconds = worst;
        *samples = total;
        return 0;
    } catch (const std::exception&) {
        return 8;
    }
}

// rehearsal_buffer(K, cap), `rounds` update_buffer calls (streams (seed, 0, candidate) and
// (seed, 0, eviction)), then ONE read_slots(req, sub) with sub = keyed or plain
// (seed, 0, purpose, k1, k2): the exact / substituted / empty branches of
// proj/src/buffer/rehearsal_buffer.cpp:88-142 and the substitute draws they consume.
// batches: rounds x n x S, labels rounds x n. out: count x S, out_labels, status[count],
// *sub_next = the substitute stream's next draw afterwards (its counter position; the
// counter itself is private), occ_out[K] the occupancy.
int ref_read_slots_scenario(std::uint32_t K, std::uint32_t cap, std::uint64_t S, std::uint32_t rounds,
                            const std::uint8_t* batches, const std::uint32_t* labels, std::uint32_t n,
                            std::uint32_t c, std::uint64_t seed, int keyed, std::uint32_t purpose,
                            std::uint64_t k1, std::uint64_t k2, const std::uint32_t* req, std::uint32_t count,
                            std::uint8_t* out, std::uint32_t* out_labels, std::uint8_t* status,
                            std::uint64_t* sub_next, std::uint32_t* occ_out) {
    try {
        rehearsal_buffer buf(K, cap);
        rng_stream cand(seed, 0, rng_stream::purpose::candidate_selection);
        rng_stream evict(seed, 0, rng_stream::purpose::eviction);
        for (std::uint32_t i = 0; i < rounds; ++i)
            buf.update_buffer(to_batch(batches + std::size_t(i) * n * S, labels + std::size_t(i) * n, n, S), c,
                              cand, evict);
        rng_stream sub = make_stream(seed, 0, purpose, keyed, k1, k2);
        std::vector<read_request> rq(count);
        for (std::uint32_t i = 0; i < count; ++i)
            rq[i] = read_request{req[2 * i], req[2 * i + 1]};
        const auto got = buf.read_slots(rq, sub);
        for (std::uint32_t i = 0; i < count; ++i) {
            status[i] = static_cast<std::uint8_t>(got[i].status);
            if (got[i].status == read_status::empty) {
                std::memset(out + std::size_t(i) * S, 0, S);
                out_labels[i] = 0;
            } else {
                std::memcpy(out + std::size_t(i) * S, got[i].value.features.data(), S);
                out_labels[i] = got[i].value.label;
            }
        }
        *sub_next = sub.next_u64();
        const auto snap = buf.snapshot();
        for (std::uint32_t k = 0; k < K; ++k)
            occ_out[k] = snap.per_class[k];
        return 0;
    } catch (const std::exception&) {
        return 8;
    }
}

// make_bias_report (proj/src/metrics/metrics.cpp:90-107): Pearson chi-square of per-slot
// hit counts against uniform, p-value by the reference's gamma_q (stats.cpp:54-96).
int ref_bias_report(const std::uint64_t* counts, std::uint64_t n, std::uint64_t rep_count,
                    std::uint64_t draws, double* statistic, double* p_value) {
    try {
        const auto r = make_bias_report(std::span<const std::uint64_t>(counts, n), rep_count, draws);
        *statistic = r.statistic;
        *p_value = r.p_value;
        return 0;
    } catch (...) {
        return 8;
    }
}

// ---- input side: DRDS files, class-incremental schedule, shards ----

// synth_dataset + write_dataset (proj/src/scenario/dataset.cpp): the reference's own writer.
int ref_write_synth_dataset(const char* path, std::uint32_t n_classes, std::uint32_t per_class,
                            std::uint32_t feature_dim, double separation, std::uint64_t seed) {
    try {
        write_dataset(synth_dataset(n_classes, per_class, feature_dim, separation, seed), path);
        return 0;
    } catch (...) {
        return -1;
    }
}

// load_dataset: 0 ok, 3 io_error (message into err), -1 other. out_* may be NULL (header only).
int ref_load_dataset(const char* path, std::uint64_t* count, std::uint32_t* dim,
                     std::uint32_t* n_classes, std::uint64_t* train, std::uint64_t* eval,
                     float* out_features, std::uint32_t* out_labels, char* err, std::size_t err_len) {
    try {
        const dataset d = load_dataset(path);
        *count = d.size();
        *dim = d.feature_dim;
        *n_classes = d.n_classes;
        *train = d.train_count;
        *eval = d.eval_count;
        if (out_features)
            std::memcpy(out_features, d.features.data(), d.features.size() * sizeof(float));
        if (out_labels)
            std::memcpy(out_labels, d.labels.data(), d.labels.size() * sizeof(std::uint32_t));
        return 0;
    } catch (const io_error& e) {
        if (err && err_len) {
            std::strncpy(err, e.what(), err_len - 1);
            err[err_len - 1] = 0;
        }
        return 3;
    } catch (...) {
        return -1;
    }
}

// train_indices_of / eval_indices_of; returns the count, writes up to cap.
std::uint64_t ref_indices_of(const char* path, const std::uint32_t* classes, std::uint32_t n,
                             int eval, std::uint64_t* out, std::uint64_t cap) {
    const dataset d = load_dataset(path);
    const std::vector<class_id> cls(classes, classes + n);
    const auto v = eval ? d.eval_indices_of(cls) : d.train_indices_of(cls);
    for (std::size_t i = 0; i < v.size() && i < cap; ++i)
        out[i] = v[i];
    return v.size();
}

int ref_make_schedule(std::uint32_t K, std::uint32_t T, std::uint64_t seed, std::uint32_t* classes,
                      std::uint32_t* sizes) {
    try {
        const auto s = make_schedule(K, T, seed);
        std::size_t c = 0;
        for (std::uint32_t t = 0; t < T; ++t) {
            sizes[t] = static_cast<std::uint32_t>(s.tasks[t].size());
            for (const auto k : s.tasks[t])
                classes[c++] = k;
        }
        return 0;
    } catch (const config_error&) {
        return 2;
    } catch (...) {
        return -1;
    }
}

// shard_batches flattened: batches concatenated in order (batch boundaries every `batch`).
int ref_shard_batches(const std::uint64_t* task_data, std::uint64_t n, std::uint32_t worker,
                      std::uint32_t n_workers, std::uint32_t batch, std::uint64_t seed,
                      std::uint64_t task_index, std::uint64_t epoch, std::uint64_t* out,
                      std::uint64_t* n_out, std::uint64_t* n_batches) {
    try {
        const std::vector<std::size_t> td(task_data, task_data + n);
        const auto b = shard_batches(td, worker, n_workers, batch, seed, task_index, epoch);
        std::uint64_t c = 0;
        for (const auto& v : b)
            for (const auto i : v)
                out[c++] = i;
        *n_out = c;
        *n_batches = b.size();
        return 0;
    } catch (const usage_error&) {
        return 7;
    } catch (...) {
        return -1;
    }
}

std::uint64_t ref_lockstep_batches(std::uint64_t task_size, std::uint32_t n_workers, std::uint32_t batch) {
    return lockstep_batches(task_size, n_workers, batch);
}

} // extern "C"
