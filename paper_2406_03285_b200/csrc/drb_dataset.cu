// Input side of the hot path: the producer of m.
//
//   DRDS dataset file -> HBM (load_dataset, proj/src/scenario/dataset.cpp:102-143)
//   class-incremental schedule and per-worker shards (proj/src/scenario/schedule.cpp:10-69)
//   dataset::gather of a batch of records into m (proj/src/scenario/dataset.cpp:66-72)
//
// HBM layout: the file's record-interleaved [count][dim f32 | u32 label] is split on the
// device into SoA features [count][dim*4 B] (rows 16 B aligned whenever dim % 4 == 0) and
// labels u32[count], so a batch gather is a straight row copy into the rehearsal buffer's
// m layout ([b][S] bytes + u32 labels[b], S = dim*4). The file is streamed through two
// pinned staging buffers (each chunk read by up to 16 pread threads, which also validate
// the labels of their slice); each chunk's H2D copy overlaps the next chunk's read, and the
// split kernel runs per chunk on the device.

#include <cuda_runtime.h>
#include <unistd.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <limits>
#include <memory>
#include <stdexcept>
#include <string>
#include <thread>
#include <unordered_set>
#include <vector>

#include "drb_internal.cuh"

namespace drb_b200 {
void set_last_error(const char* what);
}

struct drb_ds {
    int device = 0;
    uint64_t count = 0, train = 0, eval = 0;
    uint32_t dim = 0, n_classes = 0;
    uint8_t* features = nullptr;  // [count][dim*4]
    uint32_t* labels = nullptr;   // [count]
    uint32_t* err = nullptr;      // device error word of gathers (bit 0: index out of range)
    std::vector<uint32_t> host_labels;
    ~drb_ds() {
        int prev = -1;
        cudaGetDevice(&prev);
        cudaSetDevice(device);
        cudaFree(features);
        cudaFree(labels);
        cudaFree(err);
        if (prev >= 0)
            cudaSetDevice(prev);
    }
};

namespace {

struct ds_error : std::runtime_error {
    drb_status code;
    ds_error(drb_status c, const std::string& w) : std::runtime_error(w), code(c) {}
};

[[noreturn]] void fail(drb_status c, const std::string& w) { throw ds_error(c, w); }

void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess)
        fail(DRB_ERR_INTERNAL, std::string(what) + ": " + cudaGetErrorString(e));
}

template <typename F>
drb_status guarded(F&& f) {
    try {
        f();
        return DRB_OK;
    } catch (const ds_error& e) {
        drb_b200::set_last_error(e.what());
        return e.code;
    } catch (const std::bad_alloc&) {
        drb_b200::set_last_error("out of memory");
        return DRB_ERR_INTERNAL;
    } catch (const std::exception& e) {
        drb_b200::set_last_error(e.what());
        return DRB_ERR_INTERNAL;
    }
}

#define DS_REQUIRE(cond)                                  \
    do {                                                  \
        if (!(cond)) {                                    \
            drb_b200::set_last_error("null argument");    \
            return DRB_ERR_INVALID_ARGUMENT;              \
        }                                                 \
    } while (0)

struct device_scope {
    int prev = -1;
    explicit device_scope(int dev) {
        cudaGetDevice(&prev);
        if (prev != dev)
            cuda_check(cudaSetDevice(dev), "cudaSetDevice");
    }
    ~device_scope() {
        int cur = -1;
        cudaGetDevice(&cur);
        if (prev >= 0 && cur != prev)
            cudaSetDevice(prev);
    }
};

// ---- host splitmix stream (rng.cpp:12-53): shuffles of the input side only ----
constexpr uint64_t kPhiH = 0x9e3779b97f4a7c15ULL;
uint64_t mix(uint64_t z) {
    z += kPhiH;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}
struct host_rng {
    uint64_t key, ctr = 0;
    // rng_stream::keyed(seed, worker, purpose, k1, k2) (rng.cpp:19-39): k1+1, k2+1 folded in.
    host_rng(uint64_t seed, uint64_t worker, uint64_t purpose, uint64_t k1, uint64_t k2, bool keyed = true) {
        key = mix(seed);
        key = mix(key ^ (worker * 0xd1342543de82ef95ULL));
        key = mix(key ^ (purpose * 0xaf251af3b0f025b5ULL));
        key = mix(key ^ (keyed ? k1 + 1 : 0));  // the plain ctor folds 0, 0 (rng.cpp:33-34)
        key = mix(key ^ (keyed ? k2 + 1 : 0));
    }
    double next_double() { return double(next() >> 11) * 0x1.0p-53; }  // rng.cpp:54-56
    bool has_spare = false;
    double spare = 0;
    double gaussian() {  // Box-Muller with a cached spare (rng.cpp:58-72)
        if (has_spare) {
            has_spare = false;
            return spare;
        }
        double u1 = next_double();
        const double u2 = next_double();
        if (u1 <= 0.0)
            u1 = 0x1.0p-53;
        const double radius = std::sqrt(-2.0 * std::log(u1));
        const double angle = 2.0 * M_PI * u2;
        spare = radius * std::sin(angle);
        has_spare = true;
        return radius * std::cos(angle);
    }
    uint64_t next() { return mix(key ^ (++ctr * kPhiH)); }
    uint64_t bounded(uint64_t n) {  // rng.cpp:45-53
        const uint64_t thr = (0 - n) % n;
        for (;;) {
            const uint64_t v = next();
            if (v >= thr)
                return v % n;
        }
    }
};
constexpr uint64_t kDataShuffle = 4;  // rng.hpp purpose::data_shuffle
constexpr uint64_t kSynth = 7;        // rng.hpp purpose::synth

// ---- kernels ----

// One chunk of records [dim words | label word] -> SoA features rows (labels come from the
// host pass). Word-granular grid-stride loop: reads fully coalesced, writes coalesced
// within each row.
__global__ void ds_split_kernel(const uint32_t* __restrict__ rec, uint64_t n_words, uint32_t dim,
                                uint32_t* __restrict__ feat) {
    const uint32_t stride = dim + 1;
    for (uint64_t w = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; w < n_words;
         w += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t r = w / stride;
        const uint32_t f = uint32_t(w - r * stride);
        if (f < dim)
            feat[r * dim + f] = rec[w];
    }
}

// m[j] = features[idx[j]], labels[j] = labels[idx[j]] (dataset.cpp:66-72). blockIdx.y walks
// the batch rows, blockIdx.x tiles of kUnroll*blockDim words of a row: every thread issues
// its kUnroll loads before any store (kUnroll 4, 4 CTAs per SM: ~64 KB of reads in flight per SM).
template <typename V, int kUnroll>
__global__ void __launch_bounds__(256) ds_gather_kernel(const uint8_t* __restrict__ feat,
                                                        const uint32_t* __restrict__ labels, uint64_t count,
                                                        uint64_t row_bytes, const uint64_t* __restrict__ idx,
                                                        uint32_t n, uint8_t* __restrict__ out,
                                                        uint32_t* __restrict__ out_labels, uint32_t* err) {
    const uint64_t row_words = row_bytes / sizeof(V);
    const uint64_t tile = uint64_t(blockDim.x) * kUnroll;
    for (uint32_t j = blockIdx.y; j < n; j += gridDim.y) {
        const uint64_t i = idx[j];
        if (i >= count) {
            if (blockIdx.x == 0 && threadIdx.x == 0)
                atomicOr(err, 1u);
            continue;
        }
        const V* src = reinterpret_cast<const V*>(feat + i * row_bytes);
        V* dst = reinterpret_cast<V*>(out + uint64_t(j) * row_bytes);
        for (uint64_t base = blockIdx.x * tile; base < row_words; base += uint64_t(gridDim.x) * tile) {
            V v[kUnroll];
#pragma unroll
            for (int u = 0; u < kUnroll; ++u) {
                const uint64_t w = base + u * blockDim.x + threadIdx.x;
                if (w < row_words)
                    v[u] = __ldcs(src + w);  // streamed once: evict-first in L2
            }
#pragma unroll
            for (int u = 0; u < kUnroll; ++u) {
                const uint64_t w = base + u * blockDim.x + threadIdx.x;
                if (w < row_words)
                    dst[w] = v[u];
            }
        }
        if (out_labels && blockIdx.x == 0 && threadIdx.x == 0)
            out_labels[j] = labels[i];
    }
}

uint64_t read_le(const uint8_t* p, int n) {
    uint64_t v = 0;
    for (int i = 0; i < n; ++i)
        v |= uint64_t(p[i]) << (8 * i);
    return v;
}

struct file_closer {
    void operator()(FILE* f) const {
        if (f)
            fclose(f);
    }
};

struct pinned {
    void* p = nullptr;
    ~pinned() { cudaFreeHost(p); }
};
struct devbuf {
    void* p = nullptr;
    ~devbuf() { cudaFree(p); }
};

}  // namespace

extern "C" {

drb_status drb_ds_load(const char* path, int32_t device, drb_ds** out) {
    DS_REQUIRE(path && out);
    return guarded([&] {
        const std::string P(path);
        std::unique_ptr<FILE, file_closer> f(fopen(path, "rb"));
        if (!f)
            fail(DRB_ERR_IO, "cannot open dataset file: " + P);
        uint8_t hdr[22];
        const size_t got = fread(hdr, 1, sizeof hdr, f.get());
        if (got < 4 || std::memcmp(hdr, "DRDS", 4) != 0)
            fail(DRB_ERR_IO, "not a dataset file (bad magic): " + P);
        if (got < 6)
            fail(DRB_ERR_IO, "truncated dataset file: " + P);
        const uint64_t version = read_le(hdr + 4, 2);
        if (version != 1)
            fail(DRB_ERR_IO, "unsupported dataset version " + std::to_string(version) + ": " + P);
        if (got < sizeof hdr)
            fail(DRB_ERR_IO, "truncated dataset file: " + P);
        std::unique_ptr<drb_ds> ds(new drb_ds);
        ds->device = device;
        ds->count = read_le(hdr + 6, 8);
        ds->dim = uint32_t(read_le(hdr + 14, 4));
        ds->n_classes = uint32_t(read_le(hdr + 18, 4));
        const uint64_t rec_words = uint64_t(ds->dim) + 1, rec_bytes = rec_words * 4;
        device_scope g(device);
        const uint64_t row_bytes = uint64_t(ds->dim) * 4;
        // an absurd header count fails as truncated before anything is allocated
        fseek(f.get(), 0, SEEK_END);
        const uint64_t fsize = uint64_t(ftell(f.get()));
        fseek(f.get(), long(sizeof hdr), SEEK_SET);
        const uint64_t avail = (fsize - sizeof hdr) / rec_bytes;
        const uint64_t alloc_n = std::min(ds->count, avail);
        ds->host_labels.resize(alloc_n);
        cuda_check(cudaMalloc(&ds->features, std::max<uint64_t>(alloc_n * row_bytes, 16)), "ds features");
        cuda_check(cudaMalloc(&ds->labels, std::max<uint64_t>(alloc_n * 4, 4)), "ds labels");
        cuda_check(cudaMalloc(&ds->err, 4), "ds err");
        cuda_check(cudaMemset(ds->err, 0, 4), "ds err");
        cudaStream_t st;
        cuda_check(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking), "ds stream");
        std::shared_ptr<void> st_guard(nullptr, [&](void*) { cudaStreamDestroy(st); });
        const uint64_t chunk_recs =
            std::max<uint64_t>(1, std::min<uint64_t>(alloc_n, (64ull << 20) / rec_bytes));
        pinned h[2];
        devbuf d[2];
        cudaEvent_t ev[2];
        for (int b = 0; b < 2; ++b) {
            cuda_check(cudaMallocHost(&h[b].p, chunk_recs * rec_bytes), "ds staging");
            cuda_check(cudaMalloc(&d[b].p, chunk_recs * rec_bytes), "ds staging");
            cuda_check(cudaEventCreateWithFlags(&ev[b], cudaEventDisableTiming), "ds event");
        }
        std::shared_ptr<void> ev_guard(nullptr, [&](void*) {
            cudaEventDestroy(ev[0]);
            cudaEventDestroy(ev[1]);
        });
        int dev_sms = 148;
        cudaDeviceGetAttribute(&dev_sms, cudaDevAttrMultiProcessorCount, device);
        const int fd = fileno(f.get());
        const unsigned reader_threads = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
        uint64_t base = 0;
        for (int b = 0; base < alloc_n; b ^= 1) {
            const uint64_t nrec = std::min(chunk_recs, alloc_n - base);
            cuda_check(cudaEventSynchronize(ev[b]), "ds staging reuse");
            // parallel pread of the chunk into pinned memory + label scan per slice; the first
            // bad record (lowest index) wins, as in the reference's sequential read
            const uint32_t* w = static_cast<const uint32_t*>(h[b].p);
            const unsigned nt = unsigned(std::min<uint64_t>(reader_threads, nrec));
            std::vector<uint64_t> bad(nt, UINT64_MAX);
            std::vector<char> short_read(nt, 0);
            auto slice = [&](unsigned t) {
                const uint64_t r0 = nrec * t / nt, r1 = nrec * (t + 1) / nt;
                const uint64_t off = sizeof hdr + (base + r0) * rec_bytes, len = (r1 - r0) * rec_bytes;
                char* dst = static_cast<char*>(h[b].p) + r0 * rec_bytes;
                for (uint64_t got_b = 0; got_b < len;) {
                    const ssize_t k = pread(fd, dst + got_b, size_t(std::min<uint64_t>(len - got_b, 1ull << 30)),
                                            off_t(off + got_b));
                    if (k <= 0) {
                        short_read[t] = 1;
                        return;
                    }
                    got_b += uint64_t(k);
                }
                for (uint64_t r = r0; r < r1; ++r) {
                    const uint32_t lab = w[r * rec_words + ds->dim];
                    if (lab >= ds->n_classes) {
                        bad[t] = base + r;
                        return;
                    }
                    ds->host_labels[base + r] = lab;
                }
            };
            std::vector<std::thread> pool;
            for (unsigned t = 1; t < nt; ++t)
                pool.emplace_back(slice, t);
            slice(0);
            for (auto& th : pool)
                th.join();
            for (unsigned t = 0; t < nt; ++t) {
                if (short_read[t])
                    fail(DRB_ERR_IO, "truncated dataset file: " + P);
                if (bad[t] != UINT64_MAX)
                    fail(DRB_ERR_IO, "dataset label out of range at record " + std::to_string(bad[t]) + ": " + P);
            }
            cuda_check(cudaMemcpyAsync(d[b].p, h[b].p, nrec * rec_bytes, cudaMemcpyHostToDevice, st), "ds h2d");
            if (ds->dim)
                ds_split_kernel<<<dev_sms * 8, 256, 0, st>>>(static_cast<const uint32_t*>(d[b].p),
                                                            nrec * rec_words, ds->dim,
                                                            reinterpret_cast<uint32_t*>(ds->features) +
                                                                base * ds->dim);
            cuda_check(cudaGetLastError(), "ds split launch");
            cuda_check(cudaEventRecord(ev[b], st), "ds event");
            base += nrec;
        }
        if (alloc_n < ds->count)  // a record (or its label) is missing
            fail(DRB_ERR_IO, "truncated dataset file: " + P);
        cuda_check(cudaMemcpyAsync(ds->labels, ds->host_labels.data(), alloc_n * 4, cudaMemcpyHostToDevice, st),
                   "ds labels h2d");
        cuda_check(cudaStreamSynchronize(st), "ds load");
        // split sidecar (dataset.cpp:129-142)
        std::ifstream split(P + ".split");
        if (split) {
            std::string key;
            uint64_t train = 0, eval = 0;
            if (!(split >> key >> train) || key != "train" || !(split >> key >> eval) || key != "eval" ||
                train + eval != ds->count)
                fail(DRB_ERR_IO, "bad split sidecar: " + P + ".split");
            ds->train = train;
            ds->eval = eval;
        } else {
            ds->train = ds->count;
            ds->eval = 0;
        }
        *out = ds.release();
    });
}

// synth_dataset (proj/src/scenario/dataset.cpp:145-205): the Gaussian-blob dataset, drawn on
// the host with the same double arithmetic and libm, then placed in HBM like a loaded file.
drb_status drb_ds_synth(uint32_t n_classes, uint32_t per_class, uint32_t feature_dim, double separation,
                        uint64_t seed, int32_t device, drb_ds** out) {
    DS_REQUIRE(out);
    return guarded([&] {
        if (!(separation > 0.0))
            fail(DRB_ERR_CONFIG, "synth_dataset: separation must be > 0");
        host_rng rng(seed, 0, kSynth, 0, 0, /*keyed=*/false);
        std::vector<std::vector<double>> means(n_classes, std::vector<double>(feature_dim));
        double min_dist = 0.0;
        do {
            for (auto& mean : means)
                for (auto& v : mean)
                    v = rng.gaussian();
            min_dist = std::numeric_limits<double>::infinity();
            for (uint32_t a = 0; a < n_classes; ++a)
                for (uint32_t b = a + 1; b < n_classes; ++b) {
                    double d2 = 0.0;
                    for (uint32_t f = 0; f < feature_dim; ++f) {
                        const double diff = means[a][f] - means[b][f];
                        d2 += diff * diff;
                    }
                    min_dist = std::min(min_dist, std::sqrt(d2));
                }
        } while (n_classes > 1 && min_dist <= 1e-9);
        if (n_classes > 1) {
            const double scale = separation / min_dist;
            for (auto& mean : means)
                for (auto& v : mean)
                    v *= scale;
        }
        const uint32_t eval_per = per_class / 5, train_per = per_class - eval_per;
        std::unique_ptr<drb_ds> ds(new drb_ds);
        ds->device = device;
        ds->dim = feature_dim;
        ds->n_classes = n_classes;
        ds->train = uint64_t(train_per) * n_classes;
        ds->eval = uint64_t(eval_per) * n_classes;
        ds->count = ds->train + ds->eval;
        std::vector<float> feats;
        feats.reserve(ds->count * feature_dim);
        ds->host_labels.reserve(ds->count);
        for (const uint32_t rows : {train_per, eval_per})  // round-robin over classes per block
            for (uint32_t row = 0; row < rows; ++row)
                for (uint32_t c = 0; c < n_classes; ++c) {
                    for (uint32_t f = 0; f < feature_dim; ++f)
                        feats.push_back(static_cast<float>(means[c][f] + rng.gaussian()));
                    ds->host_labels.push_back(c);
                }
        device_scope g(device);
        cuda_check(cudaMalloc(&ds->features, std::max<uint64_t>(feats.size() * 4, 16)), "ds features");
        cuda_check(cudaMalloc(&ds->labels, std::max<uint64_t>(ds->count * 4, 4)), "ds labels");
        cuda_check(cudaMalloc(&ds->err, 4), "ds err");
        cuda_check(cudaMemset(ds->err, 0, 4), "ds err");
        cuda_check(cudaMemcpy(ds->features, feats.data(), feats.size() * 4, cudaMemcpyHostToDevice), "ds h2d");
        cuda_check(cudaMemcpy(ds->labels, ds->host_labels.data(), ds->count * 4, cudaMemcpyHostToDevice), "ds h2d");
        *out = ds.release();
    });
}

drb_status drb_ds_destroy(drb_ds* ds) {
    delete ds;
    return DRB_OK;
}

drb_status drb_ds_info(const drb_ds* ds, uint64_t* count, uint32_t* feature_dim, uint32_t* n_classes,
                       uint64_t* train_count, uint64_t* eval_count) {
    DS_REQUIRE(ds && count && feature_dim && n_classes && train_count && eval_count);
    *count = ds->count;
    *feature_dim = ds->dim;
    *n_classes = ds->n_classes;
    *train_count = ds->train;
    *eval_count = ds->eval;
    return DRB_OK;
}

drb_status drb_ds_device_views(const drb_ds* ds, void** features, uint32_t** labels) {
    DS_REQUIRE(ds && features && labels);
    *features = ds->features;
    *labels = ds->labels;
    return DRB_OK;
}

drb_status drb_ds_indices_of(const drb_ds* ds, const uint32_t* classes, uint32_t n_classes, int32_t eval,
                             uint64_t* out, uint64_t cap, uint64_t* n_out) {
    DS_REQUIRE(ds && n_out && (classes || n_classes == 0) && (out || cap == 0));
    return guarded([&] {
        const std::unordered_set<uint32_t> wanted(classes, classes + n_classes);
        const uint64_t lo = eval ? ds->train : 0, hi = eval ? ds->count : ds->train;
        uint64_t c = 0;
        for (uint64_t i = lo; i < hi; ++i)
            if (wanted.count(ds->host_labels[i])) {
                if (c < cap)
                    out[c] = i;
                ++c;
            }
        *n_out = c;
    });
}

drb_status drb_ds_gather(const drb_ds* ds, const uint64_t* indices, uint32_t n, void* out_batch,
                         uint32_t* out_labels, void* stream) {
    DS_REQUIRE(ds && (n == 0 || (indices && out_batch)));
    return guarded([&] {
        if (n == 0)
            return;
        device_scope g(ds->device);
        const uint64_t row_bytes = uint64_t(ds->dim) * 4;
        if (row_bytes == 0) {
            if (out_labels)
                ds_gather_kernel<uint32_t, 1><<<1, 32, 0, cudaStream_t(stream)>>>(
                    ds->features, ds->labels, ds->count, 0, indices, n, static_cast<uint8_t*>(out_batch),
                    out_labels, ds->err);
            cuda_check(cudaGetLastError(), "ds gather launch");
            return;
        }
        int sms = 148;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ds->device);
        const bool v16 = row_bytes % 16 == 0 && (reinterpret_cast<uintptr_t>(out_batch) % 16) == 0;
        const uint64_t words = row_bytes / (v16 ? 16 : 4);
        // enough CTAs per row that the batch fills every SM several times over
        // (DRB_GATHER="unroll,ctas_per_sm" overrides the 4,4 default: tools/input_bench.py sweeps)
        static const std::pair<int, int> knobs = [] {
            int u = 4, c = 4;
            if (const char* e = std::getenv("DRB_GATHER"))
                std::sscanf(e, "%d,%d", &u, &c);
            return std::make_pair(u == 2 || u == 8 ? u : 4, c > 0 ? c : 4);
        }();
        const int unroll = knobs.first;
        const uint64_t per_row = std::min<uint64_t>((words + 256 * unroll - 1) / (256 * unroll),
                                                    std::max<uint64_t>(1, (uint64_t(sms) * knobs.second + n - 1) / n));
        dim3 grid(uint32_t(per_row), std::min<uint32_t>(n, 65535));
        auto launch = [&](auto kern) {
            kern<<<grid, 256, 0, cudaStream_t(stream)>>>(ds->features, ds->labels, ds->count, row_bytes, indices, n,
                                                         static_cast<uint8_t*>(out_batch), out_labels, ds->err);
        };
        if (v16)
            unroll == 2 ? launch(ds_gather_kernel<uint4, 2>)
                        : unroll == 8 ? launch(ds_gather_kernel<uint4, 8>) : launch(ds_gather_kernel<uint4, 4>);
        else
            unroll == 2 ? launch(ds_gather_kernel<uint32_t, 2>)
                        : unroll == 8 ? launch(ds_gather_kernel<uint32_t, 8>) : launch(ds_gather_kernel<uint32_t, 4>);
        cuda_check(cudaGetLastError(), "ds gather launch");
    });
}

drb_status drb_ds_device_error(const drb_ds* ds, uint32_t* out) {
    DS_REQUIRE(ds && out);
    return guarded([&] {
        device_scope g(ds->device);
        cuda_check(cudaDeviceSynchronize(), "ds sync");
        cuda_check(cudaMemcpy(out, ds->err, 4, cudaMemcpyDeviceToHost), "ds err read");
        cuda_check(cudaMemset(ds->err, 0, 4), "ds err clear");
    });
}

drb_status drb_make_schedule(uint32_t n_classes, uint32_t n_tasks, uint64_t seed, uint32_t* classes,
                             uint32_t* task_sizes) {
    DS_REQUIRE(classes || n_classes == 0);
    DS_REQUIRE(task_sizes || n_tasks == 0);
    return guarded([&] {
        if (n_tasks == 0 || n_tasks > n_classes)
            fail(DRB_ERR_CONFIG, "make_schedule: need 1 <= T <= K (T=" + std::to_string(n_tasks) +
                                     ", K=" + std::to_string(n_classes) + ")");
        for (uint32_t i = 0; i < n_classes; ++i)
            classes[i] = i;
        host_rng rng(seed, 0, kDataShuffle, 0xabcd, 0);
        for (uint64_t i = n_classes; i > 1; --i)
            std::swap(classes[i - 1], classes[rng.bounded(i)]);
        for (uint32_t t = 0; t < n_tasks; ++t)
            task_sizes[t] = n_classes / n_tasks + (t < n_classes % n_tasks ? 1 : 0);
    });
}

drb_status drb_shard_batches(const uint64_t* task_data, uint64_t n, uint32_t worker, uint32_t n_workers,
                             uint32_t batch_size, uint64_t seed, uint64_t task_index, uint64_t epoch,
                             uint64_t* out, uint64_t cap, uint64_t* n_out) {
    DS_REQUIRE(n_out && (task_data || n == 0) && (out || cap == 0));
    return guarded([&] {
        if (worker >= n_workers)
            fail(DRB_ERR_USAGE, "shard_batches: worker id out of range");
        if (batch_size == 0)
            fail(DRB_ERR_USAGE, "shard_batches: batch_size must be > 0");
        std::vector<uint64_t> order(task_data, task_data + n);
        host_rng rng(seed, 0, kDataShuffle, task_index + 1, epoch + 1);
        for (uint64_t i = order.size(); i > 1; --i)
            std::swap(order[i - 1], order[rng.bounded(i)]);
        uint64_t c = 0;
        for (uint64_t i = worker; i < n; i += n_workers, ++c)
            if (c < cap)
                out[c] = order[i];
        *n_out = c;
    });
}

drb_status drb_lockstep_batches(uint64_t task_size, uint32_t n_workers, uint32_t batch_size, uint64_t* out) {
    DS_REQUIRE(out);
    if (n_workers == 0 || batch_size == 0) {
        drb_b200::set_last_error("lockstep_batches: n_workers and batch_size must be > 0");
        return DRB_ERR_USAGE;
    }
    *out = (task_size / n_workers + batch_size - 1) / batch_size;
    return DRB_OK;
}

}  // extern "C"
