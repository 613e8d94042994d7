// update_bench — the drop-in trainer call (proj/src/trainer/trainer.cpp:109-113,
// `reps = engine.update(m); m' = augment(m, reps)`) timed through the C++ facade, as the
// reference's own C++ trainer would make it: K calls of engine::update at the BASELINE c2
// shape (224x224x3 u8, K=100, cap 48, b=56, r=7, c=14), inputs resident in HBM, device-timed
// with CUDA events on the consuming stream.
//   serial: update(m_i, stream) on one stream — each post follows the wait for m'_{i-1}
//   split:  update(m_i, loader, trainer) — posts on the loader stream run ahead, the trainer
//           stream releases the m' it used and waits for m'_i (drb_rb_step_split)
// Prints one JSON line. Built by __graft_entry__.build(); run by bench.py.
#include <cuda_runtime.h>

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "drb_rb.hpp"

using namespace drb::b200;

#define CK(x)                                                                          \
    do {                                                                               \
        cudaError_t e_ = (x);                                                          \
        if (e_ != cudaSuccess) {                                                       \
            std::fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e_));              \
            std::exit(2);                                                              \
        }                                                                              \
    } while (0)

int main(int argc, char** argv) {
    const int steps = argc > 1 ? std::atoi(argv[1]) : 200;
    const int device = argc > 2 ? std::atoi(argv[2]) : 0;
    const uint32_t aug_ring = argc > 3 ? uint32_t(std::atoi(argv[3])) : 0;  // 0: the default (32 slots)
    CK(cudaSetDevice(device));
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
    const uint32_t K = 100, cap = 48, b = 56, r = 7, c = 14, ring = 64;
    const uint64_t S = 224 * 224 * 3;
    drb_rb_config cfg{};
    cfg.n_classes = K;
    cfg.per_class_cap = cap;
    cfg.sample_bytes = S;
    cfg.max_batch = b;
    cfg.candidate_count = c;
    cfg.rep_count = r;
    cfg.rank = 0;
    cfg.world = 1;
    cfg.seed = 1;
    cfg.device = device;
    cfg.engine_ctas = uint32_t(sms);  // no training step to share the SMs with
    cfg.aug_ring = aug_ring;          // split form: the loader runs up to aug_ring - 2 steps ahead
    rehearsal_buffer buf(cfg);
    engine eng(buf);
    eng.start();
    // device ring: a byte pattern per batch, labels cycling over the classes
    uint8_t* data = nullptr;
    uint32_t* labels = nullptr;
    CK(cudaMalloc(&data, uint64_t(ring) * b * S));
    CK(cudaMalloc(&labels, uint64_t(ring) * b * 4));
    std::vector<uint32_t> hl(uint64_t(ring) * b);
    for (size_t x = 0; x < hl.size(); ++x)
        hl[x] = uint32_t((x * 2654435761u) % K);
    CK(cudaMemcpy(labels, hl.data(), hl.size() * 4, cudaMemcpyHostToDevice));
    for (uint32_t j = 0; j < ring; ++j)
        CK(cudaMemset(data + uint64_t(j) * b * S, int(j * 37 + 11), uint64_t(b) * S));
    cudaStream_t loader, trainer;
    CK(cudaStreamCreateWithFlags(&loader, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&trainer, cudaStreamNonBlocking));
    auto batch = [&](int k) {
        const uint32_t j = uint32_t(k) % ring;
        return device_batch{data + uint64_t(j) * b * S, labels + uint64_t(j) * b, b};
    };
    const int prefill = std::getenv("UB_PREFILL") ? std::atoi(std::getenv("UB_PREFILL")) : 400;
    for (int k = 0; k < prefill; ++k)  // fill every class to capacity (replacements from here)
        eng.update(batch(k), loader, trainer);
    CK(cudaDeviceSynchronize());
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    // UB_TRACE=1: an event after every step's wait, per-step times by step range on stderr
    const bool trace = std::getenv("UB_TRACE") != nullptr;
    std::vector<cudaEvent_t> evs;
    auto timed = [&](bool split, int n, double* host_us) {
        CK(cudaDeviceSynchronize());
        if (trace)
            while (evs.size() < size_t(n))
                CK(cudaEventCreate(&evs.emplace_back()));
        CK(cudaEventRecord(e0, trainer));
        if (split)
            CK(cudaStreamWaitEvent(loader, e0, 0));
        const auto t0 = std::chrono::steady_clock::now();
        for (int k = 0; k < n; ++k) {
            if (split)
                eng.update(batch(k), loader, trainer);
            else
                eng.update(batch(k), trainer);
            if (trace)
                CK(cudaEventRecord(evs[k], trainer));
        }
        if (trace) {
            CK(cudaDeviceSynchronize());
            int lo = 0;
            for (int hi : {1, 5, 20, 50, 100, 200, 400, 800, 1600, 3200}) {
                if (hi > n)
                    hi = n;
                if (hi <= lo)
                    break;
                float ms = 0;
                CK(cudaEventElapsedTime(&ms, lo ? evs[lo - 1] : e0, evs[hi - 1]));
                std::fprintf(stderr, "%s steps [%d,%d): %.2f us/step\n", split ? "split" : "serial", lo, hi,
                             1000.0 * ms / (hi - lo));
                lo = hi;
            }
        }
        *host_us = std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count() / n;
        CK(cudaEventRecord(e1, trainer));
        CK(cudaDeviceSynchronize());
        float ms = 0;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        return 1000.0 * ms / n;
    };
    double h_split = 0, h_serial = 0, h_split20 = 0, h_serial20 = 0;
    const double split = timed(true, steps, &h_split);
    const double serial = timed(false, steps, &h_serial);
    const double split20 = timed(true, 20, &h_split20);
    const double serial20 = timed(false, 20, &h_serial20);
    eng.shutdown();
    std::printf("{\"split_us_per_step\": %.3f, \"serial_us_per_step\": %.3f, \"split_us_per_step_20\": %.3f, "
                "\"serial_us_per_step_20\": %.3f, \"host_us_per_call_split\": %.3f, \"host_us_per_call_serial\": %.3f, "
                "\"steps\": %d, \"engine_ctas\": %d, \"aug_ring\": %u}\n",
                split, serial, split20, serial20, h_split, h_serial, steps, sms, aug_ring ? aug_ring : 32u);
    cudaFree(data);
    cudaFree(labels);
    return 0;
}
