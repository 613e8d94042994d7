// C++ facade test (host code in C++ over the C ABI): the reference's engine loop
//   reps = engine.update(m); m' = augment(m, reps)
// written against include/drb_rb.hpp, checked bit-exactly against the C oracle's replay
// (oracle/drb_oracle.c, itself pinned to the reference). Also the reference buffer-test
// idioms (usage errors, KAT values). Exit code 0 = pass. Needs a GPU.
#include <cuda_runtime.h>

#include <cstdio>
#include <cstring>
#include <random>
#include <vector>

#include "../../include/drb_rb.hpp"
#include "../../oracle/drb_oracle.h"

using namespace drb::b200;

#define EXPECT(cond)                                                                \
    do {                                                                            \
        if (!(cond)) {                                                              \
            std::fprintf(stderr, "FAILED %s:%d: %s\n", __FILE__, __LINE__, #cond); \
            return 1;                                                               \
        }                                                                           \
    } while (0)

int main() {
    // KAT1 / KAT3 through the facade
    rng_stream kat(1, 0, rng_stream::purpose::candidate_selection);
    EXPECT(kat.next_u64() == 0x825944e4c99d3327ull);
    rng_stream kat3(1, 0, rng_stream::purpose::candidate_selection);
    auto sel = sample_without_replacement(64, 14, kat3);
    const std::uint32_t want3[14] = {39, 22, 63, 46, 43, 26, 56, 11, 20, 49, 32, 45, 57, 44};
    EXPECT(sel.size() == 14 && std::memcmp(sel.data(), want3, sizeof want3) == 0);

    const std::uint32_t K = 10, cap = 6, b = 32, c = 14, r = 8;
    const std::uint64_t S = 1024, seed = 9;
    rehearsal_buffer buf(K, cap, S, b, c, r, seed);
    engine eng(buf);
    bool threw = false;
    try {
        eng.update(device_batch{});
    } catch (const usage_error&) {  // update before start (engine.cpp:63-66)
        threw = true;
    }
    EXPECT(threw);
    eng.start();

    void* d_batch = nullptr;
    std::uint32_t* d_labels = nullptr;
    cudaMalloc(&d_batch, b * S);
    cudaMalloc(&d_labels, b * 4);
    void* rp = or_replay_create(1, K, cap, S, c, r, seed);
    std::mt19937 gen(1234);
    std::vector<std::uint8_t> batch(b * S), out((b + r) * S), got((b + r) * S);
    std::vector<std::uint32_t> labels(b), out_l(b + r), got_l(b + r), cnt(1);
    for (int i = 0; i < 60; ++i) {
        for (auto& x : batch)
            x = static_cast<std::uint8_t>(gen());
        for (auto& l : labels)
            l = gen() % K;
        cudaMemcpy(d_batch, batch.data(), b * S, cudaMemcpyHostToDevice);
        cudaMemcpy(d_labels, labels.data(), b * 4, cudaMemcpyHostToDevice);
        EXPECT(or_replay_step(rp, batch.data(), labels.data(), b, out.data(), out_l.data(), cnt.data()) == 0);
        augmented_batch aug = eng.update(device_batch{d_batch, d_labels, b});
        const std::uint32_t rows = aug.count();
        EXPECT(rows == cnt[0]);
        cudaMemcpy(got.data(), aug.data(), rows * S, cudaMemcpyDeviceToHost);
        cudaMemcpy(got_l.data(), aug.labels(), rows * 4, cudaMemcpyDeviceToHost);
        EXPECT(std::memcmp(got.data(), out.data(), rows * S) == 0);
        EXPECT(std::memcmp(got_l.data(), out_l.data(), rows * 4) == 0);
    }
    eng.shutdown();
    threw = false;
    try {
        eng.update(device_batch{d_batch, d_labels, b});
    } catch (const usage_error&) {  // update after shutdown
        threw = true;
    }
    EXPECT(threw);
    or_replay_destroy(rp);
    cudaFree(d_batch);
    cudaFree(d_labels);
    std::printf("facade_parity: 60 iterations bit-exact vs oracle\n");
    return 0;
}
