// Microbenchmark: latency of warp_select / warp_assign / warp_plan_draw with cold vs warm
// instruction cache (iteration 0 vs later). Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/micro/select_bench tools/micro/select_bench.cu
#include "../../paper_2406_03285_b200/csrc/drb_kernels.cu"
#include <cstdio>

using namespace drb_b200;

__global__ void bench(long long* out, uint32_t n, uint32_t k, uint32_t cap, uint32_t K) {
    __shared__ uint32_t sel[256], idx[256], lab[256], occ[1024], cl[256], cs[256], kind[256], scr[64], acc[64];
    for (uint32_t i = threadIdx.x; i < n; i += 32) lab[i] = (i * 7) % K;
    for (uint32_t i = threadIdx.x; i < K; i += 32) occ[i] = cap;
    __syncwarp();
    uint64_t ctr = 0, ectr = 0, sctr = 0;
    for (int it = 0; it < 8; ++it) {
        long long t0 = clock64();
        warp_select(0x1234567ull, ctr, n, k, sel, idx);
        long long t1 = clock64();
        uint32_t app = 0;
        warp_assign(0x7654321ull, ectr, cap, k, sel, lab, occ, cl, cs, scr, kind, app);
        long long t2 = clock64();
        uint32_t c = warp_plan_draw(0x9999ull, sctr, 7, 4800, acc);
        long long t3 = clock64();
        if (threadIdx.x == 0) {
            out[it * 4 + 0] = t1 - t0; out[it * 4 + 1] = t2 - t1; out[it * 4 + 2] = t3 - t2; out[it * 4 + 3] = c + app;
        }
        for (uint32_t i = threadIdx.x; i < K; i += 32) occ[i] = cap;
        __syncwarp();
    }
}

int main() {
    long long* d; cudaMalloc(&d, 64 * 8);
    long long h[64];
    for (int rep = 0; rep < 2; ++rep) {
        bench<<<1, 32>>>(d, 56, 14, 48, 100);
        cudaMemcpy(h, d, 64 * 8, cudaMemcpyDeviceToHost);
        printf("launch %d (cycles): ", rep);
        for (int it = 0; it < 8; ++it) printf("[sel %lld asg %lld plan %lld] ", h[it * 4], h[it * 4 + 1], h[it * 4 + 2]);
        printf("\n");
    }
    return 0;
}
