// Cost of reading %globaltimer and of a clock64 read, in SM cycles.
#include <cstdio>
#include <cstdint>
__global__ void k(long long* out, unsigned long long* sink) {
    long long t0 = clock64();
    uint64_t acc = 0;
    for (int i = 0; i < 1000; ++i) {
        uint64_t t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)::"memory");
        acc += t;
    }
    long long t1 = clock64();
    for (int i = 0; i < 1000; ++i) acc += clock64();
    long long t2 = clock64();
    out[0] = t1 - t0; out[1] = t2 - t1;
    sink[0] = acc;
}
int main() {
    long long* d; unsigned long long* s; cudaMalloc(&d, 16); cudaMalloc(&s, 8);
    long long h[2];
    for (int r = 0; r < 2; ++r) { k<<<1, 1>>>(d, s); cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost); }
    printf("globaltimer read: %.1f cycles; clock64: %.1f cycles\n", h[0] / 1000.0, h[1] / 1000.0);
}
