// Probe (tools/, not product): the resident engine's push mechanism in isolation — TMA bulk
// loads of local HBM rows into shared memory, TMA bulk stores of them into a PEER GPU's memory
// over NVLink (the B engines' X_i pushes) — on every SM of GPU 0 into GPU 1.
// One kernel, no cross-GPU waiting, so ncu can capture it (nvltx__bytes / nvlrx__bytes).
// Prints GB/s for row sizes of the BASELINE shapes. Usage: push_bw [MB per launch]
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>

#define CK(x)                                                                 \
    do {                                                                      \
        cudaError_t e_ = (x);                                                 \
        if (e_ != cudaSuccess) {                                              \
            std::printf("%s: %s\n", #x, cudaGetErrorString(e_));              \
            std::exit(1);                                                     \
        }                                                                     \
    } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// each CTA moves rows [blockIdx.x, ... step gridDim.x) of `row` bytes; stages of `stage` bytes
__global__ void push_kernel(const uint8_t* src, uint8_t* dst, uint64_t rows, uint32_t row, uint32_t stage) {
    extern __shared__ __align__(128) uint8_t buf[];
    __shared__ __align__(8) uint64_t bar;
    if (threadIdx.x != 0)
        return;
    asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    uint32_t phase = 0;
    for (uint64_t r = blockIdx.x; r < rows; r += gridDim.x) {
        for (uint32_t off = 0; off < row; off += stage) {
            const uint32_t len = row - off < stage ? row - off : stage;
            asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
            asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(smem_u32(&bar)), "r"(len) : "memory");
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                             smem_u32(buf)),
                         "l"(src + r * row + off), "r"(len), "r"(smem_u32(&bar))
                         : "memory");
            uint32_t done = 0;
            while (!done)
                asm volatile(
                    "{ .reg .pred p; mbarrier.try_wait.parity.shared.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                    : "=r"(done)
                    : "r"(smem_u32(&bar)), "r"(phase)
                    : "memory");
            phase ^= 1;
            asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst + r * row + off),
                         "r"(smem_u32(buf)), "r"(len)
                         : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main(int argc, char** argv) {
    int n = 0;
    CK(cudaGetDeviceCount(&n));
    if (n < 2) {
        std::printf("push_bw: needs 2 GPUs\n");
        return 0;
    }
    const uint64_t mb = argc > 1 ? std::strtoull(argv[1], nullptr, 10) : 512;
    int can = 0;
    CK(cudaDeviceCanAccessPeer(&can, 0, 1));
    CK(cudaSetDevice(1));
    uint8_t* dst = nullptr;
    CK(cudaMalloc(&dst, mb << 20));
    CK(cudaSetDevice(0));
    CK(cudaDeviceEnablePeerAccess(1, 0));
    uint8_t* src = nullptr;
    CK(cudaMalloc(&src, mb << 20));
    CK(cudaMemset(src, 7, mb << 20));
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    const uint32_t stage = 32768;
    CK(cudaFuncSetAttribute(push_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, stage));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    std::printf("peer access %d, %d SMs, %llu MB per launch\n", can, sms, (unsigned long long)mb);
    for (uint32_t row : {12288u, 65536u, 150528u, 301056u}) {  // c1, c5, c2/c3, c4 sample bytes
        const uint64_t rows = (mb << 20) / row;
        push_kernel<<<sms, 32, stage>>>(src, dst, rows, row, stage);  // warm
        CK(cudaEventRecord(e0));
        push_kernel<<<sms, 32, stage>>>(src, dst, rows, row, stage);
        CK(cudaEventRecord(e1));
        CK(cudaDeviceSynchronize());
        float ms = 0;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        std::printf("row %6u B: %.1f GB/s into the peer (%llu rows)\n", row, double(rows) * row / (ms * 1e6),
                    (unsigned long long)rows);
    }
    return 0;
}
