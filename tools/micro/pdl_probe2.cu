// PDL with extra cross-stream graph edges: main-stream kernel i (PDL attribute) also waits
// on a side-stream kernel's event. Does the programmatic overlap survive?
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

__device__ uint64_t gt() { uint64_t t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; }

__global__ void k(unsigned long long* st, int idx, uint64_t spin_ns) {
    extern __shared__ uint8_t sm[];
    if (threadIdx.x == 0) atomicMin(&st[2 * idx], (unsigned long long)gt());
    asm volatile("griddepcontrol.launch_dependents;");
    asm volatile("griddepcontrol.wait;" ::: "memory");
    uint64_t t0 = gt();
    while (gt() - t0 < spin_ns) {}
    sm[threadIdx.x] = 1;
    __syncthreads();
    if (threadIdx.x == 0) atomicMax(&st[2 * idx + 1], (unsigned long long)gt());
}
__global__ void side(uint64_t spin_ns) {
    extern __shared__ uint8_t sm[];
    uint64_t t0 = gt();
    while (gt() - t0 < spin_ns) {}
    sm[threadIdx.x] = 1;
}

int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    unsigned long long* st; cudaMalloc(&st, 64 * 16);
    const size_t smem = 100 * 1024, side_smem = 130 * 1024;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    cudaFuncSetAttribute(side, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)side_smem);
    cudaFuncSetAttribute(side, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    // mode 0: no side deps; 1: side dep right before each PDL launch; 2: side dep placed one
    // launch early (prewait); 3: side events recorded after each main kernel + waited by side
    for (int mode : {0, 1, 2, 3}) {
        std::vector<unsigned long long> init(64 * 2);
        for (int i = 0; i < 64; ++i) { init[2 * i] = ~0ull; init[2 * i + 1] = 0; }
        cudaMemcpy(st, init.data(), 64 * 16, cudaMemcpyHostToDevice);
        cudaStream_t s, b; cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking); cudaStreamCreateWithFlags(&b, cudaStreamNonBlocking);
        cudaEvent_t ev[32], evm[32];
        for (int i = 0; i < 32; ++i) { cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming); cudaEventCreateWithFlags(&evm[i], cudaEventDisableTiming); }
        cudaGraph_t g; cudaGraphExec_t ge;
        cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
        cudaEventRecord(evm[31], s); cudaStreamWaitEvent(b, evm[31], 0);
        const int n = 12;
        for (int i = 0; i < n; ++i) { side<<<1, 64, side_smem, b>>>(1000); cudaEventRecord(ev[i], b); }
        for (int i = 0; i < n; ++i) {
            if (mode == 1) cudaStreamWaitEvent(s, ev[i], 0);
            if (mode == 2 && i == 0) cudaStreamWaitEvent(s, ev[0], 0);
            if (mode == 2 && i + 1 < n) cudaStreamWaitEvent(s, ev[i + 1], 0);
            cudaLaunchConfig_t cfg{}; cfg.gridDim = dim3(sms - 2); cfg.blockDim = dim3(64);
            cfg.dynamicSmemBytes = smem; cfg.stream = s;
            cudaLaunchAttribute a[1]; a[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
            a[0].val.programmaticStreamSerializationAllowed = 1;
            cfg.attrs = a; cfg.numAttrs = i > 0 ? 1 : 0;
            cudaLaunchKernelEx(&cfg, k, st, i, (uint64_t)3000);
            if (mode == 3) { cudaEventRecord(evm[i], s); }
        }
        cudaEventRecord(evm[30], b); cudaStreamWaitEvent(s, evm[30], 0);
        cudaError_t e1 = cudaStreamEndCapture(s, &g);
        cudaError_t e2 = cudaGraphInstantiate(&ge, g, 0);
        cudaGraphLaunch(ge, s);
        cudaStreamSynchronize(s);
        cudaError_t e = cudaGetLastError();
        cudaMemcpy(init.data(), st, 64 * 16, cudaMemcpyDeviceToHost);
        printf("mode %d err %d/%d/%d:", mode, (int)e1, (int)e2, (int)e);
        for (int i = 1; i < n; ++i)
            printf(" %+.2f", ((long long)init[2 * i] - (long long)init[2 * i - 1]) / 1e3);
        printf("\n");
    }
    return 0;
}
