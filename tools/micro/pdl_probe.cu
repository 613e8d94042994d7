// PDL co-residency probe: does a programmatically launched secondary start while the
// primary (one CTA per SM, ~100 KB smem each) still runs? Prints per-launch start/end.
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o pdl_probe pdl_probe.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

__device__ uint64_t gt() { uint64_t t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; }

__global__ void k(unsigned long long* st, int idx, uint64_t spin_ns, int trig) {
    extern __shared__ uint8_t sm[];
    if (threadIdx.x == 0) atomicMin(&st[2 * idx], (unsigned long long)gt());
    if (trig) asm volatile("griddepcontrol.launch_dependents;");
    asm volatile("griddepcontrol.wait;" ::: "memory");
    uint64_t t0 = gt();
    while (gt() - t0 < spin_ns) {}
    sm[threadIdx.x] = 1;
    __syncthreads();
    if (threadIdx.x == 0) atomicMax(&st[2 * idx + 1], (unsigned long long)gt());
}

int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    unsigned long long* st; cudaMalloc(&st, 64 * 16);
    for (int smemkb : {100, 60, 0}) for (int graph : {0, 1}) for (int pre_spin : {0, 1}) {
        size_t smem = smemkb * 1024;
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
        int occ = 0; cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, 64, smem);
        std::vector<unsigned long long> init(64 * 2);
        for (int i = 0; i < 64; ++i) { init[2 * i] = ~0ull; init[2 * i + 1] = 0; }
        cudaMemcpy(st, init.data(), 64 * 16, cudaMemcpyHostToDevice);
        cudaStream_t s; cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
        cudaGraph_t g; cudaGraphExec_t ge;
        if (graph) cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
        for (int i = 0; i < 8; ++i) {
            cudaLaunchConfig_t cfg{}; cfg.gridDim = dim3(sms - 2); cfg.blockDim = dim3(64);
            cfg.dynamicSmemBytes = smem; cfg.stream = s;
            cudaLaunchAttribute a[1]; a[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
            a[0].val.programmaticStreamSerializationAllowed = 1;
            cfg.attrs = a; cfg.numAttrs = i > 0 ? 1 : 0;
            cudaLaunchKernelEx(&cfg, k, st, i, (uint64_t)(pre_spin ? 5000 : 2000), 1);
        }
        if (graph) { cudaStreamEndCapture(s, &g); cudaGraphInstantiate(&ge, g, 0); cudaGraphLaunch(ge, s); }
        cudaStreamSynchronize(s);
        cudaError_t e = cudaGetLastError();
        cudaMemcpy(init.data(), st, 64 * 16, cudaMemcpyDeviceToHost);
        printf("smem %3d KB occ/SM %d graph %d spin %d err %d:", smemkb, occ, graph, pre_spin ? 5000 : 2000, (int)e);
        for (int i = 1; i < 8; ++i)
            printf(" [start-prevend %+.2f]", ((long long)init[2 * i] - (long long)init[2 * i - 1]) / 1e3);
        printf("\n");
    }
    return 0;
}
