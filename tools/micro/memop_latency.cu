// Probe (tools/, not product): latency of the resident engine's feed mechanics on this GPU.
//  1. ping-pong: stream writes flag=i (cuStreamWriteValue64), a resident 1-thread kernel sees it
//     and writes ack=i, the stream waits ack>=i (cuStreamWaitValue64): per round trip.
//  2. cooperative launch + exit of an empty kernel shaped like the engine (G CTAs x 320 threads,
//     200 KB dynamic smem): per launch, back to back, and one launch alone.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)

__global__ void pong(const volatile unsigned long long* flag, volatile unsigned long long* ack, int n,
                     unsigned long long* stamps) {
    for (int i = 1; i <= n; ++i) {
        unsigned long long v;
        do {
            asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(flag) : "memory");
        } while (v < (unsigned long long)i);
        asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(ack), "l"((unsigned long long)i) : "memory");
    }
}

__global__ void empty_coop() {
    extern __shared__ char sm[];
    if (threadIdx.x == 0) sm[0] = 1;
}

int main(int argc, char** argv) {
    typedef CUresult (*wr_t)(CUstream, CUdeviceptr, cuuint64_t, unsigned int);
    wr_t wr = nullptr, wt = nullptr;
    cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPointByVersion("cuStreamWriteValue64", (void**)&wr, 12000, cudaEnableDefault, &q));
    CK(cudaGetDriverEntryPointByVersion("cuStreamWaitValue64", (void**)&wt, 12000, cudaEnableDefault, &q));
    unsigned long long *flag, *ack;
    CK(cudaMalloc(&flag, 8)); CK(cudaMalloc(&ack, 8));
    CK(cudaMemset(flag, 0, 8)); CK(cudaMemset(ack, 0, 8));
    cudaStream_t sk, s;
    CK(cudaStreamCreateWithFlags(&sk, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    const int n = 2000;
    pong<<<1, 32, 0, sk>>>(flag, ack, n, nullptr);
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
    CK(cudaEventRecord(e0, s));
    for (int i = 1; i <= n; ++i) {
        if (wr(s, (CUdeviceptr)flag, i, 0) != CUDA_SUCCESS) { printf("write failed\n"); return 1; }
        if (wt(s, (CUdeviceptr)ack, i, CU_STREAM_WAIT_VALUE_GEQ) != CUDA_SUCCESS) { printf("wait failed\n"); return 1; }
    }
    CK(cudaEventRecord(e1, s));
    CK(cudaDeviceSynchronize());
    float ms; CK(cudaEventElapsedTime(&ms, e0, e1));
    printf("memop ping-pong: %.2f us per round trip (%d)\n", 1000.0 * ms / n, n);

    // 3. back-to-back stream memory operations on one stream (no kernel involved): GPU time per op
    {
        typedef CUresult (*bt_t)(CUstream, unsigned int, CUstreamBatchMemOpParams*, unsigned int);
        bt_t bt = nullptr;
        CK(cudaGetDriverEntryPointByVersion("cuStreamBatchMemOp", (void**)&bt, 12000, cudaEnableDefault, &q));
        const int m = 2000;
        CK(cudaDeviceSynchronize());
        CK(cudaEventRecord(e0, s));
        for (int i = 1; i <= m; ++i)
            wr(s, (CUdeviceptr)flag, i, 0);
        CK(cudaEventRecord(e1, s));
        CK(cudaDeviceSynchronize());
        CK(cudaEventElapsedTime(&ms, e0, e1));
        printf("writeValue64 back to back: %.3f us per op\n", 1000.0 * ms / m);
        CK(cudaEventRecord(e0, s));
        for (int i = 1; i <= m; ++i)
            wt(s, (CUdeviceptr)flag, 1, CU_STREAM_WAIT_VALUE_GEQ);
        CK(cudaEventRecord(e1, s));
        CK(cudaDeviceSynchronize());
        CK(cudaEventElapsedTime(&ms, e0, e1));
        printf("waitValue64 (already satisfied) back to back: %.3f us per op\n", 1000.0 * ms / m);
        CUstreamBatchMemOpParams op[2];
        memset(op, 0, sizeof op);
        op[0].writeValue.operation = CU_STREAM_MEM_OP_WRITE_VALUE_64;
        op[0].writeValue.address = (CUdeviceptr)ack;
        op[0].writeValue.value64 = 7;
        op[1].waitValue.operation = CU_STREAM_MEM_OP_WAIT_VALUE_64;
        op[1].waitValue.address = (CUdeviceptr)flag;
        op[1].waitValue.value64 = 1;
        op[1].waitValue.flags = CU_STREAM_WAIT_VALUE_GEQ;
        CK(cudaEventRecord(e0, s));
        for (int i = 1; i <= m; ++i)
            bt(s, 2, op, 0);
        CK(cudaEventRecord(e1, s));
        CK(cudaDeviceSynchronize());
        CK(cudaEventElapsedTime(&ms, e0, e1));
        printf("batch [write, satisfied wait] back to back: %.3f us per batch\n", 1000.0 * ms / m);
    }
    int sms; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    CK(cudaFuncSetAttribute(empty_coop, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    for (int G : {76, 148}) {
        if (G > sms) continue;
        cudaLaunchConfig_t cfg{}; cfg.gridDim = dim3(G); cfg.blockDim = dim3(320); cfg.dynamicSmemBytes = 200 * 1024; cfg.stream = s;
        cudaLaunchAttribute a[1]; a[0].id = cudaLaunchAttributeCooperative; a[0].val.cooperative = 1; cfg.attrs = a; cfg.numAttrs = 1;
        for (int w = 0; w < 10; ++w) CK(cudaLaunchKernelEx(&cfg, empty_coop));
        CK(cudaDeviceSynchronize());
        CK(cudaEventRecord(e0, s));
        for (int w = 0; w < 200; ++w) CK(cudaLaunchKernelEx(&cfg, empty_coop));
        CK(cudaEventRecord(e1, s));
        CK(cudaDeviceSynchronize());
        CK(cudaEventElapsedTime(&ms, e0, e1));
        float one = 0;
        for (int w = 0; w < 20; ++w) {
            CK(cudaEventRecord(e0, s)); CK(cudaLaunchKernelEx(&cfg, empty_coop)); CK(cudaEventRecord(e1, s));
            CK(cudaDeviceSynchronize()); float t; CK(cudaEventElapsedTime(&t, e0, e1)); one += t;
        }
        printf("coop launch G=%d 320thr 200KB: %.2f us back-to-back, %.2f us alone\n", G, 1000.0 * ms / 200, 1000.0 * one / 20);
    }
    return 0;
}
