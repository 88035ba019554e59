// Microbenchmark: throughput of a single global ticket counter claimed by one lane per warp
// (atomicAdd), with and without work between claims, and with claims spread over S counters.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/atomic_rate tools/atomic_rate.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

__global__ void claim(uint32_t* ctr, uint32_t n, uint32_t streams, uint32_t work_ns, uint32_t* sink) {
    const uint32_t lane = threadIdx.x & 31u;
    const uint32_t gw = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    uint32_t* c = ctr + (gw % streams) * 32;  // one 128-B line per stream
    uint32_t acc = 0;
    for (;;) {
        uint32_t t = 0;
        if (lane == 0) t = atomicAdd(c, 1u);
        t = __shfl_sync(0xffffffffu, t, 0);
        if (t * streams >= n) break;
        acc += t;
        if (work_ns) __nanosleep(work_ns);
    }
    if (acc == 0xdeadbeefu) sink[0] = acc;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    uint32_t *ctr, *sink;
    cudaMalloc(&ctr, 64 * 128);
    cudaMalloc(&sink, 4);
    const uint32_t n = 8u << 20;
    for (uint32_t streams : {1u, 4u, 16u, 64u})
        for (uint32_t work : {0u, 1000u}) {
            cudaMemset(ctr, 0, 64 * 128);
            cudaEvent_t a, b;
            cudaEventCreate(&a);
            cudaEventCreate(&b);
            cudaEventRecord(a);
            claim<<<sms * 4, 256>>>(ctr, n, streams, work, sink);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms = 0;
            cudaEventElapsedTime(&ms, a, b);
            printf("streams %2u work %4u ns: %u claims in %8.3f ms = %7.1f claims/us\n", streams, work, n, ms,
                   n / (ms * 1e3));
        }
    return 0;
}
