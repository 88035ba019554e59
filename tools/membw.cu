// Microbenchmark: sustained read bandwidth from HBM (buffer >> L2) and from L2 (buffer << L2),
// with 16-byte non-coherent loads and with 1D TMA bulk copies into shared memory.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o membw tools/membw.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void rd_ldg(const uint4* __restrict__ p, size_t n16, int reps, unsigned long long* sink) {
    uint32_t acc = 0;
    for (int r = 0; r < reps; ++r)
        for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n16; i += (size_t)gridDim.x * blockDim.x) {
            uint4 v;
            asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                         : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p + i));
            acc ^= v.x ^ v.y ^ v.z ^ v.w;
        }
    if (acc == 0x12345678u) atomicAdd(sink, 1ull);
}

// Each CTA bulk-copies consecutive 32 KB chunks into a double-buffered smem ring.
__global__ void rd_tma(const char* __restrict__ p, size_t bytes, int reps, unsigned long long* sink) {
    extern __shared__ __align__(128) char smem[];
    __shared__ __align__(8) unsigned long long bar[2];
    const uint32_t CH = 32768;
    if (threadIdx.x == 0) {
        for (int b = 0; b < 2; ++b)
            asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&bar[b])));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    const size_t nch = bytes / CH;
    uint32_t phase[2] = {0, 0};
    uint32_t acc = 0;
    size_t it = 0;
    for (int r = 0; r < reps; ++r) {
        for (size_t c = blockIdx.x; c < nch; c += gridDim.x, ++it) {
            const int b = it & 1;
            if (threadIdx.x == 0) {
                uint32_t sb = (uint32_t)__cvta_generic_to_shared(&bar[b]);
                uint32_t sd = (uint32_t)__cvta_generic_to_shared(smem + b * CH);
                asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(sb), "r"(CH));
                asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                             ::"r"(sd), "l"(p + c * CH), "r"(CH), "r"(sb) : "memory");
            }
            uint32_t sb = (uint32_t)__cvta_generic_to_shared(&bar[b]);
            uint32_t done = 0;
            while (!done)
                asm volatile("{ .reg .pred P; mbarrier.try_wait.parity.shared.b64 P, [%1], %2; selp.u32 %0,1,0,P; }"
                             : "=r"(done) : "r"(sb), "r"(phase[b]));
            phase[b] ^= 1;
            acc ^= ((const uint32_t*)(smem + b * CH))[threadIdx.x];
            __syncthreads();
        }
    }
    if (acc == 0x12345678u) atomicAdd(sink, 1ull);
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const size_t big = 4ull << 30;
    char* buf;
    unsigned long long* sink;
    cudaMalloc(&buf, big);
    cudaMalloc(&sink, 8);
    cudaMemset(buf, 1, big);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaFuncSetAttribute(rd_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
    const size_t sizes[] = {16ull << 20, 32ull << 20, 64ull << 20, 96ull << 20, 4ull << 30};
    for (size_t s : sizes) {
        const int reps = s >= (1ull << 30) ? 3 : 200;
        for (int mode = 0; mode < 2; ++mode) {
            float best = 1e30f;
            for (int trial = 0; trial < 3; ++trial) {
                cudaEventRecord(a);
                if (mode == 0)
                    rd_ldg<<<sms * 8, 512>>>((const uint4*)buf, s / 16, reps, sink);
                else
                    rd_tma<<<sms * 3, 128, 65536>>>(buf, s, reps, sink);
                cudaEventRecord(b);
                cudaEventSynchronize(b);
                float ms;
                cudaEventElapsedTime(&ms, a, b);
                if (ms < best) best = ms;
            }
            printf("%-4s size %7.1f MB  reps %3d  %8.1f GB/s  (%s)\n", mode ? "tma" : "ldg", s / 1e6, reps,
                   (double)s * reps / (best * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
        }
    }
    return 0;
}
