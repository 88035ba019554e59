// Microbenchmark (experiments only): how many independent 8-byte coalesced gathers a warp keeps in
// flight with each load flavour.  Each warp repeatedly issues NB loads x[base_j + lane] (bases
// pseudo-random inside a window that fits L2), sums them, and moves on.  Prints ns per batch per warp.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/ldrate tools/ldrate.cu && build/ldrate
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int MODE>
__device__ __forceinline__ double ld(const double* p) {
    double v;
    if (MODE == 0) asm volatile("ld.global.ca.f64 %0, [%1];" : "=d"(v) : "l"(p));
    else if (MODE == 1) v = *p;
    else if (MODE == 2) asm volatile("ld.global.cg.f64 %0, [%1];" : "=d"(v) : "l"(p));
    else if (MODE == 3) asm volatile("ld.relaxed.gpu.global.f64 %0, [%1];" : "=d"(v) : "l"(p));
    else if (MODE == 4) asm volatile("ld.weak.global.f64 %0, [%1];" : "=d"(v) : "l"(p));
    else asm volatile("ld.global.nc.f64 %0, [%1];" : "=d"(v) : "l"(p));
    return v;
}

template <int MODE, int NB>
__global__ void __launch_bounds__(256) k(const double* __restrict__ x, uint64_t n, int iters, double* out) {
    const uint32_t lane = threadIdx.x & 31, gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    uint64_t s = gw * 0x9E3779B97F4A7C15ull + 12345;
    double acc = 0.0;
    for (int it = 0; it < iters; ++it) {
        double v[NB];
#pragma unroll
        for (int j = 0; j < NB; ++j) {
            s = s * 6364136223846793005ull + 1442695040888963407ull;
            const uint64_t b = (s >> 20) & (n - 1 - 64) & ~63ull | ((s >> 50) & 7);
            v[j] = ld<MODE>(x + b + lane);
        }
#pragma unroll
        for (int j = 0; j < NB; ++j) acc += v[j];
    }
    if (acc == 1.2345) out[0] = acc;
}

template <int MODE, int NB>
void run(const char* name, const double* x, uint64_t n, int ctas_per_sm, double* out) {
    int sms = 148;
    const int iters = 2000;
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    k<MODE, NB><<<sms * ctas_per_sm, 256>>>(x, n, 100, out);
    cudaEventRecord(a);
    k<MODE, NB><<<sms * ctas_per_sm, 256>>>(x, n, iters, out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    const double bytes = (double)sms * ctas_per_sm * 8 * iters * NB * 256.0;
    printf("%-12s NB=%2d warps/SM=%2d: %7.1f ns per batch per warp, %6.2f TB/s\n", name, NB, ctas_per_sm * 8,
           ms * 1e6 / iters, bytes / (ms * 1e-3) * 1e-12);
}

int main() {
    const uint64_t n = 8ull << 20;  // 64 MB window: L2 resident
    double *x, *out;
    cudaMalloc(&x, n * 8); cudaMalloc(&out, 8);
    cudaMemset(x, 0, n * 8);
    for (int c : {4, 2}) {
        run<0, 7>("ld.ca", x, n, c, out);   run<0, 14>("ld.ca", x, n, c, out);
        run<1, 7>("plain", x, n, c, out);   run<1, 14>("plain", x, n, c, out);
        run<2, 7>("ld.cg", x, n, c, out);   run<2, 14>("ld.cg", x, n, c, out);
        run<3, 7>("relaxed.gpu", x, n, c, out); run<3, 14>("relaxed.gpu", x, n, c, out);
        run<4, 7>("ld.weak", x, n, c, out); run<4, 14>("ld.weak", x, n, c, out);
        run<5, 7>("ld.nc", x, n, c, out);   run<5, 14>("ld.nc", x, n, c, out);
    }
    return 0;
}
