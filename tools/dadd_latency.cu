// Microbenchmark: latency of a chain of dependent DADDs (the bitwise hub row's critical path),
// from registers and from a shared-memory ring read with pipelined LDS.128 (k_long_rows_bitwise's
// adder loop).  One thread; prints cycles per add.
#include <cstdio>
__global__ void k_reg(double* out, double a, int n) {
    double acc = a, b = a * 0.5;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) {
        acc = __dadd_rn(acc, b); acc = __dadd_rn(acc, b); acc = __dadd_rn(acc, b); acc = __dadd_rn(acc, b);
    }
    long long t1 = clock64();
    out[0] = acc;
    out[1] = (double)(t1 - t0) / (4.0 * n);
}
__global__ void k_smem(double* out, int reps) {
    __shared__ __align__(16) double ring[1024];
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) ring[i] = 1.0 + i * 1e-3;
    __syncthreads();
    if (threadIdx.x) return;
    double acc = 0.0;
    const double2* cur = reinterpret_cast<const double2*>(ring);
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
        double2 nx[4];
        for (int j = 0; j < 4; ++j) nx[j] = cur[j];
        for (int i = 0; i + 8 <= 1024; i += 8) {
            double2 v[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) v[j] = nx[j];
            if (i + 16 <= 1024) {
#pragma unroll
                for (int j = 0; j < 4; ++j) nx[j] = cur[(i + 8) / 2 + j];
            }
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                acc = __dadd_rn(acc, v[j].x);
                acc = __dadd_rn(acc, v[j].y);
            }
        }
    }
    long long t1 = clock64();
    out[0] = acc;
    out[1] = (double)(t1 - t0) / (1024.0 * reps);
}
int main() {
    double* d;
    double h[2];
    cudaMalloc(&d, 16);
    k_reg<<<1, 1>>>(d, 1.0, 100000);
    cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    printf("dadd chain from registers: %.2f cycles per add\n", h[1]);
    k_smem<<<1, 256>>>(d, 100);
    cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    printf("dadd chain from a shared-memory ring (pipelined LDS.128): %.2f cycles per add\n", h[1]);
    return 0;
}
