// Microbenchmark: throughput of SpMV row-engine variants over SELL-32 storage of a 7-point 3D
// Laplacian, L2-resident (small grid, R sweeps in one launch) versus HBM-streamed (large grid).
// Answers: can a row engine consume matrix data from L2 faster than from HBM?  Without that,
// cross-power L2 reuse cannot speed the MPK up.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -o tools/rowengine tools/rowengine.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                   \
    do {                                                                        \
        cudaError_t e = (x);                                                    \
        if (e != cudaSuccess) {                                                 \
            fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); \
            exit(1);                                                            \
        }                                                                       \
    } while (0)

__device__ __forceinline__ uint2 ldu2(const uint2* p) {
    uint2 r;
    asm volatile("ld.global.nc.L1::no_allocate.v2.u32 {%0,%1}, [%2];" : "=r"(r.x), "=r"(r.y) : "l"(p));
    return r;
}
__device__ __forceinline__ double2 ldd2(const double2* p) {
    double2 r;
    asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0,%1}, [%2];" : "=d"(r.x), "=d"(r.y) : "l"(p));
    return r;
}
__device__ __forceinline__ uint32_t ldu(const uint32_t* p) {
    uint32_t r;
    asm volatile("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(r) : "l"(p));
    return r;
}
__device__ __forceinline__ double ldd(const double* p) {
    double r;
    asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(r) : "l"(p));
    return r;
}

// Fixed-width SELL-8 pair layout like rowdot.cuh (every chunk width 8 here: 7-point rows padded):
// entry (lane, k) at chunk*256 + (k/2)*64 + lane*2 + k%2.
struct M {
    const uint32_t* cols;
    const double* vals;
    const uint32_t* len;
    uint32_t n;
};

// V0: one row per thread, metadata -> 4 pair loads -> 8 gathers -> sum (the k_spmv_sell shape).
__global__ void __launch_bounds__(256) v0(M A, const double* __restrict__ x, double* y, int reps) {
    for (int r = 0; r < reps; ++r)
        for (uint32_t s = blockIdx.x * blockDim.x + threadIdx.x; s < A.n; s += gridDim.x * blockDim.x) {
            const uint32_t len = A.len[s];
            const uint64_t off = (uint64_t)(s >> 5) * 256 + (s & 31) * 2;
            uint32_t c[8];
            double v[8];
#pragma unroll
            for (int j = 0; j < 8; j += 2) {
                uint2 t = ldu2((const uint2*)(A.cols + off + j * 32));
                double2 w = ldd2((const double2*)(A.vals + off + j * 32));
                c[j] = t.x, c[j + 1] = t.y, v[j] = w.x, v[j + 1] = w.y;
            }
            double xv[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) xv[j] = j < (int)len ? __ldg(x + c[j]) : 0.0;
            double acc = 0.0;
#pragma unroll
            for (int j = 0; j < 8; ++j)
                if (j < (int)len) acc = __dadd_rn(acc, __dmul_rn(v[j], xv[j]));
            y[s] = acc;
        }
}

// V1: software-pipelined across rows: the next row's matrix entries load while this row's
// gathers are in flight.
__global__ void __launch_bounds__(256) v1(M A, const double* __restrict__ x, double* y, int reps) {
    const uint32_t stride = gridDim.x * blockDim.x;
    for (int r = 0; r < reps; ++r) {
        uint32_t s = blockIdx.x * blockDim.x + threadIdx.x;
        if (s >= A.n) continue;
        uint32_t c[8], len = A.len[s];
        double v[8];
        uint64_t off = (uint64_t)(s >> 5) * 256 + (s & 31) * 2;
#pragma unroll
        for (int j = 0; j < 8; j += 2) {
            uint2 t = ldu2((const uint2*)(A.cols + off + j * 32));
            double2 w = ldd2((const double2*)(A.vals + off + j * 32));
            c[j] = t.x, c[j + 1] = t.y, v[j] = w.x, v[j + 1] = w.y;
        }
        for (;;) {
            double xv[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) xv[j] = j < (int)len ? __ldg(x + c[j]) : 0.0;
            const uint32_t sn = s + stride;
            uint32_t cn[8], lenn = 0;
            double vn[8];
            if (sn < A.n) {
                lenn = A.len[sn];
                const uint64_t o = (uint64_t)(sn >> 5) * 256 + (sn & 31) * 2;
#pragma unroll
                for (int j = 0; j < 8; j += 2) {
                    uint2 t = ldu2((const uint2*)(A.cols + o + j * 32));
                    double2 w = ldd2((const double2*)(A.vals + o + j * 32));
                    cn[j] = t.x, cn[j + 1] = t.y, vn[j] = w.x, vn[j + 1] = w.y;
                }
            }
            double acc = 0.0;
#pragma unroll
            for (int j = 0; j < 8; ++j)
                if (j < (int)len) acc = __dadd_rn(acc, __dmul_rn(v[j], xv[j]));
            y[s] = acc;
            if (sn >= A.n) break;
            s = sn;
            len = lenn;
#pragma unroll
            for (int j = 0; j < 8; ++j) c[j] = cn[j], v[j] = vn[j];
        }
    }
}

// V2: two rows per thread at once (independent chains).
__global__ void __launch_bounds__(256) v2(M A, const double* __restrict__ x, double* y, int reps) {
    const uint32_t stride = gridDim.x * blockDim.x;
    for (int r = 0; r < reps; ++r)
        for (uint32_t s0 = blockIdx.x * blockDim.x + threadIdx.x; s0 < A.n; s0 += 2 * stride) {
            uint32_t c[2][8], len[2];
            double v[2][8], xv[2][8];
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const uint32_t s = s0 + h * stride;
                len[h] = s < A.n ? A.len[s] : 0;
                const uint64_t off = (uint64_t)(s >> 5) * 256 + (s & 31) * 2;
#pragma unroll
                for (int j = 0; j < 8; j += 2) {
                    uint2 t = s < A.n ? ldu2((const uint2*)(A.cols + off + j * 32)) : make_uint2(0, 0);
                    double2 w = s < A.n ? ldd2((const double2*)(A.vals + off + j * 32)) : make_double2(0, 0);
                    c[h][j] = t.x, c[h][j + 1] = t.y, v[h][j] = w.x, v[h][j + 1] = w.y;
                }
            }
#pragma unroll
            for (int h = 0; h < 2; ++h)
#pragma unroll
                for (int j = 0; j < 8; ++j) xv[h][j] = j < (int)len[h] ? __ldg(x + c[h][j]) : 0.0;
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                double acc = 0.0;
#pragma unroll
                for (int j = 0; j < 8; ++j)
                    if (j < (int)len[h]) acc = __dadd_rn(acc, __dmul_rn(v[h][j], xv[h][j]));
                if (s0 + h * stride < A.n) y[s0 + h * stride] = acc;
            }
        }
}

// V3: pure stream of the matrix arrays (no gathers): the bytes-only ceiling of the layout.
__global__ void __launch_bounds__(256) v3(M A, const double* __restrict__ x, double* y, int reps) {
    for (int r = 0; r < reps; ++r)
        for (uint32_t s = blockIdx.x * blockDim.x + threadIdx.x; s < A.n; s += gridDim.x * blockDim.x) {
            const uint64_t off = (uint64_t)(s >> 5) * 256 + (s & 31) * 2;
            double acc = 0.0;
            uint32_t ci = 0;
#pragma unroll
            for (int j = 0; j < 8; j += 2) {
                uint2 t = ldu2((const uint2*)(A.cols + off + j * 32));
                double2 w = ldd2((const double2*)(A.vals + off + j * 32));
                ci ^= t.x ^ t.y;
                acc += w.x + w.y;
            }
            y[s] = acc + (double)(ci & 1);
        }
}

int main(int argc, char** argv) {
    int dev_sms = 0;
    CK(cudaDeviceGetAttribute(&dev_sms, cudaDevAttrMultiProcessorCount, 0));
    for (int ai = 1; ai < argc; ++ai) {
        const int m = atoi(argv[ai]);
        const uint32_t n = (uint32_t)m * m * m;
        const uint32_t nch = (n + 31) / 32, ns = nch * 32;
        std::vector<uint32_t> cols((size_t)nch * 256, 0), len(ns, 0);
        std::vector<double> vals((size_t)nch * 256, 0.0);
        for (uint32_t r = 0; r < n; ++r) {
            const int X = r % m, Y = (r / m) % m, Z = r / (m * m);
            uint32_t k = 0;
            auto put = [&](uint32_t c, double v) {
                const size_t e = (size_t)(r >> 5) * 256 + (k >> 1) * 64 + (r & 31) * 2 + (k & 1);
                cols[e] = c;
                vals[e] = v;
                ++k;
            };
            if (Z > 0) put(r - m * m, -1);
            if (Y > 0) put(r - m, -1);
            if (X > 0) put(r - 1, -1);
            put(r, 6);
            if (X < m - 1) put(r + 1, -1);
            if (Y < m - 1) put(r + m, -1);
            if (Z < m - 1) put(r + m * m, -1);
            len[r] = k;
        }
        uint32_t *dc, *dl;
        double *dv, *dx, *dy;
        CK(cudaMalloc(&dc, cols.size() * 4));
        CK(cudaMalloc(&dv, vals.size() * 8));
        CK(cudaMalloc(&dl, len.size() * 4));
        CK(cudaMalloc(&dx, (size_t)ns * 8));
        CK(cudaMalloc(&dy, (size_t)ns * 8));
        CK(cudaMemcpy(dc, cols.data(), cols.size() * 4, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(dv, vals.data(), vals.size() * 8, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(dl, len.data(), len.size() * 4, cudaMemcpyHostToDevice));
        CK(cudaMemset(dx, 0, (size_t)ns * 8));
        M A{dc, dv, dl, n};
        const double mb = (cols.size() * 4 + vals.size() * 8 + len.size() * 4) / 1e6;
        const int reps = mb < 100 ? 200 : 3;
        auto run = [&](const char* name, void (*k)(M, const double*, double*, int), int ctas_per_sm) {
            const int grid = dev_sms * ctas_per_sm;
            k<<<grid, 256>>>(A, dx, dy, 1);
            CK(cudaDeviceSynchronize());
            cudaEvent_t a, b;
            cudaEventCreate(&a);
            cudaEventCreate(&b);
            cudaEventRecord(a);
            k<<<grid, 256>>>(A, dx, dy, reps);
            cudaEventRecord(b);
            CK(cudaEventSynchronize(b));
            float ms = 0;
            cudaEventElapsedTime(&ms, a, b);
            const double per = ms / reps * 1e3;  // us per sweep
            printf("m=%4d n=%10u SELL %8.1f MB  %-28s grid %5d: %9.2f us/sweep %8.1f rows/us %7.2f TB/s (SELL+len+x+y)\n",
                   m, n, mb, name, grid, per, n / per, (mb * 1e6 + 16.0 * n) / (per * 1e-6) / 1e12);
        };
        for (int c : {4, 8}) {
            run("v0 row/thread", v0, c);
            run("v1 pipelined rows", v1, c);
            run("v2 two rows/thread", v2, c);
            run("v3 matrix stream only", v3, c);
        }
        cudaFree(dc);
        cudaFree(dv);
        cudaFree(dl);
        cudaFree(dx);
        cudaFree(dy);
    }
    return 0;
}
