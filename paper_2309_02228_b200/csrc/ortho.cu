// Block orthogonalisation after each s-step Newton block (reference
// ortho.hpp, called from sstep.hpp:539-545).  Blocks are column-major with leading dimension
// `rows`, i.e. consecutive VectorBlock slices, exactly as in the reference.
//
//   block_dots   C = Q^T V                     ortho.hpp:46-63
//       bitwise mode: every entry is the reference's serial sum (acc += q_i * v_i, ascending i,
//       mul then add) -- one warp per entry, lanes form 32 products, the add chain is in order.
//       fast mode: fp64 tensor cores (mma.sync m8n8k4 f64), per-CTA partial tiles summed in a
//       fixed order (deterministic for a given grid); tolerance parity.
//   block_update V <- V - Q C                   ortho.hpp:67-92: per element, ascending k,
//       v = v - c_jk * q_k (mul then sub) -- bit-identical in both modes.
//   icgs         sweeps x (dots, update), coefficients accumulated from 0.0  ortho.hpp:97-117
//   tsqr         Householder QR of row panels in shared memory, panel R factors stacked and
//       factored again (recursively) until one panel remains; the explicit Q is formed top-down
//       by applying each panel's reflectors to its c x c block of the level above.  R gets a
//       non-negative diagonal (ortho.hpp:204-212), which makes (Q, R) unique for a full-rank
//       block, so the result matches the reference's panel tree to roundoff (the property the
//       reference's own test pins: test_ortho.cpp:161-177).
#include "device.h"

namespace mpkg_detail {

namespace {

constexpr unsigned kFull = 0xffffffffu;

// ---- block_dots, bitwise ------------------------------------------------------------------
__global__ void k_dots_serial(const double* __restrict__ q, const double* __restrict__ v,
                              uint64_t rows, uint32_t qcols, uint32_t vcols, double* __restrict__ c) {
    const uint32_t lane = threadIdx.x & 31u;
    const uint64_t e = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    if (e >= (uint64_t)qcols * vcols) return;  // warp-uniform
    const double* qk = q + (e % qcols) * rows;
    const double* vj = v + (e / qcols) * rows;
    double acc = 0.0;
    double p = lane < rows ? __dmul_rn(__ldg(qk + lane), __ldg(vj + lane)) : 0.0;
    for (uint64_t i0 = 0; i0 < rows; i0 += 32) {
        // next chunk's products are formed while this chunk's adds run
        const uint64_t in = i0 + 32 + lane;
        const double pn = in < rows ? __dmul_rn(__ldg(qk + in), __ldg(vj + in)) : 0.0;
        const uint32_t m = (uint32_t)(rows - i0 < 32 ? rows - i0 : 32);
        if (m == 32) {
#pragma unroll
            for (int t = 0; t < 32; ++t) acc = __dadd_rn(acc, __shfl_sync(kFull, p, t));
        } else {
            for (uint32_t t = 0; t < m; ++t) acc = __dadd_rn(acc, __shfl_sync(kFull, p, t));
        }
        p = pn;
    }
    if (lane == 0) c[e] = acc;
}

// ---- block_dots, fast (fp64 tensor cores) ------------------------------------------------
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

// One launch covers q columns [mq0, mq0 + 8 MT) x v columns [nv0, nv0 + 8).  Warp w walks
// 16-row blocks b = w, w + W, ... (W = all warps): lane t (group g = t/4, k-slot r = t%4) loads
// rows 16b + 4r + u (u = 0..3) of q column mq0 + 8mt + g and v column nv0 + g, and issues the
// MMA for k-step u, so the 4 k-slots of step u are rows 16b + u, +4, +8, +12.  Each column
// read per block is one full 128-byte line.  Partial 8x8 tiles are reduced over the CTA's
// warps in a fixed order and written per CTA.
template <int MT, bool VEC>
__global__ void __launch_bounds__(256) k_dots_mma(const double* __restrict__ q, const double* __restrict__ v,
                                                  uint64_t rows, uint32_t qcols, uint32_t vcols,
                                                  uint32_t mq0, uint32_t nv0, double* __restrict__ part) {
    __shared__ double red[8][MT * 64];
    const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
    const uint32_t g = lane >> 2, r = lane & 3u;
    const uint64_t W = (uint64_t)gridDim.x * 8u;
    const uint64_t n_blocks = (rows + 15) / 16;
    const double* qc[MT];
    bool qok[MT];
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) {
        const uint32_t col = mq0 + 8 * mt + g;
        qok[mt] = col < qcols;
        qc[mt] = q + (uint64_t)(qok[mt] ? col : 0) * rows;
    }
    const uint32_t vcol = nv0 + g;
    const bool vok = vcol < vcols;
    const double* vc = v + (uint64_t)(vok ? vcol : 0) * rows;
    double acc[MT][2];
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) acc[mt][0] = acc[mt][1] = 0.0;
    for (uint64_t b = blockIdx.x * 8ull + warp; b < n_blocks; b += W) {
        const uint64_t i0 = b * 16 + 4 * r;
        double a[MT][4], bv[4];
        if (VEC && i0 + 3 < rows) {  // 16 B-aligned columns: two LDG.128 per column and lane
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const double2 t = vok ? __ldg(reinterpret_cast<const double2*>(vc + i0) + h) : make_double2(0.0, 0.0);
                bv[2 * h] = t.x, bv[2 * h + 1] = t.y;
            }
#pragma unroll
            for (int mt = 0; mt < MT; ++mt)
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const double2 t = qok[mt] ? __ldg(reinterpret_cast<const double2*>(qc[mt] + i0) + h) : make_double2(0.0, 0.0);
                    a[mt][2 * h] = t.x, a[mt][2 * h + 1] = t.y;
                }
        } else if (i0 + 3 < rows) {
#pragma unroll
            for (int u = 0; u < 4; ++u) bv[u] = vok ? __ldg(vc + i0 + u) : 0.0;
#pragma unroll
            for (int mt = 0; mt < MT; ++mt)
#pragma unroll
                for (int u = 0; u < 4; ++u) a[mt][u] = qok[mt] ? __ldg(qc[mt] + i0 + u) : 0.0;
        } else {
#pragma unroll
            for (int u = 0; u < 4; ++u) bv[u] = (vok && i0 + u < rows) ? vc[i0 + u] : 0.0;
#pragma unroll
            for (int mt = 0; mt < MT; ++mt)
#pragma unroll
                for (int u = 0; u < 4; ++u) a[mt][u] = (qok[mt] && i0 + u < rows) ? qc[mt][i0 + u] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int mt = 0; mt < MT; ++mt) dmma(acc[mt][0], acc[mt][1], a[mt][u], bv[u]);
    }
    // C fragment: row g (q column), columns 2r, 2r+1 (v columns)
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) {
        red[warp][mt * 64 + g * 8 + 2 * r] = acc[mt][0];
        red[warp][mt * 64 + g * 8 + 2 * r + 1] = acc[mt][1];
    }
    __syncthreads();
    for (uint32_t e = threadIdx.x; e < MT * 64; e += blockDim.x) {
        double s = red[0][e];
#pragma unroll
        for (int w = 1; w < 8; ++w) s += red[w][e];
        part[(uint64_t)blockIdx.x * (MT * 64) + e] = s;
    }
}

// Sums the per-CTA partials in CTA order and scatters them to C (qcols x vcols, column-major).
__global__ void k_dots_finish(const double* __restrict__ part, uint32_t n_parts, uint32_t tile_entries,
                              uint32_t qcols, uint32_t vcols, uint32_t mq0, uint32_t nv0,
                              double* __restrict__ c) {
    // one warp per tile entry: lane-strided partial sums over the CTA partials, then a fixed
    // xor-butterfly (deterministic for a given grid)
    const uint32_t e = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31u;
    if (e >= tile_entries) return;
    const uint32_t mt = e / 64, m = (e % 64) / 8, n = e % 8;
    const uint32_t k = mq0 + mt * 8 + m, j = nv0 + n;
    if (k >= qcols || j >= vcols) return;  // warp-uniform
    double s = 0.0;
    for (uint32_t b = lane; b < n_parts; b += 32) s += part[(uint64_t)b * tile_entries + e];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(kFull, s, o);
    if (lane == 0) c[(uint64_t)j * qcols + k] = s;
}

// ---- block_update (bitwise in both modes) --------------------------------------------------
// v_j[i] <- v_j[i] - c_jk q_k[i] for k = 0..qcols-1 ascending (ortho.hpp:83-90).  A thread owns
// row i for up to 8 v columns [j0, j0 + 8); the coefficients sit in shared memory.
template <int VT>
__global__ void __launch_bounds__(256, 3) k_update(const double* __restrict__ q, const double* __restrict__ c,
                                                   uint64_t rows, uint32_t qcols, uint32_t vcols,
                                                   uint32_t j0, double* __restrict__ v) {
    extern __shared__ __align__(16) double cs[];  // [qcols][VT]: one k's coefficients are adjacent
    for (uint32_t e = threadIdx.x; e < VT * qcols; e += blockDim.x) {
        const uint32_t k = e / VT, jj = e % VT;
        cs[e] = j0 + jj < vcols ? c[(uint64_t)(j0 + jj) * qcols + k] : 0.0;
    }
    __syncthreads();
    const uint32_t nv = vcols - j0 < (uint32_t)VT ? vcols - j0 : (uint32_t)VT;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < rows;
         i += (uint64_t)gridDim.x * blockDim.x) {
        double x[VT];
#pragma unroll
        for (int jj = 0; jj < VT; ++jj) x[jj] = jj < (int)nv ? __ldcs(v + (uint64_t)(j0 + jj) * rows + i) : 0.0;
        auto step = [&](uint32_t k, double qk) {
            double ck[VT];
            if constexpr (VT % 2 == 0) {
#pragma unroll
                for (int jj = 0; jj < VT; jj += 2) {  // LDS.128: two coefficients per load
                    const double2 cc = *reinterpret_cast<const double2*>(cs + k * VT + jj);
                    ck[jj] = cc.x, ck[jj + 1] = cc.y;
                }
            } else {
#pragma unroll
                for (int jj = 0; jj < VT; ++jj) ck[jj] = cs[k * VT + jj];
            }
#pragma unroll
            for (int jj = 0; jj < VT; ++jj) x[jj] = __dsub_rn(x[jj], __dmul_rn(ck[jj], qk));
        };
        uint32_t k = 0;
        constexpr int U = 8;  // q loads in flight per thread
        for (; k + U <= qcols; k += U) {
            double qk[U];
#pragma unroll
            for (int u = 0; u < U; ++u) qk[u] = __ldcs(q + (uint64_t)(k + u) * rows + i);
#pragma unroll
            for (int u = 0; u < U; ++u) step(k + u, qk[u]);
        }
        for (; k < qcols; ++k) step(k, __ldcs(q + (uint64_t)k * rows + i));
#pragma unroll
        for (int jj = 0; jj < VT; ++jj)
            if (jj < (int)nv) __stcs(v + (uint64_t)(j0 + jj) * rows + i, x[jj]);
    }
}

// Fast-mode ICGS: one sweep's update fused with the NEXT sweep's dots.  A CTA takes 256-row
// tiles: first every thread updates its row exactly like k_update (ascending k, mul then sub:
// bit-identical; 8 Q loads in flight), writes it and parks it in shared memory; then each warp
// runs the fp64 tensor-core products Q^T V_new for two 16-row blocks of the tile (k_dots_mma's
// fragment layout), re-reading Q from L1/L2 where the update just brought it.  Saves one full
// HBM read of Q and V per extra sweep.
template <int MT>
__global__ void __launch_bounds__(256) k_update_dots(const double* __restrict__ q, const double* __restrict__ c,
                                                     uint64_t rows, uint32_t qcols, uint32_t vcols, uint32_t nv0,
                                                     double* __restrict__ v, double* __restrict__ part) {
    // the tile's updated rows (256 x 9, padded) during the sweep, the per-warp partial tiles after
    constexpr int kBuf = 8 * MT * 64 > 256 * 9 ? 8 * MT * 64 : 256 * 9;
    __shared__ double sbuf[kBuf];
    double (*xs)[9] = reinterpret_cast<double (*)[9]>(sbuf);
    double (*red)[MT * 64] = reinterpret_cast<double (*)[MT * 64]>(sbuf);
    extern __shared__ __align__(16) double cs[];  // [qcols][8] coefficients of V columns nv0..nv0+7
    for (uint32_t e = threadIdx.x; e < 8u * qcols; e += blockDim.x) {
        const uint32_t k = e >> 3, jj = e & 7u;
        cs[e] = nv0 + jj < vcols ? c[(uint64_t)(nv0 + jj) * qcols + k] : 0.0;
    }
    __syncthreads();
    const uint32_t t = threadIdx.x, lane = t & 31u, warp = t >> 5;
    const uint32_t g = lane >> 2, r = lane & 3u;
    const uint32_t nv = vcols - nv0 < 8u ? vcols - nv0 : 8u;
    const double* qc[MT];
    bool qok[MT];
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) {
        const uint32_t col = 8 * mt + g;
        qok[mt] = col < qcols;
        qc[mt] = q + (uint64_t)(qok[mt] ? col : 0) * rows;
    }
    double acc[MT][2];
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) acc[mt][0] = acc[mt][1] = 0.0;
    const uint64_t n_tiles = (rows + 255) / 256;
    for (uint64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
        const uint64_t i = tile * 256 + t;
        double x[8];
        if (i < rows) {
#pragma unroll
            for (int jj = 0; jj < 8; ++jj) x[jj] = jj < (int)nv ? __ldcs(v + (uint64_t)(nv0 + jj) * rows + i) : 0.0;
            uint32_t k = 0;
            constexpr int U = 8;
            for (; k + U <= qcols; k += U) {
                double qk[U];
#pragma unroll
                for (int u = 0; u < U; ++u) qk[u] = __ldg(q + (uint64_t)(k + u) * rows + i);
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const double2* c2 = reinterpret_cast<const double2*>(cs + (k + u) * 8);
#pragma unroll
                    for (int h = 0; h < 4; ++h) {
                        const double2 cc = c2[h];
                        x[2 * h] = __dsub_rn(x[2 * h], __dmul_rn(cc.x, qk[u]));
                        x[2 * h + 1] = __dsub_rn(x[2 * h + 1], __dmul_rn(cc.y, qk[u]));
                    }
                }
            }
            for (; k < qcols; ++k) {
                const double qk = __ldg(q + (uint64_t)k * rows + i);
#pragma unroll
                for (int jj = 0; jj < 8; ++jj) x[jj] = __dsub_rn(x[jj], __dmul_rn(cs[k * 8 + jj], qk));
            }
#pragma unroll
            for (int jj = 0; jj < 8; ++jj)
                if (jj < (int)nv) __stcs(v + (uint64_t)(nv0 + jj) * rows + i, x[jj]);
        } else {
#pragma unroll
            for (int jj = 0; jj < 8; ++jj) x[jj] = 0.0;
        }
#pragma unroll
        for (int jj = 0; jj < 8; ++jj) xs[t][jj] = jj < (int)nv ? x[jj] : 0.0;
        __syncthreads();
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const uint32_t rb = (2 * warp + h) * 16 + 4 * r;  // tile-local first row of this lane
            const uint64_t i0 = tile * 256 + rb;
            double a[MT][4], bv[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) bv[u] = xs[rb + u][g];
#pragma unroll
            for (int mt = 0; mt < MT; ++mt)
#pragma unroll
                for (int u = 0; u < 4; ++u) a[mt][u] = (qok[mt] && i0 + u < rows) ? __ldg(qc[mt] + i0 + u) : 0.0;
#pragma unroll
            for (int u = 0; u < 4; ++u)
#pragma unroll
                for (int mt = 0; mt < MT; ++mt) dmma(acc[mt][0], acc[mt][1], a[mt][u], bv[u]);
        }
        __syncthreads();  // xs is rewritten by the next tile
    }
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) {
        red[warp][mt * 64 + g * 8 + 2 * r] = acc[mt][0];
        red[warp][mt * 64 + g * 8 + 2 * r + 1] = acc[mt][1];
    }
    __syncthreads();
    for (uint32_t e = threadIdx.x; e < MT * 64; e += blockDim.x) {
        double s = red[0][e];
#pragma unroll
        for (int w = 1; w < 8; ++w) s += red[w][e];
        part[(uint64_t)blockIdx.x * (MT * 64) + e] = s;
    }
}

// The same fusion with the tile's Q rows staged in shared memory by the update phase (128-row
// tiles, 128 threads: the staged copy is 26 KB for 25 columns, so five CTAs fit an SM); the
// tensor-core phase then reads Q from shared memory instead of L1/L2 (knob "ortho_fused" = 2, the
// default: ICGS 1.30 ms vs 1.37 ms re-reading from L1/L2 and 1.48 ms unfused on a C4-sized block).
template <int MT>
__global__ void __launch_bounds__(128) k_update_dots_s(const double* __restrict__ q, const double* __restrict__ c,
                                                       uint64_t rows, uint32_t qcols, uint32_t vcols, uint32_t nv0,
                                                       double* __restrict__ v, double* __restrict__ part) {
    constexpr int kBuf = 4 * MT * 64 > 128 * 9 ? 4 * MT * 64 : 128 * 9;
    __shared__ double sbuf[kBuf];
    double (*xs)[9] = reinterpret_cast<double (*)[9]>(sbuf);
    double (*red)[MT * 64] = reinterpret_cast<double (*)[MT * 64]>(sbuf);
    extern __shared__ __align__(16) double cs[];  // [qcols][8] coefficients, then Q rows [128][qs_ld]
    const uint32_t qs_ld = qcols | 1u;
    double* qs = cs + 8u * qcols;
    for (uint32_t e = threadIdx.x; e < 8u * qcols; e += blockDim.x) {
        const uint32_t k = e >> 3, jj = e & 7u;
        cs[e] = nv0 + jj < vcols ? c[(uint64_t)(nv0 + jj) * qcols + k] : 0.0;
    }
    __syncthreads();
    const uint32_t t = threadIdx.x, lane = t & 31u, warp = t >> 5;
    const uint32_t g = lane >> 2, r = lane & 3u;
    const uint32_t nv = vcols - nv0 < 8u ? vcols - nv0 : 8u;
    bool qok[MT];
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) qok[mt] = 8 * mt + g < qcols;
    double acc[MT][2];
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) acc[mt][0] = acc[mt][1] = 0.0;
    const uint64_t n_tiles = (rows + 127) / 128;
    for (uint64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
        const uint64_t i = tile * 128 + t;
        double x[8];
        double* qrow = qs + t * qs_ld;
        if (i < rows) {
#pragma unroll
            for (int jj = 0; jj < 8; ++jj) x[jj] = jj < (int)nv ? __ldcs(v + (uint64_t)(nv0 + jj) * rows + i) : 0.0;
            uint32_t k = 0;
            constexpr int U = 8;
            for (; k + U <= qcols; k += U) {
                double qk[U];
#pragma unroll
                for (int u = 0; u < U; ++u) qk[u] = __ldcs(q + (uint64_t)(k + u) * rows + i);
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    qrow[k + u] = qk[u];
                    const double2* c2 = reinterpret_cast<const double2*>(cs + (k + u) * 8);
#pragma unroll
                    for (int h = 0; h < 4; ++h) {
                        const double2 cc = c2[h];
                        x[2 * h] = __dsub_rn(x[2 * h], __dmul_rn(cc.x, qk[u]));
                        x[2 * h + 1] = __dsub_rn(x[2 * h + 1], __dmul_rn(cc.y, qk[u]));
                    }
                }
            }
            for (; k < qcols; ++k) {
                const double qk = __ldcs(q + (uint64_t)k * rows + i);
                qrow[k] = qk;
#pragma unroll
                for (int jj = 0; jj < 8; ++jj) x[jj] = __dsub_rn(x[jj], __dmul_rn(cs[k * 8 + jj], qk));
            }
#pragma unroll
            for (int jj = 0; jj < 8; ++jj)
                if (jj < (int)nv) __stcs(v + (uint64_t)(nv0 + jj) * rows + i, x[jj]);
        } else {
#pragma unroll
            for (int jj = 0; jj < 8; ++jj) x[jj] = 0.0;
            for (uint32_t k = 0; k < qcols; ++k) qrow[k] = 0.0;
        }
#pragma unroll
        for (int jj = 0; jj < 8; ++jj) xs[t][jj] = jj < (int)nv ? x[jj] : 0.0;
        __syncthreads();
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const uint32_t rb = (2 * warp + h) * 16 + 4 * r;
            double a[MT][4], bv[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) bv[u] = xs[rb + u][g];
#pragma unroll
            for (int mt = 0; mt < MT; ++mt)
#pragma unroll
                for (int u = 0; u < 4; ++u) a[mt][u] = qok[mt] ? qs[(rb + u) * qs_ld + 8 * mt + g] : 0.0;
#pragma unroll
            for (int u = 0; u < 4; ++u)
#pragma unroll
                for (int mt = 0; mt < MT; ++mt) dmma(acc[mt][0], acc[mt][1], a[mt][u], bv[u]);
        }
        __syncthreads();
    }
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) {
        red[warp][mt * 64 + g * 8 + 2 * r] = acc[mt][0];
        red[warp][mt * 64 + g * 8 + 2 * r + 1] = acc[mt][1];
    }
    __syncthreads();
    for (uint32_t e = threadIdx.x; e < MT * 64; e += blockDim.x) {
        double s = red[0][e];
#pragma unroll
        for (int w = 1; w < 4; ++w) s += red[w][e];
        part[(uint64_t)blockIdx.x * (MT * 64) + e] = s;
    }
}

// coeff[e] += c[e] (ortho.hpp:112-114)
__global__ void k_accumulate(double* __restrict__ coeff, const double* __restrict__ c, uint32_t n) {
    const uint32_t e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e < n) coeff[e] = __dadd_rn(coeff[e], c[e]);
}

// ---- tsqr ---------------------------------------------------------------------------------
// Panel k of a level holds rows [rows*k/np, rows*(k+1)/np).
__device__ __forceinline__ uint64_t panel_bound(uint64_t rows, uint32_t np, uint32_t k) {
    return rows * k / np;
}

__device__ __forceinline__ bool lane_bit(uint32_t b) { return (threadIdx.x & b) != 0u; }

__device__ __forceinline__ double warp_sum(double s) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(kFull, s, o);
    return s;
}

// Householder QR of every panel of `a` (rows x c, leading dimension lda) in shared memory.
// Column j: alpha = A_jj, sigma = sum_{i>j} A_ij^2; sigma == 0 leaves tau = 0 (H = I) with
// beta = alpha, else beta = -sign(alpha) sqrt(alpha^2 + sigma), v = A_{j+1:, j} / (alpha - beta),
// tau = (beta - alpha) / beta.  The reflector is stored below the diagonal (unit leading
// entry implied), tau in taus[k*c + j].  R_k (upper c x c) goes to block k of `rstack`
// (np*c rows x c, leading dimension np*c), the reflectors back into `a` in place.
__global__ void __launch_bounds__(256) k_panel_qr(double* __restrict__ a, uint64_t lda, uint64_t rows,
                                                  uint32_t np, uint32_t c, double* __restrict__ taus,
                                                  double* __restrict__ rstack) {
    extern __shared__ double sm[];
    const uint32_t k = blockIdx.x;
    const uint64_t b0 = panel_bound(rows, np, k), b1 = panel_bound(rows, np, k + 1);
    const uint32_t P = (uint32_t)(b1 - b0);
    double* A = sm;  // [c][P]
    __shared__ double s_tau;
    const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (uint32_t l = 0; l < c; ++l)
        for (uint32_t i = threadIdx.x; i < P; i += blockDim.x) A[(uint64_t)l * P + i] = a[l * lda + b0 + i];
    __syncthreads();
    for (uint32_t j = 0; j < c; ++j) {
        double* Aj = A + (uint64_t)j * P;
        if (warp == 0) {
            double s = 0.0;
            for (uint32_t i = j + 1 + lane; i < P; i += 32) s += Aj[i] * Aj[i];
            const double sigma = warp_sum(s);
            const double alpha = Aj[j];
            double tau = 0.0, beta = alpha, scale = 0.0;
            if (sigma != 0.0) {
                const double nrm = sqrt(alpha * alpha + sigma);
                beta = alpha >= 0.0 ? -nrm : nrm;
                tau = (beta - alpha) / beta;
                scale = 1.0 / (alpha - beta);
            }
            for (uint32_t i = j + 1 + lane; i < P; i += 32) Aj[i] *= scale;  // sigma == 0: zeros
            __syncwarp();
            if (lane == 0) {
                Aj[j] = beta;
                s_tau = tau;
                taus[(uint64_t)k * c + j] = tau;
            }
        }
        __syncthreads();
        const double tau = s_tau;
        if (tau != 0.0) {
            for (uint32_t l = j + 1 + warp; l < c; l += nw) {
                double* Al = A + (uint64_t)l * P;
                double s = 0.0;
                for (uint32_t i = j + 1 + lane; i < P; i += 32) s += Aj[i] * Al[i];
                const double w = tau * (Al[j] + warp_sum(s));
                if (lane == 0) Al[j] -= w;
                for (uint32_t i = j + 1 + lane; i < P; i += 32) Al[i] -= w * Aj[i];
            }
        }
        __syncthreads();
    }
    const uint64_t ldr = (uint64_t)np * c;
    for (uint32_t e = threadIdx.x; e < c * c; e += blockDim.x) {
        const uint32_t l = e / c, i = e % c;
        rstack[l * ldr + (uint64_t)k * c + i] = i <= l ? A[(uint64_t)l * P + i] : 0.0;
    }
    for (uint32_t l = 0; l < c; ++l)
        for (uint32_t i = threadIdx.x; i < P; i += blockDim.x) a[l * lda + b0 + i] = A[(uint64_t)l * P + i];
}

// Forms the explicit thin Q of every panel times its c x c multiplier M_k (rows k*c.. of `m`,
// leading dimension ldm): Y = H_0 H_1 ... H_{c-1} [M_k; 0], applied right to left.  Reads the
// reflectors from `a` and writes Y over them.
__global__ void __launch_bounds__(256) k_panel_formq(double* __restrict__ a, uint64_t lda, uint64_t rows,
                                                     uint32_t np, uint32_t c, const double* __restrict__ taus,
                                                     const double* __restrict__ m, uint64_t ldm) {
    extern __shared__ double sm[];
    const uint32_t k = blockIdx.x;
    const uint64_t b0 = panel_bound(rows, np, k), b1 = panel_bound(rows, np, k + 1);
    const uint32_t P = (uint32_t)(b1 - b0);
    double* H = sm;                       // [c][P] reflectors
    double* Y = sm + (uint64_t)c * P;     // [c][P]
    const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (uint32_t l = 0; l < c; ++l)
        for (uint32_t i = threadIdx.x; i < P; i += blockDim.x) {
            H[(uint64_t)l * P + i] = a[l * lda + b0 + i];
            Y[(uint64_t)l * P + i] = i < c ? m[l * ldm + (uint64_t)k * c + i] : 0.0;
        }
    __syncthreads();
    for (int j = (int)c - 1; j >= 0; --j) {
        const double tau = taus[(uint64_t)k * c + j];
        if (tau == 0.0) continue;  // uniform
        const double* Hj = H + (uint64_t)j * P;
        for (uint32_t l = warp; l < c; l += nw) {
            double* Yl = Y + (uint64_t)l * P;
            double s = 0.0;
            for (uint32_t i = j + 1 + lane; i < P; i += 32) s += Hj[i] * Yl[i];
            const double w = tau * (Yl[j] + warp_sum(s));
            if (lane == 0) Yl[j] -= w;
            for (uint32_t i = j + 1 + lane; i < P; i += 32) Yl[i] -= w * Hj[i];
        }
        __syncthreads();
    }
    for (uint32_t l = 0; l < c; ++l)
        for (uint32_t i = threadIdx.x; i < P; i += blockDim.x) a[l * lda + b0 + i] = Y[(uint64_t)l * P + i];
}

// Narrow blocks (c <= 8, the s-step case): one WARP per panel of up to 32*TQ_R rows, the panel
// held in registers (lane owns rows lane + 32 r), reductions by xor-shuffle butterflies (fixed
// order, every lane holds the sum): no shared memory and no block barriers, so many panels are in
// flight per SM.  Same Householder convention as k_panel_qr.  FORM = false: factor the panel and
// write its R to `rstack`.  FORM = true: factor the panel AGAIN from the untouched input (the
// reflectors are recomputed, never stored: one read of the block instead of a write + re-read)
// and overwrite it with Y = H_0 ... H_{c-1} [M_k; 0].
constexpr int kTqC = 8;
constexpr int kTqR = 8;
constexpr uint32_t kTqPanel = 32u * kTqR;

// Butterfly sums of N independent values: the N shuffle chains interleave (ILP N).
template <int N>
__device__ __forceinline__ void warp_sum_n(double (&v)[N]) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
#pragma unroll
        for (int n = 0; n < N; ++n) v[n] += __shfl_xor_sync(kFull, v[n], o);
}

// Sums of 8 values over the warp, returned in every lane, by reduce-scatter: lanes exchange
// halves at distances 16, 8, 4 (4 + 2 + 1 shuffles), finish with a 2-level butterfly on the one
// value left, then read the 8 totals back from their holder lanes (8 shuffles): 17 double
// shuffles instead of the plain butterfly's 40.  Fixed order, the same totals in every lane.
__device__ __forceinline__ void warp_sum8(double (&v)[8]) {
    const bool h16 = lane_bit(16), h8 = lane_bit(8), h4 = lane_bit(4);
    double a[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const double send = h16 ? v[i] : v[4 + i];
        const double keep = h16 ? v[4 + i] : v[i];
        a[i] = keep + __shfl_xor_sync(kFull, send, 16);
    }
    double b[2];
#pragma unroll
    for (int i = 0; i < 2; ++i) {
        const double send = h8 ? a[i] : a[2 + i];
        const double keep = h8 ? a[2 + i] : a[i];
        b[i] = keep + __shfl_xor_sync(kFull, send, 8);
    }
    double t = (h4 ? b[1] : b[0]) + __shfl_xor_sync(kFull, h4 ? b[0] : b[1], 4);
    t += __shfl_xor_sync(kFull, t, 2);
    t += __shfl_xor_sync(kFull, t, 1);
    // lane L holds total index 4*(L>>4 & 1) + 2*(L>>3 & 1) + (L>>2 & 1)
#pragma unroll
    for (int l = 0; l < 8; ++l) v[l] = __shfl_sync(kFull, t, ((l & 4) ? 16 : 0) + ((l & 2) ? 8 : 0) + ((l & 1) ? 4 : 0));
}

// Factor kernel.  Columns l >= c and rows i >= P are loaded as zeros and stay zero through every
// update, so the arithmetic needs no column / row-count predicates; only row i <= j (r = 0,
// lane <= j) is excluded from step j's reflector.  Writes the panel's R to `rstack`, the
// reflectors over the panel in place (LAPACK layout: v below the diagonal, R on and above) and
// the compact-WY factor T (8 x 8 upper triangular, row-major, H_0 ... H_{c-1} = I - V T V^T) to
// `tmat` (64 doubles per panel), followed by the panel's V_top (64 doubles).
// UPD: the panel is ICGS's last update V - Q C computed on the fly (ascending k, mul then sub:
// block_update's arithmetic, bit for bit) instead of read -- the updated block is never written
// (TSQR overwrites it anyway), which saves a write and a read of V (mpkg_ortho_block).
template <bool UPD>
__global__ void __launch_bounds__(128) k_tsqr_factor(double* __restrict__ a, uint64_t lda, uint64_t rows,
                                                     uint32_t np, uint32_t c, double* __restrict__ rstack,
                                                     double* __restrict__ tmat, const double* __restrict__ q,
                                                     const double* __restrict__ coef, uint32_t qcols) {
    extern __shared__ __align__(16) double cs[];  // UPD: [qcols][8] coefficients
    if constexpr (UPD) {
        for (uint32_t e = threadIdx.x; e < 8u * qcols; e += blockDim.x) {
            const uint32_t kk = e >> 3, jj = e & 7u;
            cs[e] = jj < c ? coef[(uint64_t)jj * qcols + kk] : 0.0;
        }
        __syncthreads();
    }
    const uint32_t k = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint32_t lane = threadIdx.x & 31u;
    if (k >= np) return;  // warp-uniform
    const uint64_t b0 = panel_bound(rows, np, k), b1 = panel_bound(rows, np, k + 1);
    const uint32_t P = (uint32_t)(b1 - b0);
    double A[kTqR][kTqC];
    if constexpr (UPD) {
        // A = V - Q C, k outermost: each step loads the lane's 8 rows of KU Q columns at once
#pragma unroll
        for (int l = 0; l < kTqC; ++l)
#pragma unroll
            for (int r = 0; r < kTqR; ++r) {
                const uint32_t i = lane + 32u * r;
                A[r][l] = ((uint32_t)l < c && i < P) ? __ldcs(a + (uint64_t)l * lda + b0 + i) : 0.0;
            }
        uint32_t kk = 0;
        constexpr int KU = 4;  // Q columns per step: 32 loads in flight per lane
        for (; kk + KU <= qcols; kk += KU) {
            double qv[KU][kTqR];
#pragma unroll
            for (int u = 0; u < KU; ++u)
#pragma unroll
                for (int r = 0; r < kTqR; ++r) {
                    const uint32_t i = lane + 32u * r;
                    qv[u][r] = i < P ? __ldcs(q + (uint64_t)(kk + u) * lda + b0 + i) : 0.0;
                }
#pragma unroll
            for (int u = 0; u < KU; ++u)
#pragma unroll
                for (int l = 0; l < kTqC; ++l) {
                    const double cl = cs[(kk + u) * 8 + l];
#pragma unroll
                    for (int r = 0; r < kTqR; ++r) A[r][l] = __dsub_rn(A[r][l], __dmul_rn(cl, qv[u][r]));
                }
        }
        for (; kk < qcols; ++kk) {
            double qv[kTqR];
#pragma unroll
            for (int r = 0; r < kTqR; ++r) {
                const uint32_t i = lane + 32u * r;
                qv[r] = i < P ? __ldcs(q + (uint64_t)kk * lda + b0 + i) : 0.0;
            }
#pragma unroll
            for (int l = 0; l < kTqC; ++l) {
                const double cl = cs[kk * 8 + l];
#pragma unroll
                for (int r = 0; r < kTqR; ++r) A[r][l] = __dsub_rn(A[r][l], __dmul_rn(cl, qv[r]));
            }
        }
        // rows past the panel and columns past c are exact zeros (0 - c * 0, and c = 0 for l >= c)
    } else {
#pragma unroll
        for (int l = 0; l < kTqC; ++l)
#pragma unroll
            for (int r = 0; r < kTqR; ++r) {
                const uint32_t i = lane + 32u * r;
                A[r][l] = ((uint32_t)l < c && i < P) ? a[(uint64_t)l * lda + b0 + i] : 0.0;
            }
    }
    // Lane i < 8 builds row i of T column by column (dlarft, forward, columnwise):
    // T_jj = tau_j, T_{0:j,j} = -tau_j T_{0:j,0:j} (V_{:,0:j}^T v_j).  The Gram entries v_m . v_j
    // (m < j) ride in the free slots of step j's 8-wide reduction (slots l > j carry w_l).
    double trow[kTqC];
#pragma unroll
    for (int j = 0; j < kTqC; ++j) trow[j] = 0.0;
#pragma unroll
    for (int j = 0; j < kTqC; ++j) {
        if ((uint32_t)j >= c) break;  // uniform
        const bool below = lane > (uint32_t)j, diag = lane == (uint32_t)j;
        const double a0 = below ? A[0][j] : 0.0;
        double sg[1] = {a0 * a0};
#pragma unroll
        for (int r = 1; r < kTqR; ++r) sg[0] += A[r][j] * A[r][j];
        const double alpha = __shfl_sync(kFull, A[0][j], j);
        warp_sum_n(sg);
        const double sigma = sg[0];
        double t = 0.0, beta = alpha, scale = 0.0;
        if (sigma != 0.0) {
            const double nrm = sqrt(alpha * alpha + sigma);
            beta = alpha >= 0.0 ? -nrm : nrm;
            t = (beta - alpha) / beta;
            scale = 1.0 / (alpha - beta);
        }
        const double vj = diag ? 1.0 : a0 * scale;  // row-0 reflector entry (0 above the diagonal)
        A[0][j] = below ? vj : (diag ? beta : A[0][j]);
#pragma unroll
        for (int r = 1; r < kTqR; ++r) A[r][j] *= scale;
        if (t != 0.0) {  // uniform; tau_j = 0 leaves T's column j zero and the block unchanged
            double w[kTqC];
#pragma unroll
            for (int l = 0; l < kTqC; ++l) {
                // l > j: v_j . A_l (the update);  l < j: v_l . v_j (T);  l == j: unused
                const double x0 = l > j ? A[0][l] : (l < j ? (lane == (uint32_t)l ? 1.0 : (lane > (uint32_t)l ? A[0][l] : 0.0)) : 0.0);
                w[l] = vj * x0;
                if (l != j) {
#pragma unroll
                    for (int r = 1; r < kTqR; ++r) w[l] += A[r][j] * A[r][l];
                }
            }
            warp_sum8(w);
            double sT = 0.0;
#pragma unroll
            for (int m = 0; m < j; ++m) sT += trow[m] * w[m];
            trow[j] = diag ? t : (lane < (uint32_t)j ? -t * sT : 0.0);
#pragma unroll
            for (int l = j + 1; l < kTqC; ++l) {
                const double wl = t * w[l];
                A[0][l] -= wl * vj;
#pragma unroll
                for (int r = 1; r < kTqR; ++r) A[r][l] -= wl * A[r][j];
            }
        }
    }
    if (lane < 8) {
        // T, then V_top (the panel's first 8 reflector rows: unit diagonal, zero above): the
        // apply kernel's sub-panel warps read it from here, since sub-panel 0 overwrites those
        // rows of the block with Y
#pragma unroll
        for (int j = 0; j < kTqC; ++j) tmat[(uint64_t)k * 128 + lane * 8 + j] = trow[j];
#pragma unroll
        for (int l = 0; l < kTqC; ++l)
            tmat[(uint64_t)k * 128 + 64 + lane * 8 + l] = lane == (uint32_t)l ? 1.0 : (lane < (uint32_t)l ? 0.0 : A[0][l]);
    }
    const uint64_t ldr = (uint64_t)np * c;
    if (lane < c)
#pragma unroll
        for (int l = 0; l < kTqC; ++l)
            if ((uint32_t)l < c) rstack[(uint64_t)l * ldr + (uint64_t)k * c + lane] = lane <= (uint32_t)l ? A[0][l] : 0.0;
#pragma unroll
    for (int l = 0; l < kTqC; ++l)
#pragma unroll
        for (int r = 0; r < kTqR; ++r) {
            const uint32_t i = lane + 32u * r;
            if ((uint32_t)l < c && i < P) a[(uint64_t)l * lda + b0 + i] = A[r][l];
        }
}

// Apply kernel: Y = (I - V T V^T) [M_k; 0] = [M_k; 0] - V (T (V_top^T M_k)), V_top the panel's
// top 8 rows (M_k is zero below row c).  No reduction over the panel: the two 8 x 8 products go
// through per-warp shared memory, then every row is an 8 x 8 matvec.  Overwrites the reflectors.
constexpr int kAR = 4;                 // apply: rows per lane (one warp per 32*kAR-row sub-panel)
constexpr uint32_t kSub = kTqR / kAR;  // apply warps per factor panel

__global__ void __launch_bounds__(128) k_tsqr_apply(double* __restrict__ a, uint64_t lda, uint64_t rows,
                                                    uint32_t np, uint32_t c, const double* __restrict__ tmat,
                                                    const double* __restrict__ m, uint64_t ldm) {
    __shared__ double sh[4][3][64];  // per warp: V_top / S, M, T
    const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint32_t k = gw / kSub, r0 = (gw % kSub) * kAR;  // panel, first 32-row group of the sub-panel
    const uint32_t lane = threadIdx.x & 31u, wib = threadIdx.x >> 5;
    if (k >= np) return;  // warp-uniform
    double* Vs = sh[wib][0];
    double* Ms = sh[wib][1];
    double* Ts = sh[wib][2];
    const uint64_t b0 = panel_bound(rows, np, k), b1 = panel_bound(rows, np, k + 1);
    const uint32_t P = (uint32_t)(b1 - b0);
    double m0[kTqC];
#pragma unroll
    for (int l = 0; l < kTqC; ++l) m0[l] = ((uint32_t)l < c && lane < c) ? m[(uint64_t)l * ldm + (uint64_t)k * c + lane] : 0.0;
    if (lane < 8) {
#pragma unroll
        for (int l = 0; l < kTqC; ++l) Ms[lane * 8 + l] = m0[l];
    }
    Ts[lane] = tmat[(uint64_t)k * 128 + lane];
    Ts[lane + 32] = tmat[(uint64_t)k * 128 + lane + 32];
    Vs[lane] = tmat[(uint64_t)k * 128 + 64 + lane];  // V_top as stored by the factor kernel
    Vs[lane + 32] = tmat[(uint64_t)k * 128 + 96 + lane];
    __syncwarp();
    // W = V_top^T M (entries e = lane, lane + 32: row e/8, column e%8)
    double wv[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const uint32_t e = lane + 32u * h, j = e >> 3, l = e & 7u;
        double s = 0.0;
#pragma unroll
        for (int i = 0; i < 8; ++i) s += Vs[i * 8 + j] * Ms[i * 8 + l];
        wv[h] = s;
    }
    __syncwarp();
    Ms[lane] = wv[0];
    Ms[lane + 32] = wv[1];
    __syncwarp();
    // S = T W (T upper triangular)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const uint32_t e = lane + 32u * h, j = e >> 3, l = e & 7u;
        double s = 0.0;
#pragma unroll
        for (int q = 0; q < 8; ++q) s += Ts[j * 8 + q] * Ms[q * 8 + l];
        wv[h] = s;
    }
    Vs[lane] = wv[0];  // V_top no longer read (all lanes passed the W loop before the last sync)
    Vs[lane + 32] = wv[1];
    __syncwarp();
    // Y = [M; 0] - V S on this warp's sub-panel (S recomputed per warp: two 8 x 8 products)
    {
        double A[kAR][kTqC];
#pragma unroll
        for (int l = 0; l < kTqC; ++l)
#pragma unroll
            for (int r = 0; r < kAR; ++r) {
                const uint32_t i = lane + 32u * (r0 + r);
                double v = ((uint32_t)l < c && i < P) ? a[(uint64_t)l * lda + b0 + i] : 0.0;
                if (r0 + r == 0) v = lane == (uint32_t)l ? 1.0 : (lane < (uint32_t)l ? 0.0 : v);
                A[r][l] = v;
            }
#pragma unroll 1
        for (uint32_t l = 0; l < c; ++l) {  // one S column (8 LDS) at a time keeps registers low
            double sc[kTqC];
#pragma unroll
            for (int j = 0; j < kTqC; ++j) sc[j] = Vs[j * 8 + l];
            double ml = 0.0;
#pragma unroll
            for (int t = 0; t < kTqC; ++t) ml = (uint32_t)t == l ? m0[t] : ml;
#pragma unroll
            for (int r = 0; r < kAR; ++r) {
                double y = (r0 + r == 0) ? ml : 0.0;
#pragma unroll
                for (int j = 0; j < kTqC; ++j) y -= A[r][j] * sc[j];
                const uint32_t i = lane + 32u * (r0 + r);
                if (i < P) a[(uint64_t)l * lda + b0 + i] = y;
            }
        }
    }
}

// Top of the tree: R (c x c, column-major) with row j negated when R_jj < 0 and the strictly
// lower part zero (ortho.hpp:204-212, 221-226); M = diag(sign) for the top panel's Q.
__global__ void k_sign_fix(const double* __restrict__ rtop, uint32_t c, double* __restrict__ r,
                           double* __restrict__ m) {
    for (uint32_t e = threadIdx.x; e < c * c; e += blockDim.x) {
        const uint32_t l = e / c, i = e % c;
        const double sg = rtop[(uint64_t)i * c + i] < 0.0 ? -1.0 : 1.0;
        r[e] = i <= l ? sg * rtop[e] : 0.0;
        m[e] = i == l ? (rtop[(uint64_t)l * c + l] < 0.0 ? -1.0 : 1.0) : 0.0;
    }
}

}  // namespace

// ---- host side ----------------------------------------------------------------------------

void gpu_block_dots(mpkg_ctx_s* ctx, const double* q, const double* v, uint64_t rows, uint32_t qcols,
                    uint32_t vcols, double* c) {
    if (!qcols || !vcols) return;
    if (rows == 0) {
        MPKG_CUDA(cudaMemsetAsync(c, 0, 8ull * qcols * vcols, ctx->stream));
        return;
    }
    const auto ev = timing_begin(ctx);
    if (ctx->mode == MPKG_MODE_BITWISE) {
        const uint64_t threads = 32ull * qcols * vcols;
        k_dots_serial<<<(unsigned)((threads + 255) / 256), 256, 0, ctx->stream>>>(q, v, rows, qcols, vcols, c);
        MPKG_LAUNCH_CHECK();
        ctx->launches += 1;
    } else {
        const uint64_t n_blocks = (rows + 15) / 16;
        const unsigned grid = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((uint64_t)ctx->sm_count * 4u, (n_blocks + 7) / 8));
        for (uint32_t nv0 = 0; nv0 < vcols; nv0 += 8) {
            for (uint32_t mq0 = 0; mq0 < qcols; mq0 += 64) {
                const uint32_t left = (qcols - mq0 + 7) / 8;
                const int MT = left >= 8 ? 8 : left > 4 ? 8 : left > 2 ? 4 : left > 1 ? 2 : 1;
                const uint32_t te = MT * 64u;
                ctx->chain_ws.ensure((uint64_t)grid * te);
                double* part = ctx->chain_ws.p;
                // every column 16 B aligned: even row count and aligned base pointers
                const bool vec = rows % 2 == 0 && ((uintptr_t)q | (uintptr_t)v) % 16 == 0;
#define MPKG_DOTS(M)                                                                                       \
    (vec ? k_dots_mma<M, true><<<grid, 256, 0, ctx->stream>>>(q, v, rows, qcols, vcols, mq0, nv0, part)    \
         : k_dots_mma<M, false><<<grid, 256, 0, ctx->stream>>>(q, v, rows, qcols, vcols, mq0, nv0, part))
                switch (MT) {
                    case 1: MPKG_DOTS(1); break;
                    case 2: MPKG_DOTS(2); break;
                    case 4: MPKG_DOTS(4); break;
                    default: MPKG_DOTS(8); break;
                }
#undef MPKG_DOTS
                MPKG_LAUNCH_CHECK();
                k_dots_finish<<<(te * 32 + 255) / 256, 256, 0, ctx->stream>>>(part, grid, te, qcols, vcols, mq0, nv0, c);
                MPKG_LAUNCH_CHECK();
                ctx->launches += 2;
            }
        }
    }
    timing_end(ctx, ev);
}

void gpu_block_update(mpkg_ctx_s* ctx, const double* q, const double* c, uint64_t rows, uint32_t qcols,
                      uint32_t vcols, double* v) {
    if (!qcols || !vcols || !rows) return;
    const auto ev = timing_begin(ctx);
    const unsigned grid = grid_for(rows, 256, (unsigned)ctx->sm_count * 8u);
    for (uint32_t j0 = 0; j0 < vcols; j0 += 8) {
        const uint32_t nv = std::min<uint32_t>(8, vcols - j0);
        const size_t smem = 8ull * qcols * (nv > 4 ? 8 : nv > 2 ? 4 : nv > 1 ? 2 : 1);
        if (nv > 4) {
            if (smem > 48 * 1024)
                MPKG_CUDA(cudaFuncSetAttribute(k_update<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            k_update<8><<<grid, 256, smem, ctx->stream>>>(q, c, rows, qcols, vcols, j0, v);
        } else if (nv > 2) {
            if (smem > 48 * 1024)
                MPKG_CUDA(cudaFuncSetAttribute(k_update<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            k_update<4><<<grid, 256, smem, ctx->stream>>>(q, c, rows, qcols, vcols, j0, v);
        } else if (nv > 1) {
            k_update<2><<<grid, 256, smem, ctx->stream>>>(q, c, rows, qcols, vcols, j0, v);
        } else {
            k_update<1><<<grid, 256, smem, ctx->stream>>>(q, c, rows, qcols, vcols, j0, v);
        }
        MPKG_LAUNCH_CHECK();
        ctx->launches += 1;
    }
    timing_end(ctx, ev);
}

// V <- V - Q c (bitwise, as k_update) and c_next = Q^T V_new (fast-mode products), fused.
void gpu_update_dots(mpkg_ctx_s* ctx, const double* q, const double* c, uint64_t rows, uint32_t qcols,
                     uint32_t vcols, double* v, double* c_next) {
    const auto ev = timing_begin(ctx);
    const uint64_t n_tiles = (rows + 255) / 256;
    const unsigned grid = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((uint64_t)ctx->sm_count * 3u, n_tiles));
    const uint32_t left = (qcols + 7) / 8;
    const int MT = left > 4 ? 8 : left > 2 ? 4 : left > 1 ? 2 : 1;
    const uint32_t te = MT * 64u;
    ctx->chain_ws.ensure((uint64_t)grid * te);
    double* part = ctx->chain_ws.p;
    const size_t smem = 64ull * qcols;
    const bool staged = ctx->ortho_fused == 2;
    unsigned grid_s = grid;
    const size_t smem_s = 64ull * qcols + 8ull * 128 * (qcols | 1u);
    if (staged) {
        static const void* fs[4] = {(const void*)k_update_dots_s<1>, (const void*)k_update_dots_s<2>,
                                    (const void*)k_update_dots_s<4>, (const void*)k_update_dots_s<8>};
        const void* f = fs[MT == 1 ? 0 : MT == 2 ? 1 : MT == 4 ? 2 : 3];
        MPKG_CUDA(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_s));
        int per_sm = 0;
        MPKG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, f, 128, smem_s));
        grid_s = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((uint64_t)ctx->sm_count * std::max(per_sm, 1), (rows + 127) / 128));
        ctx->chain_ws.ensure((uint64_t)grid_s * te);
        part = ctx->chain_ws.p;
    }
    for (uint32_t nv0 = 0; nv0 < vcols; nv0 += 8) {
        if (staged) {
            switch (MT) {
                case 1: k_update_dots_s<1><<<grid_s, 128, smem_s, ctx->stream>>>(q, c, rows, qcols, vcols, nv0, v, part); break;
                case 2: k_update_dots_s<2><<<grid_s, 128, smem_s, ctx->stream>>>(q, c, rows, qcols, vcols, nv0, v, part); break;
                case 4: k_update_dots_s<4><<<grid_s, 128, smem_s, ctx->stream>>>(q, c, rows, qcols, vcols, nv0, v, part); break;
                default: k_update_dots_s<8><<<grid_s, 128, smem_s, ctx->stream>>>(q, c, rows, qcols, vcols, nv0, v, part); break;
            }
        } else switch (MT) {
            case 1: k_update_dots<1><<<grid, 256, smem, ctx->stream>>>(q, c, rows, qcols, vcols, nv0, v, part); break;
            case 2: k_update_dots<2><<<grid, 256, smem, ctx->stream>>>(q, c, rows, qcols, vcols, nv0, v, part); break;
            case 4: k_update_dots<4><<<grid, 256, smem, ctx->stream>>>(q, c, rows, qcols, vcols, nv0, v, part); break;
            default: k_update_dots<8><<<grid, 256, smem, ctx->stream>>>(q, c, rows, qcols, vcols, nv0, v, part); break;
        }
        MPKG_LAUNCH_CHECK();
        k_dots_finish<<<(te * 32 + 255) / 256, 256, 0, ctx->stream>>>(part, staged ? grid_s : grid, te, qcols, vcols, 0, nv0, c_next);
        MPKG_LAUNCH_CHECK();
        ctx->launches += 2;
    }
    timing_end(ctx, ev);
}

void gpu_icgs(mpkg_ctx_s* ctx, const double* q, uint64_t rows, uint32_t qcols, double* v, uint32_t vcols,
              int sweeps, double* coeff, const double** last_c) {
    const uint32_t ne = qcols * vcols;
    if (!ne) return;
    MPKG_CUDA(cudaMemsetAsync(coeff, 0, 8ull * ne, ctx->stream));
    ctx->ortho_c.ensure(2ull * ne);  // per-context workspace: no allocation on the steady-state path
    double* cbuf = ctx->ortho_c.p;
    double* cnext = cbuf + ne;
    auto accumulate = [&](const double* cc) {
        k_accumulate<<<(ne + 255) / 256, 256, 0, ctx->stream>>>(coeff, cc, ne);
        MPKG_LAUNCH_CHECK();
        ctx->launches += 1;
    };
    // fast mode, several sweeps: each update but the last also produces the next sweep's dots
    const bool fuse = ctx->mode == MPKG_MODE_FAST && ctx->ortho_fused != 0 && sweeps >= 2 && qcols <= 64 && rows > 0;
    bool have_c = false;  // cbuf already holds this sweep's Q^T V (from a fused update)
    for (int sw = 0; sw < sweeps; ++sw) {
        if (!have_c) gpu_block_dots(ctx, q, v, rows, qcols, vcols, cbuf);
        if (fuse && sw + 1 < sweeps) {
            gpu_update_dots(ctx, q, cbuf, rows, qcols, vcols, v, cnext);
            accumulate(cbuf);
            std::swap(cbuf, cnext);
            have_c = true;
            continue;
        }
        accumulate(cbuf);
        if (last_c && sw + 1 == sweeps) {  // the caller applies the last update (mpkg_ortho_block)
            *last_c = cbuf;
            return;
        }
        gpu_block_update(ctx, q, cbuf, rows, qcols, vcols, v);
        have_c = false;
    }
}

// sstep.hpp:539-545: ICGS against the basis, then TSQR of the block.  For s-step blocks (c <= 8,
// q <= 64) the last ICGS update runs inside TSQR's level-0 factor kernel; every result is
// bit-identical to the two calls in sequence.
void gpu_ortho_block(mpkg_ctx_s* ctx, const double* q, uint64_t rows, uint32_t qcols, double* v, uint32_t vcols,
                     int sweeps, double* coeff, double* r) {
    if (qcols == 0 || vcols == 0 || vcols > (uint32_t)kTqC || qcols > 64 || rows < vcols ||
        (rows + kTqPanel - 1) / kTqPanel <= 1) {
        if (qcols) gpu_icgs(ctx, q, rows, qcols, v, vcols, sweeps, coeff);
        gpu_tsqr(ctx, v, rows, vcols, r);
        return;
    }
    const double* last_c = nullptr;
    gpu_icgs(ctx, q, rows, qcols, v, vcols, sweeps, coeff, &last_c);
    gpu_tsqr(ctx, v, rows, vcols, r, q, last_c, qcols);
}

// Panel rows per level: shared memory holds two P x c panels in k_panel_formq.
uint32_t tsqr_panel_rows(uint32_t c) { return std::max<uint32_t>(4096u / c, 2u * c); }

void gpu_tsqr(mpkg_ctx_s* ctx, double* v, uint64_t rows, uint32_t c, double* r, const double* upd_q,
              const double* upd_coef, uint32_t upd_qcols) {
    if (!c) return;
    // c <= 8 (s-step blocks): warp-per-panel register kernels on 64-row panels; wider blocks: the
    // shared-memory CTA-per-panel kernels
    const bool narrow = c <= (uint32_t)kTqC;
    const uint32_t Pmax = narrow ? kTqPanel : tsqr_panel_rows(c);
    struct Level {
        double* a;
        uint64_t lda, rows;
        uint32_t np;
        double* taus;
        double* rstack;
    };
    // level sizes
    std::vector<Level> lv;
    std::vector<uint64_t> lv_rows, lv_np;
    uint64_t rr = rows;
    while (true) {
        const uint64_t np = std::max<uint64_t>(1, (rr + Pmax - 1) / Pmax);
        lv_rows.push_back(rr);
        lv_np.push_back(np);
        if (np == 1) break;
        rr = np * c;
    }
    uint64_t ws = (uint64_t)c * c;  // M for the top panel
    const uint64_t tslot = narrow ? 128u : c;  // narrow: compact-WY T + V_top per panel, else taus
    for (size_t L = 0; L < lv_rows.size(); ++L) ws += lv_np[L] * tslot + lv_np[L] * c * c;
    ctx->tsqr_ws.ensure(ws);  // per-context workspace, stream-ordered reuse
    double* p = ctx->tsqr_ws.p;
    double* mtop = p;
    p += (uint64_t)c * c;
    for (size_t L = 0; L < lv_rows.size(); ++L) {
        Level l{};
        l.rows = lv_rows[L];
        l.np = (uint32_t)lv_np[L];
        l.a = L == 0 ? v : lv[L - 1].rstack;
        l.lda = L == 0 ? rows : lv_rows[L];
        l.taus = p;
        p += (uint64_t)l.np * tslot;
        l.rstack = p;
        p += (uint64_t)l.np * c * c;
        lv.push_back(l);
    }
    const auto ev = timing_begin(ctx);
    if (narrow) {
        for (const Level& l : lv) {
            const unsigned g = (l.np * 32u + 127u) / 128u;
            if (upd_q && &l == &lv.front())  // level 0 of mpkg_ortho_block: ICGS's last update fused in
                k_tsqr_factor<true><<<g, 128, 64ull * upd_qcols, ctx->stream>>>(l.a, l.lda, l.rows, l.np, c, l.rstack,
                                                                             l.taus, upd_q, upd_coef, upd_qcols);
            else
                k_tsqr_factor<false><<<g, 128, 0, ctx->stream>>>(l.a, l.lda, l.rows, l.np, c, l.rstack, l.taus,
                                                              nullptr, nullptr, 0);
            MPKG_LAUNCH_CHECK();
        }
        k_sign_fix<<<1, 256, 0, ctx->stream>>>(lv.back().rstack, c, r, mtop);
        MPKG_LAUNCH_CHECK();
        const double* m = mtop;
        uint64_t ldm = c;
        for (size_t L = lv.size(); L-- > 0;) {
            const Level& l = lv[L];
            k_tsqr_apply<<<(l.np * kSub * 32u + 127u) / 128u, 128, 0, ctx->stream>>>(l.a, l.lda, l.rows, l.np, c,
                                                                           l.taus, m, ldm);
            MPKG_LAUNCH_CHECK();
            m = l.a;
            ldm = l.lda;
        }
        ctx->launches += 2 * lv.size() + 1;
        timing_end(ctx, ev);
        return;
    }
    size_t smem_max = 0;
    for (const Level& l : lv) {
        const uint64_t pr = (l.rows + l.np - 1) / l.np;
        smem_max = std::max<size_t>(smem_max, 16ull * c * pr);
    }
    MPKG_CUDA(cudaFuncSetAttribute(k_panel_qr, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_max));
    MPKG_CUDA(cudaFuncSetAttribute(k_panel_formq, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_max));
    for (const Level& l : lv) {
        const uint64_t pr = (l.rows + l.np - 1) / l.np;
        k_panel_qr<<<l.np, 256, 8ull * c * pr, ctx->stream>>>(l.a, l.lda, l.rows, l.np, c, l.taus, l.rstack);
        MPKG_LAUNCH_CHECK();
    }
    k_sign_fix<<<1, 256, 0, ctx->stream>>>(lv.back().rstack, c, r, mtop);
    MPKG_LAUNCH_CHECK();
    const double* m = mtop;
    uint64_t ldm = c;
    for (size_t L = lv.size(); L-- > 0;) {
        const Level& l = lv[L];
        const uint64_t pr = (l.rows + l.np - 1) / l.np;
        k_panel_formq<<<l.np, 256, 16ull * c * pr, ctx->stream>>>(l.a, l.lda, l.rows, l.np, c, l.taus, m, ldm);
        MPKG_LAUNCH_CHECK();
        m = l.a;
        ldm = l.lda;
    }
    ctx->launches += 2 * lv.size() + 1;
    timing_end(ctx, ev);
}

}  // namespace mpkg_detail
