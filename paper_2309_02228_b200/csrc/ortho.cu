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
template <int MT>
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
        if (i0 + 3 < rows) {
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
    const uint32_t e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= tile_entries) return;
    const uint32_t mt = e / 64, m = (e % 64) / 8, n = e % 8;
    const uint32_t k = mq0 + mt * 8 + m, j = nv0 + n;
    if (k >= qcols || j >= vcols) return;
    double s = 0.0;
    for (uint32_t b = 0; b < n_parts; ++b) s += part[(uint64_t)b * tile_entries + e];
    c[(uint64_t)j * qcols + k] = s;
}

// ---- block_update (bitwise in both modes) --------------------------------------------------
// v_j[i] <- v_j[i] - c_jk q_k[i] for k = 0..qcols-1 ascending (ortho.hpp:83-90).  A thread owns
// row i for up to 8 v columns [j0, j0 + 8); the coefficients sit in shared memory.
template <int VT>
__global__ void __launch_bounds__(256) k_update(const double* __restrict__ q, const double* __restrict__ c,
                                                uint64_t rows, uint32_t qcols, uint32_t vcols,
                                                uint32_t j0, double* __restrict__ v) {
    extern __shared__ double cs[];  // [VT][qcols]
    for (uint32_t e = threadIdx.x; e < VT * qcols; e += blockDim.x) {
        const uint32_t jj = e / qcols, k = e % qcols;
        cs[e] = j0 + jj < vcols ? c[(uint64_t)(j0 + jj) * qcols + k] : 0.0;
    }
    __syncthreads();
    const uint32_t nv = vcols - j0 < (uint32_t)VT ? vcols - j0 : (uint32_t)VT;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < rows;
         i += (uint64_t)gridDim.x * blockDim.x) {
        double x[VT];
#pragma unroll
        for (int jj = 0; jj < VT; ++jj) x[jj] = jj < (int)nv ? __ldcs(v + (uint64_t)(j0 + jj) * rows + i) : 0.0;
        uint32_t k = 0;
        for (; k + 4 <= qcols; k += 4) {
            double qk[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) qk[u] = __ldg(q + (uint64_t)(k + u) * rows + i);
#pragma unroll
            for (int u = 0; u < 4; ++u)
#pragma unroll
                for (int jj = 0; jj < VT; ++jj) x[jj] = __dsub_rn(x[jj], __dmul_rn(cs[jj * qcols + k + u], qk[u]));
        }
        for (; k < qcols; ++k) {
            const double qk = __ldg(q + (uint64_t)k * rows + i);
#pragma unroll
            for (int jj = 0; jj < VT; ++jj) x[jj] = __dsub_rn(x[jj], __dmul_rn(cs[jj * qcols + k], qk));
        }
#pragma unroll
        for (int jj = 0; jj < VT; ++jj)
            if (jj < (int)nv) __stcs(v + (uint64_t)(j0 + jj) * rows + i, x[jj]);
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
                switch (MT) {
                    case 1: k_dots_mma<1><<<grid, 256, 0, ctx->stream>>>(q, v, rows, qcols, vcols, mq0, nv0, part); break;
                    case 2: k_dots_mma<2><<<grid, 256, 0, ctx->stream>>>(q, v, rows, qcols, vcols, mq0, nv0, part); break;
                    case 4: k_dots_mma<4><<<grid, 256, 0, ctx->stream>>>(q, v, rows, qcols, vcols, mq0, nv0, part); break;
                    default: k_dots_mma<8><<<grid, 256, 0, ctx->stream>>>(q, v, rows, qcols, vcols, mq0, nv0, part); break;
                }
                MPKG_LAUNCH_CHECK();
                k_dots_finish<<<(te + 127) / 128, 128, 0, ctx->stream>>>(part, grid, te, qcols, vcols, mq0, nv0, c);
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

void gpu_icgs(mpkg_ctx_s* ctx, const double* q, uint64_t rows, uint32_t qcols, double* v, uint32_t vcols,
              int sweeps, double* coeff) {
    const uint32_t ne = qcols * vcols;
    if (!ne) return;
    MPKG_CUDA(cudaMemsetAsync(coeff, 0, 8ull * ne, ctx->stream));
    ctx->ortho_c.ensure(ne);  // per-context workspace: no allocation on the steady-state path
    double* cbuf = ctx->ortho_c.p;
    for (int sw = 0; sw < sweeps; ++sw) {
        gpu_block_dots(ctx, q, v, rows, qcols, vcols, cbuf);
        gpu_block_update(ctx, q, cbuf, rows, qcols, vcols, v);
        k_accumulate<<<(ne + 255) / 256, 256, 0, ctx->stream>>>(coeff, cbuf, ne);
        MPKG_LAUNCH_CHECK();
        ctx->launches += 1;
    }
}

// Panel rows per level: shared memory holds two P x c panels in k_panel_formq.
uint32_t tsqr_panel_rows(uint32_t c) { return std::max<uint32_t>(4096u / c, 2u * c); }

void gpu_tsqr(mpkg_ctx_s* ctx, double* v, uint64_t rows, uint32_t c, double* r) {
    if (!c) return;
    const uint32_t Pmax = tsqr_panel_rows(c);
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
    for (size_t L = 0; L < lv_rows.size(); ++L) ws += lv_np[L] * c + lv_np[L] * c * c;
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
        p += (uint64_t)l.np * c;
        l.rstack = p;
        p += (uint64_t)l.np * c * c;
        lv.push_back(l);
    }
    const auto ev = timing_begin(ctx);
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
