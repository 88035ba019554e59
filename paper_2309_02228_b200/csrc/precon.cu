// Jacobi-preconditioned chains on the GPU (reference jacobi.hpp and the
// s-step chain of sstep.hpp:68-157).  Every stage is one row-parallel launch over the matrix's
// SELL copy with the reference's per-row formula, so the results are bit-identical to the
// reference's sequential and cache-blocked paths (jacobi.hpp states both are bitwise equal):
//   scaled SpMV     acc += a_rk * (d_c * x_c)                     jacobi.hpp:100-110
//   Jacobi sweep    z_r = d_r v_r - d_r * sum_{k != diag} a_rk z_k  jacobi.hpp:83-96
//   diagonal scale  z_r = d_r v_r                                 jacobi.hpp:114-117
//   terminal        y_r = sum_k a_rk z_k  (- a src_r (+ b2 src2_r))  csr.hpp:115-123, sstep.hpp:68-88
// each a sequential stored-order accumulation with __dmul_rn / __dadd_rn (no FMA).
#include <cub/device/device_scan.cuh>

#include "device.h"
#include "rowdot.cuh"

namespace mpkg_detail {

namespace {

constexpr uint32_t kNoDiag = 0xffffffffu;  // csr.hpp:231

// csr.hpp:233-243 diagonal_positions (lower_bound in the sorted row) + jacobi.hpp:48-64.
__global__ void k_diag_info(const uint32_t* __restrict__ rp, const uint32_t* __restrict__ ci,
                            const double* __restrict__ v, uint32_t n, uint32_t* __restrict__ pos,
                            uint32_t* __restrict__ kd, double* __restrict__ inv,
                            uint32_t* __restrict__ bad_missing, uint32_t* __restrict__ bad_zero) {
    for (uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r < n;
         r += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t lo = rp[r], hi = rp[r + 1];
        const uint32_t b = lo, e = hi;
        while (lo < hi) {
            const uint32_t mid = lo + ((hi - lo) >> 1);
            if (ci[mid] < r)
                lo = mid + 1;
            else
                hi = mid;
        }
        const bool found = lo < e && ci[lo] == r;
        pos[r] = found ? lo : kNoDiag;
        kd[r] = found ? lo - b : kNoDiag;
        if (!found) {
            atomicMin(bad_missing, (uint32_t)r);
            inv[r] = 0.0;
        } else if (v[lo] == 0.0) {
            atomicMin(bad_zero, (uint32_t)r);
            inv[r] = 0.0;
        } else {
            inv[r] = __ddiv_rn(1.0, v[lo]);
        }
    }
}

__global__ void k_diag_scale(uint32_t n, const double* __restrict__ d, const double* __restrict__ v,
                             double* __restrict__ z) {
    for (uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r < n;
         r += (uint64_t)gridDim.x * blockDim.x)
        z[r] = __dmul_rn(d[r], v[r]);
}

enum { kPlain = 0, kScaled = 1, kSkipDiag = 2, kRange = 3 };
enum { kEpiStore = 0, kEpiJacobi = 1, kEpiShift = 2, kEpiResid = 3 };

// Stored-order row dot over SELL-32 (layout in rowdot.cuh), groups of 8 entries in flight.
// kScaled gathers d_c and x_c and forms d_c * x_c first (the reference's parenthesisation);
// kSkipDiag leaves out the row's diagonal entry (index kskip inside the row); kRange keeps only
// the entries [kb, ke) of the row (GS2's strict lower / upper part).
template <int MODE>
__device__ __forceinline__ double pc_row_dot(const uint32_t* __restrict__ cols,
                                             const double* __restrict__ vals, uint64_t off,
                                             uint32_t L, uint32_t lane, uint32_t len,
                                             const double* __restrict__ src,
                                             const double* __restrict__ d, uint32_t kskip,
                                             uint32_t kb = 0, uint32_t ke = 0xffffffffu) {
    constexpr int G = 8;
    double acc = 0.0;
    const uint32_t Lp = L & ~1u;
    for (uint32_t k0 = 0; k0 < len; k0 += G) {
        uint32_t c[G];
        double v[G], x[G];
#pragma unroll
        for (int j = 0; j < G; j += 2) {  // whole SELL pairs: one 8 B + one 16 B load
            const uint32_t k = k0 + j;
            if (k + 1 < Lp) {
                const uint64_t e = off + (k >> 1) * 64u + lane * 2u;
                const uint2 cc = __ldg(reinterpret_cast<const uint2*>(cols + e));
                const double2 vv = __ldg(reinterpret_cast<const double2*>(vals + e));
                c[j] = cc.x, c[j + 1] = cc.y, v[j] = vv.x, v[j + 1] = vv.y;
            } else {
#pragma unroll
                for (int i = 0; i < 2; ++i) {
                    const uint32_t kk = k + i;
                    const uint64_t e = off + sell_pos(kk, Lp, lane);
                    c[j + i] = kk < len ? __ldg(cols + e) : 0u;
                    v[j + i] = kk < len ? __ldg(vals + e) : 0.0;
                }
            }
        }
#pragma unroll
        for (int j = 0; j < G; ++j) {
            const bool use = k0 + j < len && (MODE != kSkipDiag || k0 + j != kskip) &&
                             (MODE != kRange || (k0 + j >= kb && k0 + j < ke));
            x[j] = use ? __ldg(src + c[j]) : 0.0;
            if (MODE == kScaled && use) x[j] = __dmul_rn(__ldg(d + c[j]), x[j]);
        }
#pragma unroll
        for (int j = 0; j < G; ++j)
            if (k0 + j < len && (MODE != kSkipDiag || k0 + j != kskip) &&
                (MODE != kRange || (k0 + j >= kb && k0 + j < ke)))
                acc = __dadd_rn(acc, __dmul_rn(v[j], x[j]));
    }
    return acc;
}

// One stage over every row of the identity-order SELL.
template <int MODE, int EPI>
__global__ void __launch_bounds__(256) k_pc_stage(
    const uint32_t* __restrict__ cols, const double* __restrict__ vals,
    const uint64_t* __restrict__ chunk_off, const uint32_t* __restrict__ row_len, uint32_t n,
    const double* __restrict__ src, const double* __restrict__ d, const uint32_t* __restrict__ kd,
    const double* __restrict__ v, const double* __restrict__ own, const double* __restrict__ own2,
    double a, double b2, double* __restrict__ dst) {
    for (uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r < n;
         r += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t len = row_len[r];
        const uint64_t off = chunk_off[r >> 5];
        const uint32_t L = (uint32_t)((chunk_off[(r >> 5) + 1] - off) >> 5);
        const double acc = pc_row_dot<MODE>(cols, vals, off, L, (uint32_t)(r & 31), len, src, d,
                                            MODE == kSkipDiag ? kd[r] : 0u);
        double out;
        if constexpr (EPI == kEpiResid)
            out = __dsub_rn(v[r], acc);
        else if constexpr (EPI == kEpiJacobi)
            out = __dsub_rn(__dmul_rn(d[r], v[r]), __dmul_rn(d[r], acc));
        else if constexpr (EPI == kEpiShift)
            out = shift_epilogue(acc, a, b2, own[r], b2 != 0.0 ? own2[r] : 0.0);
        else
            out = acc;
        dst[r] = out;
    }
}

// GS2 stage 0 (gs2.hpp:70-82): g = d_r (v_r - sum_k a_rk z_k) over the full row;
// inner iteration j (gs2.hpp:89-104): g = g0_r - d_r * sum_{k in lower/upper} a_rk g_prev_k.
// The iterate update z_next = z_prev + g is fused into the last stage of a sweep.
template <bool INNER>
__global__ void __launch_bounds__(256) k_gs2_stage(
    const uint32_t* __restrict__ cols, const double* __restrict__ vals,
    const uint64_t* __restrict__ chunk_off, const uint32_t* __restrict__ row_len, uint32_t n,
    const double* __restrict__ src, const double* __restrict__ d, const uint32_t* __restrict__ kd,
    bool forward, const double* __restrict__ v, const double* __restrict__ g0,
    double* __restrict__ g_out, const double* __restrict__ z_prev, double* __restrict__ z_next) {
    for (uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r < n;
         r += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t len = row_len[r];
        const uint64_t off = chunk_off[r >> 5];
        const uint32_t L = (uint32_t)((chunk_off[(r >> 5) + 1] - off) >> 5);
        double g;
        if constexpr (INNER) {
            const uint32_t kb = forward ? 0u : kd[r] + 1u, ke = forward ? kd[r] : len;
            const double acc = pc_row_dot<kRange>(cols, vals, off, L, (uint32_t)(r & 31), len, src, d, 0u, kb, ke);
            g = __dsub_rn(g0[r], __dmul_rn(d[r], acc));
        } else {
            const double acc = pc_row_dot<kPlain>(cols, vals, off, L, (uint32_t)(r & 31), len, src, d, 0u);
            g = __dmul_rn(d[r], __dsub_rn(v[r], acc));
        }
        g_out[r] = g;
        if (z_next) z_next[r] = __dadd_rn(z_prev[r], g);
    }
}

// Grow-only per-context workspace for the chains' intermediate vectors (no allocation per call).
double* chain_workspace(mpkg_ctx_s* ctx, uint64_t count) {
    ctx->chain_ws.ensure(std::max<uint64_t>(count, 1));
    return ctx->chain_ws.p;
}

// Product-form polynomial terminal (poly.hpp:200-224): t = A z_src (scaled for the fused
// one-sweep Jacobi inner), then the root update for the power's role (0 real, 1 first / 2 second
// member of a conjugate pair) into w_out and the accumulated result acc.
template <bool FUSED>
__global__ void __launch_bounds__(256) k_poly_terminal(
    const uint32_t* __restrict__ cols, const double* __restrict__ vals,
    const uint64_t* __restrict__ chunk_off, const uint32_t* __restrict__ row_len, uint32_t n,
    const double* __restrict__ z_src, const double* __restrict__ d, int role, double re, double mod,
    const double* __restrict__ w_in, const double* __restrict__ w_pm2, double* __restrict__ w_out,
    double* __restrict__ acc) {
    for (uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r < n;
         r += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t len = row_len[r];
        const uint64_t off = chunk_off[r >> 5];
        const uint32_t L = (uint32_t)((chunk_off[(r >> 5) + 1] - off) >> 5);
        const double t = pc_row_dot<FUSED ? kScaled : kPlain>(cols, vals, off, L, (uint32_t)(r & 31), len,
                                                             z_src, d, 0u);
        if (role == 0) {
            acc[r] = __dadd_rn(acc[r], __ddiv_rn(w_in[r], re));
            w_out[r] = __dsub_rn(w_in[r], __ddiv_rn(t, re));
        } else if (role == 1) {
            const double u = __dsub_rn(__dmul_rn(__dmul_rn(2.0, re), w_in[r]), t);
            w_out[r] = u;
            acc[r] = __dadd_rn(acc[r], __ddiv_rn(u, mod));
        } else {
            w_out[r] = __dsub_rn(w_pm2[r], __ddiv_rn(t, mod));
        }
    }
}

__global__ void k_poly_tail(uint32_t n, const double* __restrict__ w, double th, double* __restrict__ acc) {
    for (uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r < n;
         r += (uint64_t)gridDim.x * blockDim.x)
        acc[r] = __dadd_rn(acc[r], __ddiv_rn(w[r], th));
}

struct Stage {
    mpkg_ctx_s* ctx;
    const Sell& S;
    uint32_t n;
    unsigned grid() const { return grid_for(n, 256, (unsigned)ctx->sm_count * 8u); }
};

template <int MODE, int EPI>
void stage(const Stage& st, const double* src, const mpkg_jacobi_s* J, const double* v,
           const double* own, const double* own2, double a, double b2, double* dst) {
    const auto ev = timing_begin(st.ctx);
    k_pc_stage<MODE, EPI><<<st.grid(), 256, 0, st.ctx->stream>>>(
        st.S.cols.p, st.S.vals.p, st.S.chunk_off.p, st.S.row_len.p, st.n, src, J->inv.p, J->kdiag.p,
        v, own, own2, a, b2, dst);
    MPKG_LAUNCH_CHECK();
    timing_end(st.ctx, ev);
    st.ctx->launches += 1;
}

void scale(mpkg_ctx_s* ctx, const mpkg_jacobi_s* J, const double* v, double* z) {
    k_diag_scale<<<grid_for(J->n, 256, (unsigned)ctx->sm_count * 8u), 256, 0, ctx->stream>>>(
        J->n, J->inv.p, v, z);
    MPKG_LAUNCH_CHECK();
    ctx->launches += 1;
}

// z^1 = D^{-1} v, z^{j+1} = sweep(z^j) for j < sweeps: leaves z^sweeps in the returned buffer
// (one of the two workspace slices).
const double* jacobi_chain(mpkg_ctx_s* ctx, const mpkg_jacobi_s* J, const Stage& st, const double* v,
                           double* w0, double* w1) {
    scale(ctx, J, v, w0);
    double* cur = w0;
    double* nxt = w1;
    for (int j = 1; j < J->sweeps; ++j) {
        stage<kSkipDiag, kEpiJacobi>(st, cur, J, v, nullptr, nullptr, 0.0, 0.0, nxt);
        std::swap(cur, nxt);
    }
    return cur;
}

// One K-sweep GS2 from z[0]: z holds K+1 slices, g gamma+1 slices (gs2.hpp:126-158 in order).
void gs2_sweeps(const Stage& st, const mpkg_gs2_s* G, const double* v, double* z, double* g) {
    const uint32_t n = st.n;
    for (int p = 1; p <= G->sweeps; ++p) {
        const double* z_prev = z + (uint64_t)(p - 1) * n;
        double* z_next = z + (uint64_t)p * n;
        auto launch = [&](auto inner, const double* src, const double* gprev, double* gout, double* zn) {
            constexpr bool I = decltype(inner)::value;
            const auto ev = timing_begin(st.ctx);
            k_gs2_stage<I><<<st.grid(), 256, 0, st.ctx->stream>>>(
                st.S.cols.p, st.S.vals.p, st.S.chunk_off.p, st.S.row_len.p, n, src, G->diag.inv.p,
                G->diag.kdiag.p, G->forward, v, g, gout, z_prev, zn);
            MPKG_LAUNCH_CHECK();
            timing_end(st.ctx, ev);
            st.ctx->launches += 1;
            (void)gprev;
        };
        launch(std::false_type{}, z_prev, nullptr, g, G->gamma == 0 ? z_next : nullptr);
        for (int j = 1; j <= G->gamma; ++j)
            launch(std::true_type{}, g + (uint64_t)(j - 1) * n, nullptr, g + (uint64_t)j * n,
                   j == G->gamma ? z_next : nullptr);
    }
}

// One zero-guess GS2 sweep z[0] (all zero) -> z[1] with the g bank (the polynomial's inner,
// poly.hpp:168-187).
void gs2_single_sweep(const Stage& st, const mpkg_gs2_s* G, const double* v, double* z, double* g) {
    const uint32_t n = st.n;
    auto launch = [&](auto inner, const double* src, double* gout, double* zn) {
        constexpr bool I = decltype(inner)::value;
        const auto ev = timing_begin(st.ctx);
        k_gs2_stage<I><<<st.grid(), 256, 0, st.ctx->stream>>>(
            st.S.cols.p, st.S.vals.p, st.S.chunk_off.p, st.S.row_len.p, n, src, G->diag.inv.p,
            G->diag.kdiag.p, G->forward, v, g, gout, z, zn);
        MPKG_LAUNCH_CHECK();
        timing_end(st.ctx, ev);
        st.ctx->launches += 1;
    };
    launch(std::false_type{}, z, g, G->gamma == 0 ? z + n : nullptr);
    for (int j = 1; j <= G->gamma; ++j)
        launch(std::true_type{}, g + (uint64_t)(j - 1) * n, g + (uint64_t)j * n, j == G->gamma ? z + n : nullptr);
}

}  // namespace

void gpu_gs2_chain(mpkg_ctx_s* ctx, const mpkg_gs2_s* G, mpkg_csr_s* A, const double* d_v,
                   double* d_z, int terminal, double* d_out) {
    const uint32_t n = G->diag.n;
    if (n == 0) return;
    const Stage st{ctx, csr_sell(A), n};
    double* ws = chain_workspace(ctx, (uint64_t)(G->sweeps + G->gamma + 2) * n);
    double* zb = ws;
    double* gb = ws + (uint64_t)(G->sweeps + 1) * n;
    MPKG_CUDA(cudaMemcpyAsync(zb, d_z, 8ull * n, cudaMemcpyDeviceToDevice, ctx->stream));
    gs2_sweeps(st, G, d_v, zb, gb);
    const double* zk = zb + (uint64_t)G->sweeps * n;
    const mpkg_jacobi_s* J = &G->diag;
    if (terminal == 1)  // gs2.hpp:147-149 apply_a
        stage<kPlain, kEpiStore>(st, zk, J, nullptr, nullptr, nullptr, 0.0, 0.0, d_out);
    else if (terminal == 2)  // residual_rows
        stage<kPlain, kEpiResid>(st, zk, J, d_v, nullptr, nullptr, 0.0, 0.0, d_out);
    MPKG_CUDA(cudaMemcpyAsync(d_z, zk, 8ull * n, cudaMemcpyDeviceToDevice, ctx->stream));
    MPKG_CUDA(cudaStreamSynchronize(ctx->stream));
}

void gpu_sstep_gs2(mpkg_ctx_s* ctx, const mpkg_gs2_s* G, mpkg_csr_s* A, double* d_block,
                   uint64_t rows, int ns, const double* a, const double* b2) {
    const uint32_t n = G->diag.n;
    if (n == 0) return;
    const Stage st{ctx, csr_sell(A), n};
    double* ws = chain_workspace(ctx, (uint64_t)(G->sweeps + G->gamma + 2) * n);
    double* zb = ws;
    double* gb = ws + (uint64_t)(G->sweeps + 1) * n;
    MPKG_CUDA(cudaMemsetAsync(zb, 0, 8ull * n, ctx->stream));  // slice 0: the permanent zero guess
    for (int p = 1; p <= ns; ++p) {
        const double* src = d_block + (uint64_t)(p - 1) * rows;
        const double* src2 = p >= 2 ? d_block + (uint64_t)(p - 2) * rows : src;
        gs2_sweeps(st, G, src, zb, gb);
        stage<kPlain, kEpiShift>(st, zb + (uint64_t)G->sweeps * n, &G->diag, nullptr, src, src2,
                                 a[p - 1], b2[p - 1], d_block + (uint64_t)p * rows);
    }
    MPKG_CUDA(cudaStreamSynchronize(ctx->stream));
}

void gpu_poly_apply(mpkg_ctx_s* ctx, mpkg_csr_s* A, const mpkg_jacobi_s* J, const mpkg_gs2_s* G,
                    const double* re, const double* im, const uint8_t* role, int degree,
                    const double* d_v, double* d_z) {
    const uint32_t n = A->n_rows;
    if (n == 0) return;
    const Stage st{ctx, csr_sell(A), n};
    // workspace: degree w slices | 2 inner slices (Jacobi ping-pong or GS2 {zero, z1}) | g bank
    const int gamma = G ? G->gamma : 0;
    double* ws = chain_workspace(ctx, (uint64_t)(degree + 2 + gamma + 1) * n);
    double* w = ws;
    double* zb = ws + (uint64_t)degree * n;
    double* gb = zb + 2ull * n;
    MPKG_CUDA(cudaMemcpyAsync(w, d_v, 8ull * n, cudaMemcpyDeviceToDevice, ctx->stream));
    MPKG_CUDA(cudaMemsetAsync(d_z, 0, 8ull * n, ctx->stream));
    if (G) MPKG_CUDA(cudaMemsetAsync(zb, 0, 8ull * n, ctx->stream));  // GS2's permanent zero guess
    for (int pw = 1; pw <= degree - 1; ++pw) {
        const double* w_in = w + (uint64_t)(pw - 1) * n;
        const double* z_src = w_in;
        bool fused = false;
        const double* dinv = nullptr;
        if (J) {  // poly.hpp:150-167
            if (J->sweeps == 1) {
                fused = true;
                dinv = J->inv.p;
            } else {
                z_src = jacobi_chain(ctx, J, st, w_in, zb, zb + n);
            }
        } else if (G) {  // poly.hpp:168-187: one zero-guess GS2 sweep into zb[1]
            gs2_single_sweep(st, G, w_in, zb, gb);
            z_src = zb + n;
        }
        const double th = re[pw - 1];
        const double mod = th * th + im[pw - 1] * im[pw - 1];  // poly.hpp:193 (host, no FMA)
        const double* w_pm2 = pw >= 2 ? w + (uint64_t)(pw - 2) * n : w_in;
        double* w_out = w + (uint64_t)pw * n;
        const auto ev = timing_begin(ctx);
        if (fused)
            k_poly_terminal<true><<<st.grid(), 256, 0, ctx->stream>>>(
                st.S.cols.p, st.S.vals.p, st.S.chunk_off.p, st.S.row_len.p, n, z_src, dinv, role[pw - 1], th,
                mod, w_in, w_pm2, w_out, d_z);
        else
            k_poly_terminal<false><<<st.grid(), 256, 0, ctx->stream>>>(
                st.S.cols.p, st.S.vals.p, st.S.chunk_off.p, st.S.row_len.p, n, z_src, nullptr, role[pw - 1], th,
                mod, w_in, w_pm2, w_out, d_z);
        MPKG_LAUNCH_CHECK();
        timing_end(ctx, ev);
        ctx->launches += 1;
    }
    if (role[degree - 1] == 0) {  // poly.hpp:271-278 trailing real root
        k_poly_tail<<<grid_for(n, 256, (unsigned)ctx->sm_count * 8u), 256, 0, ctx->stream>>>(
            n, w + (uint64_t)(degree - 1) * n, re[degree - 1], d_z);
        MPKG_LAUNCH_CHECK();
        ctx->launches += 1;
    }
    MPKG_CUDA(cudaStreamSynchronize(ctx->stream));
}

void gpu_jacobi_setup(mpkg_ctx_s* ctx, const mpkg_csr_s* A, mpkg_jacobi_s* J) {
    const uint32_t n = A->n_rows;
    cudaStream_t st = ctx->stream;
    J->n = n;
    J->pos.alloc(std::max<uint32_t>(n, 1));
    J->kdiag.alloc(std::max<uint32_t>(n, 1));
    J->inv.alloc(std::max<uint32_t>(n, 1));
    if (n == 0) return;
    DevBuf<uint32_t> bad(2);
    MPKG_CUDA(cudaMemsetAsync(bad.p, 0xff, 8, st));
    k_diag_info<<<grid_for(n, 256, (unsigned)ctx->sm_count * 8u), 256, 0, st>>>(
        A->row_ptr.p, A->col_idx.p, A->values.p, n, J->pos.p, J->kdiag.p, J->inv.p, bad.p, bad.p + 1);
    MPKG_LAUNCH_CHECK();
    ctx->launches += 1;
    uint32_t h[2];
    MPKG_CUDA(cudaMemcpyAsync(h, bad.p, 8, cudaMemcpyDeviceToHost, st));
    MPKG_CUDA(cudaStreamSynchronize(st));
    // jacobi.hpp:54-61 reports the FIRST failing row, whichever the failure
    if (h[0] != kNoDiag && h[0] <= h[1])
        fail(MPKG_EINTERNAL, "jacobi_setup: missing diagonal entry at row " + std::to_string(h[0]));
    if (h[1] != kNoDiag)
        fail(MPKG_EINTERNAL, "jacobi_setup: zero diagonal entry at row " + std::to_string(h[1]));
}

void gpu_jacobi_apply(mpkg_ctx_s* ctx, const mpkg_jacobi_s* J, mpkg_csr_s* A, const double* d_v,
                      double* d_z) {
    const uint32_t n = J->n;
    if (n == 0) return;
    double* w = chain_workspace(ctx, 2ull * n);
    const Stage st{ctx, csr_sell(A), n};
    const double* z = jacobi_chain(ctx, J, st, d_v, w, w + n);
    MPKG_CUDA(cudaMemcpyAsync(d_z, z, 8ull * n, cudaMemcpyDeviceToDevice, ctx->stream));
    MPKG_CUDA(cudaStreamSynchronize(ctx->stream));
}

void gpu_jacobi_op(mpkg_ctx_s* ctx, const mpkg_jacobi_s* J, mpkg_csr_s* A, const double* d_v,
                   double* d_y) {
    const uint32_t n = J->n;
    if (n == 0) return;
    const Stage st{ctx, csr_sell(A), n};
    if (J->sweeps == 1) {  // jacobi.hpp:133-136: one fused-scaling stage
        stage<kScaled, kEpiStore>(st, d_v, J, nullptr, nullptr, nullptr, 0.0, 0.0, d_y);
        return;
    }
    double* w = chain_workspace(ctx, 2ull * n);
    const double* z = jacobi_chain(ctx, J, st, d_v, w, w + n);
    stage<kPlain, kEpiStore>(st, z, J, nullptr, nullptr, nullptr, 0.0, 0.0, d_y);
    MPKG_CUDA(cudaStreamSynchronize(ctx->stream));
}

void gpu_sstep_jacobi(mpkg_ctx_s* ctx, const mpkg_jacobi_s* J, mpkg_csr_s* A, double* d_block,
                      uint64_t rows, int ns, const double* a, const double* b2) {
    const uint32_t n = J->n;
    if (n == 0) return;
    const Stage st{ctx, csr_sell(A), n};
    double* w = chain_workspace(ctx, 2ull * n);
    for (int p = 1; p <= ns; ++p) {
        const double* src = d_block + (uint64_t)(p - 1) * rows;
        const double* src2 = p >= 2 ? d_block + (uint64_t)(p - 2) * rows : src;
        double* dst = d_block + (uint64_t)p * rows;
        if (J->sweeps == 1) {  // sstep.hpp:91-116 scaled_shifted_spmv_rows
            stage<kScaled, kEpiShift>(st, src, J, nullptr, src, src2, a[p - 1], b2[p - 1], dst);
        } else {  // stage 0, sweeps, then sstep.hpp:68-88 shifted_terminal_rows on z^sweeps
            const double* z = jacobi_chain(ctx, J, st, src, w, w + n);
            stage<kPlain, kEpiShift>(st, z, J, nullptr, src, src2, a[p - 1], b2[p - 1], dst);
        }
    }
    MPKG_CUDA(cudaStreamSynchronize(ctx->stream));
}

}  // namespace mpkg_detail
