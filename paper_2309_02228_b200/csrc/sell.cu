// SELL-32 construction from a device CSR, and the one-launch-per-power row kernel used by
// spmv / baseline_mpk (csr.hpp:126-142, mpk.hpp:59-75, mpk.hpp:160-180).
#include <cub/device/device_scan.cuh>

#include "device.h"
#include "rowdot.cuh"

namespace mpkg_detail {

namespace {

__global__ void k_sell_lengths(const uint32_t* __restrict__ rp, uint32_t n_rows,
                               const uint32_t* __restrict__ slot_row, uint32_t n_slots,
                               uint32_t* __restrict__ row_len) {
    for (uint64_t s = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; s < n_slots;
         s += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t r = slot_row ? slot_row[s] : (uint32_t)s;
        row_len[s] = r < n_rows ? rp[r + 1] - rp[r] : 0u;
    }
}

// One warp per chunk: L = max row length in the chunk; entries = 32*L.
// Rows longer than `cap` ("long rows") are left out of the SELL arrays; the fused kernel
// processes them CTA-cooperatively from the CSR (mpk_exec.cu).
__global__ void k_sell_chunk_sizes(const uint32_t* __restrict__ row_len, uint32_t n_chunks,
                                   uint32_t cap, uint64_t* __restrict__ chunk_entries) {
    const uint32_t lane = threadIdx.x & 31;
    for (uint64_t c = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5; c < n_chunks;
         c += ((uint64_t)gridDim.x * blockDim.x) >> 5) {
        uint32_t L = row_len[c * 32 + lane];
        if (L > cap) L = 0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) L = max(L, __shfl_xor_sync(0xffffffffu, L, o));
        if (lane == 0) chunk_entries[c] = 32ull * L;
    }
}

__global__ void k_sell_fill(const uint32_t* __restrict__ rp, const uint32_t* __restrict__ ci,
                            const double* __restrict__ v, uint32_t n_rows,
                            const uint32_t* __restrict__ slot_row,
                            const uint64_t* __restrict__ chunk_off,
                            const uint32_t* __restrict__ row_len, uint32_t n_slots, uint32_t cap,
                            const uint32_t* __restrict__ col_map, uint32_t* __restrict__ cols,
                            double* __restrict__ vals) {
    for (uint64_t s = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; s < n_slots;
         s += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t len = row_len[s];
        if (len == 0 || len > cap) continue;
        const uint32_t r = slot_row ? slot_row[s] : (uint32_t)s;
        const uint64_t c = s >> 5;
        const uint32_t lane = (uint32_t)(s & 31);
        const uint64_t off = chunk_off[c];
        const uint32_t L = (uint32_t)((chunk_off[c + 1] - off) >> 5);
        const uint32_t Lp = L & ~1u;
        const uint32_t b = rp[r];
        for (uint32_t k = 0; k < len; ++k) {
            const uint64_t e = off + sell_pos(k, Lp, lane);
            cols[e] = col_map ? col_map[ci[b + k]] : ci[b + k];
            vals[e] = v[b + k];
        }
    }
}

// KIND 0: dst = A src; KIND 1: shifted epilogue (mpk.hpp:135-153).
template <int KIND>
__global__ void __launch_bounds__(256) k_spmv_sell(
    const uint32_t* __restrict__ cols, const double* __restrict__ vals,
    const uint64_t* __restrict__ chunk_off, const uint32_t* __restrict__ row_len,
    const uint32_t* __restrict__ slot_row, uint32_t n_slots, uint32_t n_rows,
    const double* __restrict__ src, double* __restrict__ dst, const double* __restrict__ src2,
    double a, double b2) {
    MPKG_PDL_ENTRY();
    for (uint64_t s = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; s < n_slots;
         s += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t len = row_len[s];
        const uint32_t r = slot_row ? slot_row[s] : (uint32_t)s;
        const uint64_t c = s >> 5;
        const uint64_t off = chunk_off[c];
        const uint32_t L = (uint32_t)((chunk_off[c + 1] - off) >> 5);
        if (r >= n_rows) continue;  // padding slot
        double acc = sell_row_dot<true, 8>(cols, vals, off, L, (uint32_t)(s & 31), len, src,
                                           l2_policy_first());
        if (KIND == 1)
            acc = shift_epilogue(acc, a, b2, __ldg(src + r), b2 != 0.0 ? __ldg(src2 + r) : 0.0);
        dst[r] = acc;
    }
}

}  // namespace

void build_sell(mpkg_ctx_s* ctx, const mpkg_csr_s* A, const uint32_t* d_slot_row,
                const uint32_t* d_col_map, Sell& S, uint32_t long_cap) {
    S.long_cap = long_cap;
    cudaStream_t st = ctx->stream;
    S.n_rows = A->n_rows;
    S.n_slots = (A->n_rows + 31u) & ~31u;
    S.n_chunks = S.n_slots / 32;
    S.row_len.alloc(S.n_slots);
    if (S.n_slots == 0) {
        S.chunk_off.alloc(1);
        MPKG_CUDA(cudaMemsetAsync(S.chunk_off.p, 0, sizeof(uint64_t), st));
        S.n_entries = 0;
        return;
    }
    k_sell_lengths<<<grid_for(S.n_slots, 256), 256, 0, st>>>(A->row_ptr.p, A->n_rows, d_slot_row,
                                                            S.n_slots, S.row_len.p);
    MPKG_LAUNCH_CHECK();
    DevBuf<uint64_t> sizes(S.n_chunks + 1);
    MPKG_CUDA(cudaMemsetAsync(sizes.p + S.n_chunks, 0, sizeof(uint64_t), st));
    k_sell_chunk_sizes<<<grid_for((uint64_t)S.n_chunks * 32, 256), 256, 0, st>>>(
        S.row_len.p, S.n_chunks, long_cap, sizes.p);
    MPKG_LAUNCH_CHECK();
    S.chunk_off.alloc(S.n_chunks + 1);
    size_t tmp_bytes = 0;
    MPKG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, sizes.p, S.chunk_off.p,
                                            (int)(S.n_chunks + 1), st));
    DevBuf<uint8_t> tmp(tmp_bytes);
    MPKG_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, tmp_bytes, sizes.p, S.chunk_off.p,
                                            (int)(S.n_chunks + 1), st));
    MPKG_CUDA(cudaMemcpyAsync(&S.n_entries, S.chunk_off.p + S.n_chunks, sizeof(uint64_t),
                              cudaMemcpyDeviceToHost, st));
    MPKG_CUDA(cudaStreamSynchronize(st));
    S.cols.alloc(S.n_entries + 4);
    S.vals.alloc(S.n_entries + 2);
    MPKG_CUDA(cudaMemsetAsync(S.cols.p, 0, S.cols.bytes(), st));
    MPKG_CUDA(cudaMemsetAsync(S.vals.p, 0, S.vals.bytes(), st));
    if (d_slot_row) {
        S.slot_row.alloc(S.n_slots);
        MPKG_CUDA(cudaMemcpyAsync(S.slot_row.p, d_slot_row, sizeof(uint32_t) * S.n_slots,
                                  cudaMemcpyDeviceToDevice, st));
    }
    k_sell_fill<<<grid_for(S.n_slots, 256), 256, 0, st>>>(
        A->row_ptr.p, A->col_idx.p, A->values.p, A->n_rows, d_slot_row, S.chunk_off.p,
        S.row_len.p, S.n_slots, long_cap, d_col_map, S.cols.p, S.vals.p);
    MPKG_LAUNCH_CHECK();
    ctx->launches += 3;
}

Sell& csr_sell(mpkg_csr_s* A) {
    if (!A->sell) {
        auto S = std::make_unique<Sell>();
        build_sell(A->ctx, A, nullptr, nullptr, *S, 0xffffffffu);
        A->sell = std::move(S);
    }
    return *A->sell;
}

void launch_spmv_sell(mpkg_ctx_s* ctx, const Sell& S, bool shifted, const double* src,
                      double* dst, const double* src2, double a, double b2) {
    if (S.n_slots == 0) return;
    const auto ev = timing_begin(ctx);
    launch_spmv_sell_raw(ctx, S, shifted, src, dst, src2, a, b2);
    timing_end(ctx, ev);
}

void launch_spmv_sell_raw(mpkg_ctx_s* ctx, const Sell& S, bool shifted, const double* src,
                          double* dst, const double* src2, double a, double b2, bool pdl) {
    if (S.n_slots == 0) return;
    const unsigned grid = grid_for(S.n_slots, 256, (unsigned)ctx->sm_count * 8u);
    const uint32_t* slot_row = S.slot_row.n ? S.slot_row.p : nullptr;
    launch_maybe_pdl(pdl, shifted ? k_spmv_sell<1> : k_spmv_sell<0>, grid, 256, ctx->stream,
                     (const uint32_t*)S.cols.p, (const double*)S.vals.p, (const uint64_t*)S.chunk_off.p,
                     (const uint32_t*)S.row_len.p, slot_row, (uint32_t)S.n_slots, (uint32_t)S.n_rows,
                     src, dst, src2, a, b2);
    MPKG_LAUNCH_CHECK();
    ctx->launches += 1;
}

}  // namespace mpkg_detail
