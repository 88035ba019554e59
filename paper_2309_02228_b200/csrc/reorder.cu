// GPU-private locality order inside BFS levels (SURVEY §7 hard part 7).
//
// The reference's perm sorts each level by ORIGINAL row index (levels.hpp:131-145).  After a
// random scramble (config C2) that order is random inside a level, so the x-gathers of 32
// consecutive rows touch 32 unrelated cache lines.  The executor therefore runs the rows of
// A_perm in a second order sigma that never leaves a level: level 0 keeps the A_perm order;
// every row of level l >= 1 is keyed by the smallest sigma position of its neighbours in level
// l-1, and level l is stably sorted by that key (a Cuthill-McKee sweep restricted to the
// level structure).  sigma is invisible at the API: outputs are written back at their A_perm
// positions and each row keeps its stored entry order, so results stay bit-identical.
#include <cub/device/device_radix_sort.cuh>

#include <algorithm>

#include "device.h"

namespace mpkg_detail {

namespace {

// key[v] = min pos[c] over the row's columns c < lvl_begin (i.e. its neighbours in level l-1;
// rows are sorted by column and levels are contiguous, so these are the leading entries).
__global__ void k_cm_keys(const uint32_t* __restrict__ rp, const uint32_t* __restrict__ ci,
                          uint32_t lvl_begin, uint32_t lvl_end, const uint32_t* __restrict__ pos,
                          uint32_t* __restrict__ keys, uint32_t* __restrict__ vals) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < lvl_end - lvl_begin;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t v = lvl_begin + (uint32_t)i;
        uint32_t key = 0xffffffffu;
        for (uint32_t k = rp[v]; k < rp[v + 1]; ++k) {
            const uint32_t c = ci[k];
            if (c >= lvl_begin) break;
            key = min(key, pos[c]);
        }
        keys[i] = key;
        vals[i] = v;
    }
}

// SELL-C-sigma key: longer rows first (radix sort ascending on ~len), ties by A_perm index.
__global__ void k_len_keys(const uint32_t* __restrict__ rp, uint32_t lvl_begin, uint32_t lvl_end,
                           uint32_t* __restrict__ keys, uint32_t* __restrict__ vals) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < lvl_end - lvl_begin;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t v = lvl_begin + (uint32_t)i;
        keys[i] = 0xffffffffu - (rp[v + 1] - rp[v]);
        vals[i] = v;
    }
}

__global__ void k_cm_place(const uint32_t* __restrict__ sorted_rows, uint32_t lvl_begin,
                           uint32_t count, uint32_t* __restrict__ slot_row,
                           uint32_t* __restrict__ pos) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < count;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t r = sorted_rows[i];
        slot_row[lvl_begin + i] = r;
        pos[r] = lvl_begin + (uint32_t)i;
    }
}

__global__ void k_identity_order(uint32_t n, uint32_t n_slots, uint32_t* slot_row, uint32_t* pos) {
    for (uint64_t s = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; s < n_slots;
         s += (uint64_t)gridDim.x * blockDim.x) {
        slot_row[s] = s < n ? (uint32_t)s : 0xffffffffu;
        if (s < n) pos[s] = (uint32_t)s;
    }
}

__global__ void k_max_len(const uint32_t* __restrict__ rp, uint32_t n, uint32_t* __restrict__ out) {
    uint32_t m = 0;
    for (uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r < n;
         r += (uint64_t)gridDim.x * blockDim.x)
        m = max(m, rp[r + 1] - rp[r]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0) atomicMax(out, m);
}

// Sum over consecutive rows of |first column(r+1) - first column(r)| (first column = the row's
// smallest neighbour, normally in the previous level): small when consecutive rows of A_perm
// gather from nearby x, ~level width / 3 when the order inside levels is random.
__global__ void k_first_col_jump(const uint32_t* __restrict__ rp, const uint32_t* __restrict__ ci,
                                 uint32_t n, unsigned long long* __restrict__ out) {
    unsigned long long acc = 0;
    for (uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r + 1 < n;
         r += (uint64_t)gridDim.x * blockDim.x) {
        if (rp[r] == rp[r + 1] || rp[r + 1] == rp[r + 2]) continue;
        const uint32_t a = ci[rp[r]], b = ci[rp[r + 1]];
        acc += a > b ? a - b : b - a;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0) atomicAdd(out, acc);
}

}  // namespace

double gpu_mean_first_col_jump(mpkg_ctx_s* ctx, const mpkg_csr_s* A) {
    if (A->n_rows < 2) return 0.0;
    DevBuf<unsigned long long> d(1);
    MPKG_CUDA(cudaMemsetAsync(d.p, 0, 8, ctx->stream));
    k_first_col_jump<<<grid_for(A->n_rows, 256, (unsigned)ctx->sm_count * 4u), 256, 0, ctx->stream>>>(
        A->row_ptr.p, A->col_idx.p, A->n_rows, d.p);
    MPKG_LAUNCH_CHECK();
    ctx->launches += 1;
    unsigned long long h = 0;
    MPKG_CUDA(cudaMemcpyAsync(&h, d.p, 8, cudaMemcpyDeviceToHost, ctx->stream));
    MPKG_CUDA(cudaStreamSynchronize(ctx->stream));
    return (double)h / (double)(A->n_rows - 1);
}

uint32_t gpu_max_row_len(mpkg_ctx_s* ctx, const mpkg_csr_s* A) {
    if (A->n_rows == 0) return 0;
    DevBuf<uint32_t> d(1);
    MPKG_CUDA(cudaMemsetAsync(d.p, 0, 4, ctx->stream));
    k_max_len<<<grid_for(A->n_rows, 256, (unsigned)ctx->sm_count * 4u), 256, 0, ctx->stream>>>(A->row_ptr.p, A->n_rows, d.p);
    MPKG_LAUNCH_CHECK();
    ctx->launches += 1;
    uint32_t h = 0;
    MPKG_CUDA(cudaMemcpyAsync(&h, d.p, 4, cudaMemcpyDeviceToHost, ctx->stream));
    MPKG_CUDA(cudaStreamSynchronize(ctx->stream));
    return h;
}

// slot_row[s] = A_perm row held by slot s (0xffffffff for padding slots >= n), pos = inverse.
// mode 1: Cuthill-McKee inside levels; mode 2: longest rows first inside levels (SELL-C-sigma,
// for power-law row lengths).
void gpu_level_cm_order(mpkg_ctx_s* ctx, const mpkg_csr_s* A, const std::vector<uint32_t>& level_ptr,
                        uint32_t n_slots, DevBuf<uint32_t>& slot_row, DevBuf<uint32_t>& pos,
                        int mode) {
    const uint32_t n = A->n_rows;
    cudaStream_t st = ctx->stream;
    slot_row.alloc(std::max<uint32_t>(n_slots, 1));
    pos.alloc(std::max<uint32_t>(n, 1));
    k_identity_order<<<grid_for(n_slots, 256), 256, 0, st>>>(n, n_slots, slot_row.p, pos.p);
    MPKG_LAUNCH_CHECK();
    ctx->launches += 1;
    const uint32_t nl = level_ptr.empty() ? 0 : (uint32_t)level_ptr.size() - 1;
    uint32_t max_level = 0;
    for (uint32_t l = 0; l < nl; ++l) max_level = std::max(max_level, level_ptr[l + 1] - level_ptr[l]);
    if (max_level == 0 || (mode == 1 && nl < 2)) return;
    DevBuf<uint32_t> keys(max_level), keys_out(max_level), vals(max_level), vals_out(max_level);
    size_t tmp_bytes = 0;
    MPKG_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, keys.p, keys_out.p, vals.p,
                                              vals_out.p, (int)max_level, 0, 32, st));
    DevBuf<uint8_t> tmp(tmp_bytes);
    int pos_bits = 1;
    while ((1ull << pos_bits) <= (uint64_t)n) ++pos_bits;
    for (uint32_t l = mode == 1 ? 1 : 0; l < nl; ++l) {
        const uint32_t b = level_ptr[l], e = level_ptr[l + 1], cnt = e - b;
        if (cnt == 0) continue;
        if (mode == 1)
            k_cm_keys<<<grid_for(cnt, 256), 256, 0, st>>>(A->row_ptr.p, A->col_idx.p, b, e, pos.p,
                                                         keys.p, vals.p);
        else
            k_len_keys<<<grid_for(cnt, 256), 256, 0, st>>>(A->row_ptr.p, b, e, keys.p, vals.p);
        MPKG_LAUNCH_CHECK();
        size_t tb = tmp_bytes;
        // CM: key 0xffffffff (no neighbour in l-1: possible for a nonsymmetric pattern) sorts last
        MPKG_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, tb, keys.p, keys_out.p, vals.p,
                                                  vals_out.p, (int)cnt, 0,
                                                  mode == 1 ? std::min(32, pos_bits + 1) : 32, st));
        k_cm_place<<<grid_for(cnt, 256), 256, 0, st>>>(vals_out.p, b, cnt, slot_row.p, pos.p);
        MPKG_LAUNCH_CHECK();
        ctx->launches += 3;
    }
}

}  // namespace mpkg_detail
