// GPU symmetric permutation, bit-exact with the reference's permute (csr.hpp:159-188):
// B[perm[i], perm[j]] = A[i, j], each row's (new column, value) pairs sorted by column.
// Rows are relabelled and gathered in parallel, then every row is sorted by key: short rows by
// one warp in registers (bitonic network over <= 64 entries), longer rows by
// cub::DeviceSegmentedSort.  Columns are unique within a row, so a sort by column alone equals
// the reference's std::sort on (column, value) pairs.
#include <cub/device/device_scan.cuh>
#include <cub/device/device_segmented_sort.cuh>

#include "device.h"

namespace mpkg_detail {

namespace {

__global__ void k_perm_check(const uint32_t* __restrict__ perm, uint32_t n,
                             uint32_t* __restrict__ seen, uint32_t* __restrict__ bad) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t p = perm[i];
        if (p >= n || atomicExch(seen + p, 1u) != 0u) atomicOr(bad, 1u);
    }
}

__global__ void k_new_lengths(const uint32_t* __restrict__ rp, const uint32_t* __restrict__ perm,
                              uint32_t n, uint32_t* __restrict__ len_new) {
    for (uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r < n;
         r += (uint64_t)gridDim.x * blockDim.x)
        len_new[perm[r]] = rp[r + 1] - rp[r];
}

// Warp per old row: relabel columns, gather into the new row position.  Rows of length <= 64
// are sorted in registers here (bitonic over 64 keys, 2 per lane); longer rows are flagged for
// the segmented sort.
__global__ void k_permute_rows(const uint32_t* __restrict__ rp, const uint32_t* __restrict__ ci,
                               const double* __restrict__ v, const uint32_t* __restrict__ perm,
                               uint32_t n, const uint32_t* __restrict__ rp_new,
                               uint32_t* __restrict__ ci_new, double* __restrict__ v_new,
                               uint32_t* __restrict__ long_rows) {
    const uint32_t lane = threadIdx.x & 31;
    for (uint64_t r = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5; r < n;
         r += ((uint64_t)gridDim.x * blockDim.x) >> 5) {
        const uint32_t b = rp[r], len = rp[r + 1] - b;
        const uint32_t o = rp_new[perm[r]];
        if (len <= 64) {
            uint32_t k0 = 0xffffffffu, k1 = 0xffffffffu;
            double v0 = 0.0, v1 = 0.0;
            if (lane < len) k0 = perm[ci[b + lane]], v0 = v[b + lane];
            if (lane + 32 < len) k1 = perm[ci[b + lane + 32]], v1 = v[b + lane + 32];
            // element index e = lane (k0) and lane+32 (k1); bitonic sort of 64 elements.
            for (uint32_t size = 2; size <= 64; size <<= 1) {
                for (uint32_t stride = size >> 1; stride > 0; stride >>= 1) {
                    if (stride == 32) {
                        // partner of e=lane is e=lane+32 (same lane, other register)
                        const bool asc = ((lane & size) == 0);  // size==64 -> ascending
                        if ((k0 > k1) == asc) {
                            uint32_t tk = k0; k0 = k1; k1 = tk;
                            double tv = v0; v0 = v1; v1 = tv;
                        }
                    } else {
                        const uint32_t pk0 = __shfl_xor_sync(0xffffffffu, k0, stride);
                        const double pv0 = __shfl_xor_sync(0xffffffffu, v0, stride);
                        const uint32_t pk1 = __shfl_xor_sync(0xffffffffu, k1, stride);
                        const double pv1 = __shfl_xor_sync(0xffffffffu, v1, stride);
                        const bool lower = (lane & stride) == 0;
                        const bool asc0 = ((lane & size) == 0);
                        const bool asc1 = (((lane + 32) & size) == 0);
                        // keep min if (lower && asc) || (!lower && !asc)
                        const bool keep_min0 = lower == asc0;
                        const bool keep_min1 = lower == asc1;
                        if (keep_min0 ? (pk0 < k0) : (pk0 > k0)) k0 = pk0, v0 = pv0;
                        if (keep_min1 ? (pk1 < k1) : (pk1 > k1)) k1 = pk1, v1 = pv1;
                    }
                }
            }
            if (lane < len) ci_new[o + lane] = k0, v_new[o + lane] = v0;
            if (lane + 32 < len) ci_new[o + lane + 32] = k1, v_new[o + lane + 32] = v1;
            if (lane == 0) long_rows[perm[r]] = 0;
        } else {
            for (uint32_t k = lane; k < len; k += 32) {
                ci_new[o + k] = perm[ci[b + k]];
                v_new[o + k] = v[b + k];
            }
            if (lane == 0) long_rows[perm[r]] = 1;
        }
    }
}

__global__ void k_long_offsets(const uint32_t* __restrict__ rp_new,
                               const uint32_t* __restrict__ long_rows,
                               const uint32_t* __restrict__ long_pos, uint32_t n,
                               uint32_t* __restrict__ beg, uint32_t* __restrict__ end) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x)
        if (long_rows[i]) {
            beg[long_pos[i]] = rp_new[i];
            end[long_pos[i]] = rp_new[i + 1];
        }
}

__global__ void k_permute_vector(const double* __restrict__ in, const uint32_t* __restrict__ perm,
                                 uint32_t n, double* __restrict__ out, bool inverse) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        if (inverse)
            out[i] = in[perm[i]];
        else
            out[perm[i]] = in[i];
    }
}

__global__ void k_gather_u32(const uint32_t* __restrict__ src, const uint32_t* __restrict__ idx,
                             uint32_t m, uint32_t* __restrict__ out) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m;
         i += (uint64_t)gridDim.x * blockDim.x)
        out[i] = src[idx[i]];
}

}  // namespace

void gpu_check_permutation(mpkg_ctx_s* ctx, const uint32_t* d_perm, uint32_t n) {
    if (n == 0) return;
    cudaStream_t st = ctx->stream;
    DevBuf<uint32_t> seen(n), bad(1);
    MPKG_CUDA(cudaMemsetAsync(seen.p, 0, seen.bytes(), st));
    MPKG_CUDA(cudaMemsetAsync(bad.p, 0, sizeof(uint32_t), st));
    k_perm_check<<<grid_for(n, 256), 256, 0, st>>>(d_perm, n, seen.p, bad.p);
    MPKG_LAUNCH_CHECK();
    ctx->launches += 1;
    uint32_t h = 0;
    MPKG_CUDA(cudaMemcpyAsync(&h, bad.p, sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
    MPKG_CUDA(cudaStreamSynchronize(st));
    if (h) fail(MPKG_EINVAL, "permute: not a permutation");
}

void gpu_permute(mpkg_ctx_s* ctx, const mpkg_csr_s* A, const uint32_t* d_perm, mpkg_csr_s* B) {
    const uint32_t n = A->n_rows;
    cudaStream_t st = ctx->stream;
    B->ctx = ctx;
    B->device = ctx->device;
    B->n_rows = n;
    B->n_cols = n;
    B->nnz = A->nnz;
    B->row_ptr.alloc(n + 1);
    B->col_idx.alloc((uint64_t)A->nnz + 1);
    B->values.alloc((uint64_t)A->nnz + 1);
    if (n == 0) {
        MPKG_CUDA(cudaMemsetAsync(B->row_ptr.p, 0, sizeof(uint32_t), st));
        return;
    }
    DevBuf<uint32_t> len_new(n + 1);
    MPKG_CUDA(cudaMemsetAsync(len_new.p + n, 0, sizeof(uint32_t), st));
    k_new_lengths<<<grid_for(n, 256), 256, 0, st>>>(A->row_ptr.p, d_perm, n, len_new.p);
    MPKG_LAUNCH_CHECK();
    size_t tb = 0;
    MPKG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, len_new.p, B->row_ptr.p, (int)(n + 1), st));
    DevBuf<uint8_t> tmp(tb);
    MPKG_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, tb, len_new.p, B->row_ptr.p, (int)(n + 1), st));
    DevBuf<uint32_t> long_rows(n + 1), long_pos(n + 1);
    MPKG_CUDA(cudaMemsetAsync(long_rows.p + n, 0, sizeof(uint32_t), st));
    const unsigned wgrid = grid_for((uint64_t)n * 32, 256, (unsigned)ctx->sm_count * 16u);
    k_permute_rows<<<wgrid, 256, 0, st>>>(A->row_ptr.p, A->col_idx.p, A->values.p, d_perm, n,
                                          B->row_ptr.p, B->col_idx.p, B->values.p, long_rows.p);
    MPKG_LAUNCH_CHECK();
    ctx->launches += 3;
    size_t tb2 = 0;
    MPKG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb2, long_rows.p, long_pos.p, (int)(n + 1), st));
    tmp.ensure(tb2);
    MPKG_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, tb2, long_rows.p, long_pos.p, (int)(n + 1), st));
    uint32_t n_long = 0;
    MPKG_CUDA(cudaMemcpyAsync(&n_long, long_pos.p + n, sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
    MPKG_CUDA(cudaStreamSynchronize(st));
    if (n_long) {
        DevBuf<uint32_t> beg(n_long), end(n_long);
        k_long_offsets<<<grid_for(n, 256), 256, 0, st>>>(B->row_ptr.p, long_rows.p, long_pos.p, n,
                                                         beg.p, end.p);
        MPKG_LAUNCH_CHECK();
        // Sort the long rows in place through a copy of the entries.
        DevBuf<uint32_t> kin(A->nnz);
        DevBuf<double> vin(A->nnz);
        MPKG_CUDA(cudaMemcpyAsync(kin.p, B->col_idx.p, sizeof(uint32_t) * A->nnz,
                                  cudaMemcpyDeviceToDevice, st));
        MPKG_CUDA(cudaMemcpyAsync(vin.p, B->values.p, sizeof(double) * A->nnz,
                                  cudaMemcpyDeviceToDevice, st));
        size_t sb = 0;
        MPKG_CUDA(cub::DeviceSegmentedSort::SortPairs(nullptr, sb, kin.p, B->col_idx.p, vin.p,
                                                      B->values.p, (int)A->nnz, (int)n_long,
                                                      beg.p, end.p, st));
        DevBuf<uint8_t> stmp(sb);
        MPKG_CUDA(cub::DeviceSegmentedSort::SortPairs(stmp.p, sb, kin.p, B->col_idx.p, vin.p,
                                                      B->values.p, (int)A->nnz, (int)n_long,
                                                      beg.p, end.p, st));
        ctx->launches += 2;
        MPKG_CUDA(cudaStreamSynchronize(st));
    }
}

void gpu_permute_vector(mpkg_ctx_s* ctx, uint32_t n, const double* d_in, const uint32_t* d_perm,
                        double* d_out, bool inverse) {
    if (n == 0) return;
    k_permute_vector<<<grid_for(n, 256), 256, 0, ctx->stream>>>(d_in, d_perm, n, d_out, inverse);
    MPKG_LAUNCH_CHECK();
    ctx->launches += 1;
}

namespace {
// Entries of row r0+i with column in [c0, c1).
__global__ void k_block_counts(const uint32_t* __restrict__ rp, const uint32_t* __restrict__ ci,
                               uint32_t r0, uint32_t m, uint32_t c0, uint32_t c1,
                               uint32_t* __restrict__ cnt) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m;
         i += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t c = 0;
        for (uint32_t k = rp[r0 + i]; k < rp[r0 + i + 1]; ++k) c += ci[k] >= c0 && ci[k] < c1;
        cnt[i] = c;
    }
}
__global__ void k_block_fill(const uint32_t* __restrict__ rp, const uint32_t* __restrict__ ci,
                             const double* __restrict__ v, uint32_t r0, uint32_t m, uint32_t c0,
                             uint32_t c1, const uint32_t* __restrict__ brp, uint32_t* __restrict__ bci,
                             double* __restrict__ bv) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m;
         i += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t o = brp[i];
        for (uint32_t k = rp[r0 + i]; k < rp[r0 + i + 1]; ++k)
            if (ci[k] >= c0 && ci[k] < c1) {
                bci[o] = ci[k] - c0;
                bv[o++] = v[k];
            }
    }
}
}  // namespace

// B = A[r0:r1, c0:c1] with column indices shifted by -c0; kept entries stay in stored order (the
// local matrix of a level-range shard, multi.py).
void gpu_csr_block(mpkg_ctx_s* ctx, const mpkg_csr_s* A, uint32_t r0, uint32_t r1, uint32_t c0,
                   uint32_t c1, mpkg_csr_s* B) {
    cudaStream_t st = ctx->stream;
    const uint32_t m = r1 - r0;
    B->ctx = ctx;
    B->device = ctx->device;
    B->n_rows = m;
    B->n_cols = c1 - c0;
    B->row_ptr.alloc(m + 1);
    DevBuf<uint32_t> cnt(m + 1);
    MPKG_CUDA(cudaMemsetAsync(cnt.p + m, 0, sizeof(uint32_t), st));
    if (m)
        k_block_counts<<<grid_for(m, 256), 256, 0, st>>>(A->row_ptr.p, A->col_idx.p, r0, m, c0, c1, cnt.p);
    MPKG_LAUNCH_CHECK();
    size_t tb = 0;
    MPKG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, cnt.p, B->row_ptr.p, (int)(m + 1), st));
    DevBuf<uint8_t> tmp(tb);
    MPKG_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, tb, cnt.p, B->row_ptr.p, (int)(m + 1), st));
    uint32_t nnz = 0;
    MPKG_CUDA(cudaMemcpyAsync(&nnz, B->row_ptr.p + m, sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
    MPKG_CUDA(cudaStreamSynchronize(st));
    B->nnz = nnz;
    B->col_idx.alloc((uint64_t)nnz + 1);
    B->values.alloc((uint64_t)nnz + 1);
    if (m)
        k_block_fill<<<grid_for(m, 256), 256, 0, st>>>(A->row_ptr.p, A->col_idx.p, A->values.p, r0, m, c0,
                                                      c1, B->row_ptr.p, B->col_idx.p, B->values.p);
    MPKG_LAUNCH_CHECK();
    ctx->launches += 3;
}

void gpu_gather_row_ptr(mpkg_ctx_s* ctx, const mpkg_csr_s* A, const uint32_t* d_idx, uint32_t m,
                        uint32_t* h_out) {
    if (m == 0) return;
    DevBuf<uint32_t> out(m);
    k_gather_u32<<<grid_for(m, 256), 256, 0, ctx->stream>>>(A->row_ptr.p, d_idx, m, out.p);
    MPKG_LAUNCH_CHECK();
    ctx->launches += 1;
    MPKG_CUDA(cudaMemcpyAsync(h_out, out.p, sizeof(uint32_t) * m, cudaMemcpyDeviceToHost,
                              ctx->stream));
    MPKG_CUDA(cudaStreamSynchronize(ctx->stream));
}

}  // namespace mpkg_detail
