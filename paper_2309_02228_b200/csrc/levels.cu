// GPU level construction, bit-exact with the reference's build_levels (levels.hpp:65-147).
//
// The reference: (i) symmetrises the pattern (union of A and A^T, self loops dropped,
// levels.hpp:73-92); (ii) visits candidates in (union-degree, index) order and roots a FIFO BFS
// at the first unvisited one (levels.hpp:101-129); (iii) counting-sorts rows by (level, original
// index) (levels.hpp:131-145).  Because every component is rooted at its (degree, index)
// minimum and BFS distances do not depend on the traversal order, the same structure comes out
// of a data-parallel pipeline:
//   1. union degree per row without materialising A^T: for each stored (r,c), c != r, count it
//      for r, and count it for c too when (c,r) is not stored (binary search in row c);
//      asymmetric entries also feed an "extra" adjacency c -> r so the BFS sees the union;
//   2. connected components by lock-free union-find (hook larger root under smaller);
//   3. per component the (degree<<32 | index) minimum via 64-bit atomicMin -> the root;
//   4. multi-source level-synchronous BFS from all roots at once (a vertex's level is its
//      distance to its own component's root, exactly the reference's level);
//   5. stable radix sort of (level, index) -> inv_perm, perm by scatter; level_ptr from the BFS
//      frontier sizes.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include <algorithm>

#include "device.h"

namespace mpkg_detail {

namespace {

constexpr uint32_t kUnvisited = 0xffffffffu;

__device__ __forceinline__ bool row_contains(const uint32_t* __restrict__ rp,
                                             const uint32_t* __restrict__ ci, uint32_t row,
                                             uint32_t col) {
    uint32_t lo = rp[row], hi = rp[row + 1];
    while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        const uint32_t v = ci[mid];
        if (v == col) return true;
        if (v < col)
            lo = mid + 1;
        else
            hi = mid;
    }
    return false;
}

// Warp per row.  deg[] and ext_cnt[] must be zeroed.
__global__ void k_union_degree(const uint32_t* __restrict__ rp, const uint32_t* __restrict__ ci,
                               uint32_t n, uint32_t* __restrict__ deg,
                               uint32_t* __restrict__ ext_cnt) {
    const uint32_t lane = threadIdx.x & 31;
    for (uint64_t r = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5; r < n;
         r += ((uint64_t)gridDim.x * blockDim.x) >> 5) {
        uint32_t own = 0;
        for (uint32_t k = rp[r] + lane; k < rp[r + 1]; k += 32) {
            const uint32_t c = ci[k];
            if (c == r) continue;
            ++own;
            if (!row_contains(rp, ci, c, (uint32_t)r)) {
                atomicAdd(deg + c, 1u);
                atomicAdd(ext_cnt + c, 1u);
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) own += __shfl_xor_sync(0xffffffffu, own, o);
        if (lane == 0 && own) atomicAdd(deg + r, own);
    }
}

__global__ void k_ext_fill(const uint32_t* __restrict__ rp, const uint32_t* __restrict__ ci,
                           uint32_t n, const uint32_t* __restrict__ ext_ptr,
                           uint32_t* __restrict__ ext_cur, uint32_t* __restrict__ ext_idx) {
    const uint32_t lane = threadIdx.x & 31;
    for (uint64_t r = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5; r < n;
         r += ((uint64_t)gridDim.x * blockDim.x) >> 5) {
        for (uint32_t k = rp[r] + lane; k < rp[r + 1]; k += 32) {
            const uint32_t c = ci[k];
            if (c == r) continue;
            if (!row_contains(rp, ci, c, (uint32_t)r))
                ext_idx[ext_ptr[c] + atomicAdd(ext_cur + c, 1u)] = (uint32_t)r;
        }
    }
}

__global__ void k_iota(uint32_t* __restrict__ a, uint32_t n) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x)
        a[i] = (uint32_t)i;
}

__device__ __forceinline__ uint32_t uf_find(uint32_t* parent, uint32_t x) {
    uint32_t p = parent[x];
    while (p != x) {
        const uint32_t gp = parent[p];
        if (gp != p) parent[x] = gp;  // path halving (benign race)
        x = p;
        p = gp;
    }
    return x;
}

// Union-find over every stored entry (the union pattern is symmetric for connectivity).
__global__ void k_uf_union(const uint32_t* __restrict__ rp, const uint32_t* __restrict__ ci,
                           uint32_t n, uint32_t* parent) {
    const uint32_t lane = threadIdx.x & 31;
    for (uint64_t r = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5; r < n;
         r += ((uint64_t)gridDim.x * blockDim.x) >> 5) {
        for (uint32_t k = rp[r] + lane; k < rp[r + 1]; k += 32) {
            uint32_t a = (uint32_t)r, b = ci[k];
            if (a == b) continue;
            while (true) {
                a = uf_find(parent, a);
                b = uf_find(parent, b);
                if (a == b) break;
                if (a < b) {
                    const uint32_t t = a;
                    a = b;
                    b = t;
                }
                // hook root a (larger) under b
                if (atomicCAS(parent + a, a, b) == a) break;
            }
        }
    }
}

__global__ void k_uf_flatten_key(uint32_t* parent, const uint32_t* __restrict__ deg, uint32_t n,
                                 unsigned long long* __restrict__ comp_key) {
    for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < n;
         v += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t root = uf_find(parent, (uint32_t)v);
        parent[v] = root;
        const unsigned long long key = ((unsigned long long)deg[v] << 32) | v;
        atomicMin(comp_key + root, key);
    }
}

// Roots get level 0 and enter frontier 0.
__global__ void k_init_roots(const uint32_t* __restrict__ comp, uint32_t n,
                             const unsigned long long* __restrict__ comp_key,
                             uint32_t* __restrict__ level, uint32_t* __restrict__ queue,
                             uint32_t* __restrict__ counts) {
    for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < n;
         v += (uint64_t)gridDim.x * blockDim.x) {
        const bool root = (uint32_t)(comp_key[comp[v]] & 0xffffffffull) == (uint32_t)v;
        level[v] = root ? 0u : kUnvisited;
        if (root) queue[atomicAdd(counts, 1u)] = (uint32_t)v;
    }
}

// Expands frontier L (queue[start_L .. start_L+count_L)) into frontier L+1, warp per vertex.
// counts[L] = frontier size, starts are the running sums of counts.
__global__ void k_bfs_level(const uint32_t* __restrict__ rp, const uint32_t* __restrict__ ci,
                            const uint32_t* __restrict__ ext_ptr,
                            const uint32_t* __restrict__ ext_idx, uint32_t* __restrict__ level,
                            uint32_t* __restrict__ queue, uint32_t* __restrict__ counts,
                            uint32_t* __restrict__ starts, uint32_t L) {
    const uint32_t cnt = counts[L];
    if (cnt == 0) return;
    const uint32_t start = starts[L];
    const uint32_t next_start = start + cnt;
    if (blockIdx.x == 0 && threadIdx.x == 0) starts[L + 1] = next_start;
    const uint32_t lane = threadIdx.x & 31;
    for (uint64_t i = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5; i < cnt;
         i += ((uint64_t)gridDim.x * blockDim.x) >> 5) {
        const uint32_t u = queue[start + i];
        for (uint32_t k = rp[u] + lane; k < rp[u + 1]; k += 32) {
            const uint32_t v = ci[k];
            if (level[v] == kUnvisited && atomicCAS(level + v, kUnvisited, L + 1) == kUnvisited)
                queue[next_start + atomicAdd(counts + L + 1, 1u)] = v;
        }
        for (uint32_t k = ext_ptr[u] + lane; k < ext_ptr[u + 1]; k += 32) {
            const uint32_t v = ext_idx[k];
            if (level[v] == kUnvisited && atomicCAS(level + v, kUnvisited, L + 1) == kUnvisited)
                queue[next_start + atomicAdd(counts + L + 1, 1u)] = v;
        }
    }
}

__global__ void k_scatter_perm(const uint32_t* __restrict__ inv_perm, uint32_t n,
                               uint32_t* __restrict__ perm) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x)
        perm[inv_perm[i]] = (uint32_t)i;
}

__global__ void k_validate(const uint32_t* __restrict__ rp, const uint32_t* __restrict__ ci,
                           uint32_t n, const uint32_t* __restrict__ levels,
                           const uint32_t* __restrict__ inv_perm, uint32_t* __restrict__ bad) {
    const uint32_t lane = threadIdx.x & 31;
    for (uint64_t r = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5; r < n;
         r += ((uint64_t)gridDim.x * blockDim.x) >> 5) {
        const uint32_t lr = levels[inv_perm[r]];
        for (uint32_t k = rp[r] + lane; k < rp[r + 1]; k += 32) {
            const uint32_t lc = levels[inv_perm[ci[k]]];
            const uint32_t d = lr > lc ? lr - lc : lc - lr;
            if (d > 1) atomicOr(bad, 1u);
        }
    }
}

}  // namespace

void gpu_build_levels(mpkg_ctx_s* ctx, const mpkg_csr_s* A, mpkg_levels_s* L) {
    const uint32_t n = A->n_rows;
    cudaStream_t st = ctx->stream;
    L->n_rows = n;
    L->levels.alloc(n);
    L->perm.alloc(n);
    L->inv_perm.alloc(n);
    if (n == 0) {
        L->n_levels = 0;
        L->level_ptr.assign(1, 0);
        L->d_level_ptr.alloc(1);
        MPKG_CUDA(cudaMemsetAsync(L->d_level_ptr.p, 0, sizeof(uint32_t), st));
        return;
    }
    const unsigned wgrid = grid_for((uint64_t)n * 32, 256, (unsigned)ctx->sm_count * 16u);
    const unsigned tgrid = grid_for(n, 256, (unsigned)ctx->sm_count * 16u);

    // 1. union degree + extra (asymmetric) adjacency
    DevBuf<uint32_t> deg(n), ext_cnt(n + 1), ext_ptr(n + 1);
    MPKG_CUDA(cudaMemsetAsync(deg.p, 0, deg.bytes(), st));
    MPKG_CUDA(cudaMemsetAsync(ext_cnt.p, 0, ext_cnt.bytes(), st));
    k_union_degree<<<wgrid, 256, 0, st>>>(A->row_ptr.p, A->col_idx.p, n, deg.p, ext_cnt.p);
    MPKG_LAUNCH_CHECK();
    size_t tmp_bytes = 0;
    MPKG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, ext_cnt.p, ext_ptr.p, (int)(n + 1), st));
    DevBuf<uint8_t> tmp(tmp_bytes);
    MPKG_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, tmp_bytes, ext_cnt.p, ext_ptr.p, (int)(n + 1), st));
    uint32_t n_ext = 0;
    MPKG_CUDA(cudaMemcpyAsync(&n_ext, ext_ptr.p + n, sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
    MPKG_CUDA(cudaStreamSynchronize(st));
    DevBuf<uint32_t> ext_idx(n_ext + 1);
    if (n_ext) {
        MPKG_CUDA(cudaMemsetAsync(ext_cnt.p, 0, ext_cnt.bytes(), st));
        k_ext_fill<<<wgrid, 256, 0, st>>>(A->row_ptr.p, A->col_idx.p, n, ext_ptr.p, ext_cnt.p,
                                          ext_idx.p);
        MPKG_LAUNCH_CHECK();
    }

    // 2. connected components
    DevBuf<uint32_t> parent(n);
    k_iota<<<tgrid, 256, 0, st>>>(parent.p, n);
    k_uf_union<<<wgrid, 256, 0, st>>>(A->row_ptr.p, A->col_idx.p, n, parent.p);
    MPKG_LAUNCH_CHECK();
    // 3. component roots: argmin (degree, index)
    DevBuf<unsigned long long> comp_key(n);
    MPKG_CUDA(cudaMemsetAsync(comp_key.p, 0xff, comp_key.bytes(), st));
    k_uf_flatten_key<<<tgrid, 256, 0, st>>>(parent.p, deg.p, n, comp_key.p);
    MPKG_LAUNCH_CHECK();

    // 4. multi-source BFS; queue holds each vertex exactly once, frontier by frontier.
    DevBuf<uint32_t> queue(n), counts(n + 2), starts(n + 2);
    MPKG_CUDA(cudaMemsetAsync(counts.p, 0, counts.bytes(), st));
    MPKG_CUDA(cudaMemsetAsync(starts.p, 0, starts.bytes(), st));
    uint32_t* level = L->levels.p;
    k_init_roots<<<tgrid, 256, 0, st>>>(parent.p, n, comp_key.p, level, queue.p, counts.p);
    MPKG_LAUNCH_CHECK();
    ctx->launches += 6;
    const unsigned bfs_grid = (unsigned)ctx->sm_count * 8u;
    uint32_t n_levels = 0;
    std::vector<uint32_t> hcounts;
    for (uint32_t base = 0; base < n; base += 32) {
        const uint32_t end = std::min<uint32_t>(n, base + 32);
        for (uint32_t l = base; l < end; ++l)
            k_bfs_level<<<bfs_grid, 256, 0, st>>>(A->row_ptr.p, A->col_idx.p, ext_ptr.p,
                                                  ext_idx.p, level, queue.p, counts.p, starts.p, l);
        MPKG_LAUNCH_CHECK();
        ctx->launches += end - base;
        uint32_t last = 0;
        MPKG_CUDA(cudaMemcpyAsync(&last, counts.p + end, sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
        MPKG_CUDA(cudaStreamSynchronize(st));
        if (last == 0) break;
    }
    hcounts.resize(n + 1);
    MPKG_CUDA(cudaMemcpyAsync(hcounts.data(), counts.p, sizeof(uint32_t) * (n + 1),
                              cudaMemcpyDeviceToHost, st));
    MPKG_CUDA(cudaStreamSynchronize(st));
    while (n_levels < n && hcounts[n_levels] != 0) ++n_levels;
    L->n_levels = n_levels;
    L->level_ptr.assign(n_levels + 1, 0);
    uint64_t acc = 0;
    for (uint32_t l = 0; l < n_levels; ++l) {
        acc += hcounts[l];
        L->level_ptr[l + 1] = (uint32_t)acc;
    }
    if (acc != n) fail(MPKG_EINTERNAL, "build_levels: BFS did not reach every row");
    L->d_level_ptr.alloc(n_levels + 1);
    MPKG_CUDA(cudaMemcpyAsync(L->d_level_ptr.p, L->level_ptr.data(), sizeof(uint32_t) * (n_levels + 1),
                              cudaMemcpyHostToDevice, st));

    // 5. stable sort by level (values: original index) -> inv_perm; perm by scatter.
    DevBuf<uint32_t> idx(n), keys_out(n);
    k_iota<<<tgrid, 256, 0, st>>>(idx.p, n);
    int end_bit = 1;
    while ((1ull << end_bit) < (uint64_t)n_levels) ++end_bit;
    size_t sort_bytes = 0;
    MPKG_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, sort_bytes, level, keys_out.p, idx.p,
                                              L->inv_perm.p, (int)n, 0, end_bit, st));
    DevBuf<uint8_t> sort_tmp(sort_bytes);
    MPKG_CUDA(cub::DeviceRadixSort::SortPairs(sort_tmp.p, sort_bytes, level, keys_out.p, idx.p,
                                              L->inv_perm.p, (int)n, 0, end_bit, st));
    k_scatter_perm<<<tgrid, 256, 0, st>>>(L->inv_perm.p, n, L->perm.p);
    MPKG_LAUNCH_CHECK();
    ctx->launches += 3;
    MPKG_CUDA(cudaStreamSynchronize(st));
}

bool gpu_validate_levels(mpkg_ctx_s* ctx, const mpkg_csr_s* A, const mpkg_levels_s* L) {
    if (A->n_rows != L->n_rows || A->n_rows != A->n_cols) return false;
    const uint32_t n = A->n_rows;
    if (n == 0) return true;
    cudaStream_t st = ctx->stream;
    DevBuf<uint32_t> bad(1);
    MPKG_CUDA(cudaMemsetAsync(bad.p, 0, sizeof(uint32_t), st));
    k_validate<<<grid_for((uint64_t)n * 32, 256, (unsigned)ctx->sm_count * 16u), 256, 0, st>>>(
        A->row_ptr.p, A->col_idx.p, n, L->levels.p, L->inv_perm.p, bad.p);
    MPKG_LAUNCH_CHECK();
    ctx->launches += 1;
    uint32_t h = 0;
    MPKG_CUDA(cudaMemcpyAsync(&h, bad.p, sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
    MPKG_CUDA(cudaStreamSynchronize(st));
    return h == 0;
}

}  // namespace mpkg_detail
