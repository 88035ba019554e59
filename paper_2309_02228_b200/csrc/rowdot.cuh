// The per-row bitwise SpMV formula over SELL-32 storage, shared by every power kernel.
//
// Reference formula (csr.hpp:115-123, mpk.hpp:68-73): acc = 0.0; acc += values[k] * x[col[k]]
// for the row's entries in stored (ascending column) order.  One thread owns one row's
// accumulation and uses __dmul_rn + __dadd_rn so that nvcc can never contract to DFMA: the
// result is bit-identical to the reference's x86-64 build (which has no FMA: the reference
// CMakeLists sets no -march).
//
// SELL-32 chunk layout (chunk of 32 slots, maximum row length L, entries start at `off`, a
// multiple of 32; Lp = 2*floor(L/2)).  Columns and values share ONE interleave, so a flat entry
// index addresses both arrays:
//   k < Lp:  off + (k/2)*64 + lane*2 + k%2     (lane reads 8 B of columns / 16 B of values)
//   k == Lp: off + Lp*32 + lane                (odd L: the last entry)
// Every warp-wide load is one contiguous 256 B (cols) / 512 B (vals) segment; padding exists only
// where rows of one chunk differ in length (column 0, value 0) and is never accumulated (0*Inf
// would be NaN).
#pragma once

#include <cstdint>

namespace mpkg_detail {

__device__ __forceinline__ uint32_t sell_pos(uint32_t k, uint32_t Lp, uint32_t lane) {
    return k < Lp ? (k >> 1) * 64u + lane * 2u + (k & 1u) : Lp * 32u + lane;
}

// Streaming loads of matrix data: read-only for the kernel's lifetime, no L1 allocation, with
// an L2 eviction-priority policy.
__device__ __forceinline__ uint2 ld_mat_u2(const uint2* p, uint64_t pol) {
    uint2 r;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.u32 {%0,%1}, [%2], %3;"
                 : "=r"(r.x), "=r"(r.y)
                 : "l"(p), "l"(pol));
    return r;
}
__device__ __forceinline__ uint32_t ld_mat_u32(const uint32_t* p, uint64_t pol) {
    uint32_t r;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.u32 %0, [%1], %2;"
                 : "=r"(r)
                 : "l"(p), "l"(pol));
    return r;
}
__device__ __forceinline__ double2 ld_mat_d2(const double2* p, uint64_t pol) {
    double2 r;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.f64 {%0,%1}, [%2], %3;"
                 : "=d"(r.x), "=d"(r.y)
                 : "l"(p), "l"(pol));
    return r;
}
__device__ __forceinline__ double ld_mat_d(const double* p, uint64_t pol) {
    double r;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;"
                 : "=d"(r)
                 : "l"(p), "l"(pol));
    return r;
}

__device__ __forceinline__ uint64_t l2_policy_first() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ uint64_t l2_policy_last() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}

// Vector gathers.  READONLY: the source slice is not written during the launch (x, or any slice
// in the one-launch-per-power baseline) -> non-coherent texture path.  Otherwise the slice is
// produced by other CTAs of the same launch and is read only after an acquire on its tile flag:
// plain (coherent, L1-cacheable) loads.
template <bool READONLY>
__device__ __forceinline__ double ld_vec(const double* p) {
    if constexpr (READONLY) {
        return __ldg(p);
    } else {
        return *p;
    }
}

// Row dot product straight from global memory, with memory-level parallelism: the row is
// processed in groups of G entries (G even); all G columns, G values and G x-gathers of a group
// are issued before the group's strictly sequential accumulation.  Loads are predicated on
// k < L (the chunk's stored width: in bounds for every lane); accumulation on k < len, in stored
// order.
template <bool READONLY, int G>
__device__ __forceinline__ double sell_row_dot(const uint32_t* __restrict__ cols,
                                               const double* __restrict__ vals, uint64_t off,
                                               uint32_t L, uint32_t lane, uint32_t len,
                                               const double* src, uint64_t pol) {
    static_assert(G % 2 == 0, "group must be even");
    double acc = 0.0;
    const uint32_t Lp = L & ~1u;
    for (uint32_t k0 = 0; k0 < len; k0 += G) {
        uint32_t c[G];
        double v[G], x[G];
#pragma unroll
        for (int j = 0; j < G; j += 2) {
            const uint32_t k = k0 + j;
            if (k + 1 < Lp) {
                const uint64_t e = off + (k >> 1) * 64u + lane * 2u;
                const uint2 cc = ld_mat_u2(reinterpret_cast<const uint2*>(cols + e), pol);
                const double2 vv = ld_mat_d2(reinterpret_cast<const double2*>(vals + e), pol);
                c[j] = cc.x, c[j + 1] = cc.y, v[j] = vv.x, v[j + 1] = vv.y;
            } else {
#pragma unroll
                for (int i = 0; i < 2; ++i) {
                    const uint32_t kk = k + i;
                    const uint64_t e = off + sell_pos(kk, Lp, lane);
                    c[j + i] = kk < L ? ld_mat_u32(cols + e, pol) : 0u;
                    v[j + i] = kk < L ? ld_mat_d(vals + e, pol) : 0.0;
                }
            }
        }
#pragma unroll
        for (int j = 0; j < G; ++j) x[j] = (k0 + j < len) ? ld_vec<READONLY>(src + c[j]) : 0.0;
#pragma unroll
        for (int j = 0; j < G; ++j)
            if (k0 + j < len) acc = __dadd_rn(acc, __dmul_rn(v[j], x[j]));
    }
    return acc;
}

// Register-light, software-pipelined row dot straight from global memory: the next pair's
// column indices and values are loaded while the current pair's x-gathers are in flight, so
// each pair costs one dependent round trip instead of two.  Same additions, same order.
template <bool READONLY>
__device__ __forceinline__ double sell_row_dot_pipe(const uint32_t* __restrict__ cols,
                                                    const double* __restrict__ vals, uint64_t off,
                                                    uint32_t L, uint32_t lane, uint32_t len,
                                                    const double* src, uint64_t pol) {
    double acc = 0.0;
    const uint32_t Lp = L & ~1u;
    const uint32_t npairs = (len < Lp ? len : Lp) >> 1;  // full pairs inside this row
    const uint2* cp = reinterpret_cast<const uint2*>(cols + off) + lane;
    const double2* vp = reinterpret_cast<const double2*>(vals + off) + lane;
    uint32_t k = 0;
    if (npairs) {
        uint2 c = ld_mat_u2(cp, pol);
        double2 v = ld_mat_d2(vp, pol);
        for (uint32_t j = 0; j < npairs; ++j) {
            const double x0 = ld_vec<READONLY>(src + c.x);
            const double x1 = ld_vec<READONLY>(src + c.y);
            const double2 vc = v;
            if (j + 1 < npairs) {  // prefetch the next pair while the gathers are in flight
                c = ld_mat_u2(cp + (j + 1) * 32, pol);
                v = ld_mat_d2(vp + (j + 1) * 32, pol);
            }
            acc = __dadd_rn(acc, __dmul_rn(vc.x, x0));
            acc = __dadd_rn(acc, __dmul_rn(vc.y, x1));
        }
        k = npairs * 2;
    }
    for (; k < len; ++k) {
        const uint64_t e = off + sell_pos(k, Lp, lane);
        acc = __dadd_rn(acc, __dmul_rn(ld_mat_d(vals + e, pol), ld_vec<READONLY>(src + ld_mat_u32(cols + e, pol))));
    }
    return acc;
}

// Same as sell_row_dot with the tile's COLUMN indices staged in shared memory (TMA, identical
// layout, offsets relative to the tile start `rel`) and the values streamed from global memory:
// gather addresses are available at shared-memory latency, so each group's G gathers issue at
// once and overlap the value loads.
template <bool READONLY, int G>
__device__ __forceinline__ double sell_row_dot_staged(const uint32_t* cols_s,
                                                      const double* __restrict__ vals,
                                                      uint32_t rel, uint64_t off, uint32_t L,
                                                      uint32_t lane, uint32_t len,
                                                      const double* src, uint64_t pol) {
    static_assert(G % 2 == 0, "group must be even");
    double acc = 0.0;
    const uint32_t Lp = L & ~1u;
    for (uint32_t k0 = 0; k0 < len; k0 += G) {
        double v[G], x[G];
#pragma unroll
        for (int j = 0; j < G; j += 2) {
            const uint32_t k = k0 + j;
            if (k + 1 < Lp) {
                const uint32_t e = (k >> 1) * 64u + lane * 2u;
                const uint2 cc = *reinterpret_cast<const uint2*>(cols_s + rel + e);
                const double2 vv = ld_mat_d2(reinterpret_cast<const double2*>(vals + off + e), pol);
                v[j] = vv.x, v[j + 1] = vv.y;
                x[j] = k < len ? ld_vec<READONLY>(src + cc.x) : 0.0;
                x[j + 1] = k + 1 < len ? ld_vec<READONLY>(src + cc.y) : 0.0;
            } else {
#pragma unroll
                for (int i = 0; i < 2; ++i) {
                    const uint32_t kk = k + i;
                    const uint32_t e = sell_pos(kk, Lp, lane);
                    v[j + i] = kk < len ? ld_mat_d(vals + off + e, pol) : 0.0;
                    x[j + i] = kk < len ? ld_vec<READONLY>(src + cols_s[rel + e]) : 0.0;
                }
            }
        }
#pragma unroll
        for (int j = 0; j < G; ++j)
            if (k0 + j < len) acc = __dadd_rn(acc, __dmul_rn(v[j], x[j]));
    }
    return acc;
}

// Sequential, stored-order sum of a row's products already computed in shared memory in the
// SELL layout (two-phase tile kernel): same additions in the same order as sell_row_dot.
__device__ __forceinline__ double sell_row_sum_smem(const double* prod, uint32_t rel, uint32_t L,
                                                    uint32_t lane, uint32_t len) {
    double acc = 0.0;
    const uint32_t Lp = L & ~1u;
    uint32_t k = 0;
    for (; k + 1 < len && k + 1 < Lp; k += 2) {
        const double2 p = *reinterpret_cast<const double2*>(prod + rel + (k >> 1) * 64u + lane * 2u);
        acc = __dadd_rn(acc, p.x);
        acc = __dadd_rn(acc, p.y);
    }
    for (; k < len; ++k) acc = __dadd_rn(acc, prod[rel + sell_pos(k, Lp, lane)]);
    return acc;
}

// Epilogues (mpk.hpp:135-153): real shift dst = acc - a*src[r]; second member of a conjugate
// pair dst = acc - a*src[r] + b2*src2[r] (left to right, no contraction).
__device__ __forceinline__ double shift_epilogue(double acc, double a, double b2, double own,
                                                 double own2) {
    double r = __dsub_rn(acc, __dmul_rn(a, own));
    if (b2 != 0.0) r = __dadd_rn(r, __dmul_rn(b2, own2));
    return r;
}

}  // namespace mpkg_detail
