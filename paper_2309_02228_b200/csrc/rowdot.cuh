// The per-row bitwise SpMV formula over SELL-32 storage, shared by every power kernel.
//
// Reference formula (csr.hpp:115-123, mpk.hpp:68-73): acc = 0.0; acc += values[k] * x[col[k]]
// for the row's entries in stored (ascending column) order.  One thread owns one row and uses
// __dmul_rn + __dadd_rn so that nvcc can never contract to DFMA: the result is bit-identical to
// the reference's x86-64 build (which has no FMA: proj/CMakeLists.txt sets no -march).
//
// SELL-32 chunk layout (chunk of 32 slots, maximum row length L, entries start at `off`, a
// multiple of 32):
//   columns: k < Lq = 4*floor(L/4):  off + (k/4)*128 + lane*4 + k%4        (uint4 per lane)
//            k >= Lq:                off + Lq*32 + (k-Lq)*32 + lane         (u32 per lane)
//   values:  k < Lp = 2*floor(L/2):  off + (k/2)*64 + lane*2 + k%2          (double2 per lane)
//            k == Lp (odd L):        off + Lp*32 + lane                     (double per lane)
// Every warp-wide load is a contiguous 512 B (uint4/double2) or 128/256 B (scalar remainder)
// segment; padding exists only where rows of one chunk differ in length, and padded entries
// are never loaded or accumulated (0*Inf would be NaN).
#pragma once

#include <cstdint>

namespace mpkg_detail {

// Streaming loads of matrix data: read-only for the kernel's lifetime, no L1 allocation.
__device__ __forceinline__ uint4 ld_mat_u4(const uint4* p) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}
__device__ __forceinline__ uint32_t ld_mat_u32(const uint32_t* p) {
    uint32_t r;
    asm volatile("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(r) : "l"(p));
    return r;
}
__device__ __forceinline__ double2 ld_mat_d2(const double2* p) {
    double2 r;
    asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0,%1}, [%2];"
                 : "=d"(r.x), "=d"(r.y)
                 : "l"(p));
    return r;
}
__device__ __forceinline__ double ld_mat_d(const double* p) {
    double r;
    asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(r) : "l"(p));
    return r;
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

template <bool READONLY>
__device__ __forceinline__ double sell_row_dot(const uint32_t* __restrict__ cols,
                                               const double* __restrict__ vals, uint64_t off,
                                               uint32_t L, uint32_t lane, uint32_t len,
                                               const double* src) {
    double acc = 0.0;
    const uint32_t Lq = L & ~3u;
    const uint32_t Lp = L & ~1u;
    const uint4* cq = reinterpret_cast<const uint4*>(cols + off) + lane;
    const double2* vp = reinterpret_cast<const double2*>(vals + off) + lane;
    uint32_t k = 0;
    const uint32_t full_q = (len < Lq ? len : Lq) & ~3u;
    for (; k < full_q; k += 4) {
        const uint4 c = ld_mat_u4(cq + (k >> 2) * 32);
        const double2 v0 = ld_mat_d2(vp + (k >> 1) * 32);
        const double2 v1 = ld_mat_d2(vp + ((k >> 1) + 1) * 32);
        const double x0 = ld_vec<READONLY>(src + c.x);
        const double x1 = ld_vec<READONLY>(src + c.y);
        const double x2 = ld_vec<READONLY>(src + c.z);
        const double x3 = ld_vec<READONLY>(src + c.w);
        acc = __dadd_rn(acc, __dmul_rn(v0.x, x0));
        acc = __dadd_rn(acc, __dmul_rn(v0.y, x1));
        acc = __dadd_rn(acc, __dmul_rn(v1.x, x2));
        acc = __dadd_rn(acc, __dmul_rn(v1.y, x3));
    }
    for (; k < len; ++k) {
        uint32_t c;
        if (k < Lq)
            c = ld_mat_u32(cols + off + (k >> 2) * 128 + lane * 4 + (k & 3));
        else
            c = ld_mat_u32(cols + off + Lq * 32 + (k - Lq) * 32 + lane);
        double v;
        if (k < Lp)
            v = ld_mat_d(vals + off + (k >> 1) * 64 + lane * 2 + (k & 1));
        else
            v = ld_mat_d(vals + off + Lp * 32 + lane);
        acc = __dadd_rn(acc, __dmul_rn(v, ld_vec<READONLY>(src + c)));
    }
    return acc;
}

// Value loads with an L2 eviction-priority hint (evict_last while the tile is re-read later in
// the pass, evict_first on its last use).
__device__ __forceinline__ double2 ld_mat_d2_hint(const double2* p, uint64_t pol) {
    double2 r;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.f64 {%0,%1}, [%2], %3;"
                 : "=d"(r.x), "=d"(r.y)
                 : "l"(p), "l"(pol));
    return r;
}
__device__ __forceinline__ double ld_mat_d_hint(const double* p, uint64_t pol) {
    double r;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;"
                 : "=d"(r)
                 : "l"(p), "l"(pol));
    return r;
}

// Same formula with the tile's COLUMN indices staged in shared memory by TMA (identical SELL
// layout, offsets relative to the tile start) and the values streamed from global memory: the
// gather addresses are available at shared-memory latency, so the x gathers (the long-latency
// chain) issue immediately while the value loads overlap them.
template <bool READONLY>
__device__ __forceinline__ double sell_row_dot_smem(const uint32_t* cols_s, const double* __restrict__ vals,
                                                    uint32_t off_rel, uint64_t off, uint32_t L,
                                                    uint32_t lane, uint32_t len, const double* src,
                                                    uint64_t pol) {
    double acc = 0.0;
    const uint32_t Lq = L & ~3u;
    const uint32_t Lp = L & ~1u;
    const uint4* cq = reinterpret_cast<const uint4*>(cols_s + off_rel) + lane;
    const double2* vp = reinterpret_cast<const double2*>(vals + off) + lane;
    uint32_t k = 0;
    const uint32_t full_q = (len < Lq ? len : Lq) & ~3u;
#pragma unroll 2
    for (; k < full_q; k += 4) {
        const uint4 c = cq[(k >> 2) * 32];
        const double2 v0 = ld_mat_d2_hint(vp + (k >> 1) * 32, pol);
        const double2 v1 = ld_mat_d2_hint(vp + ((k >> 1) + 1) * 32, pol);
        const double x0 = ld_vec<READONLY>(src + c.x);
        const double x1 = ld_vec<READONLY>(src + c.y);
        const double x2 = ld_vec<READONLY>(src + c.z);
        const double x3 = ld_vec<READONLY>(src + c.w);
        acc = __dadd_rn(acc, __dmul_rn(v0.x, x0));
        acc = __dadd_rn(acc, __dmul_rn(v0.y, x1));
        acc = __dadd_rn(acc, __dmul_rn(v1.x, x2));
        acc = __dadd_rn(acc, __dmul_rn(v1.y, x3));
    }
    for (; k < len; ++k) {
        const uint32_t c = k < Lq ? cols_s[off_rel + (k >> 2) * 128 + lane * 4 + (k & 3)]
                                  : cols_s[off_rel + Lq * 32 + (k - Lq) * 32 + lane];
        const double v = k < Lp ? ld_mat_d_hint(vals + off + (k >> 1) * 64 + lane * 2 + (k & 1), pol)
                                : ld_mat_d_hint(vals + off + Lp * 32 + lane, pol);
        acc = __dadd_rn(acc, __dmul_rn(v, ld_vec<READONLY>(src + c)));
    }
    return acc;
}

// Memory-level-parallel variant: the row is processed in groups of G entries (G % 4 == 0).
// All G column indices, G x-gathers and G values of a group are issued before the group's
// strictly sequential accumulation, so one row keeps up to 2G independent loads in flight
// instead of one quad.  Loads are predicated on k < L (the chunk's stored width: in bounds for
// every lane, padding entries hold column 0 / value 0); accumulation on k < len, in stored
// order: bit-identical to sell_row_dot.
template <bool READONLY, bool STAGED, int G>
__device__ __forceinline__ double sell_row_dot_mlp(const uint32_t* cols, const double* __restrict__ vals,
                                                   uint64_t off_c, uint64_t off_v, uint32_t L,
                                                   uint32_t lane, uint32_t len, const double* src,
                                                   uint64_t pol) {
    static_assert(G % 4 == 0, "group must be a multiple of 4");
    double acc = 0.0;
    const uint32_t Lq = L & ~3u;
    const uint32_t Lp = L & ~1u;
    for (uint32_t k0 = 0; k0 < len; k0 += G) {
        uint32_t c[G];
        double v[G], x[G];
#pragma unroll
        for (int j = 0; j < G; j += 4) {
            const uint32_t k = k0 + j;
            if (k + 3 < Lq) {
                const uint4* cq = reinterpret_cast<const uint4*>(cols + off_c) + (k >> 2) * 32 + lane;
                const uint4 q4 = STAGED ? *cq : ld_mat_u4(cq);
                c[j] = q4.x, c[j + 1] = q4.y, c[j + 2] = q4.z, c[j + 3] = q4.w;
            } else {
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const uint32_t kk = k + i;
                    const uint32_t* pc = kk < Lq ? cols + off_c + (kk >> 2) * 128 + lane * 4 + (kk & 3)
                                                 : cols + off_c + Lq * 32 + (kk - Lq) * 32 + lane;
                    c[j + i] = kk < L ? (STAGED ? *pc : ld_mat_u32(pc)) : 0u;
                }
            }
        }
#pragma unroll
        for (int j = 0; j < G; j += 2) {
            const uint32_t k = k0 + j;
            if (k + 1 < Lp) {
                const double2 d = ld_mat_d2_hint(
                    reinterpret_cast<const double2*>(vals + off_v) + (k >> 1) * 32 + lane, pol);
                v[j] = d.x, v[j + 1] = d.y;
            } else {
#pragma unroll
                for (int i = 0; i < 2; ++i) {
                    const uint32_t kk = k + i;
                    const double* pv = kk < Lp ? vals + off_v + (kk >> 1) * 64 + lane * 2 + (kk & 1)
                                               : vals + off_v + Lp * 32 + lane;
                    v[j + i] = kk < L ? ld_mat_d_hint(pv, pol) : 0.0;
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

// Epilogues (mpk.hpp:135-153): real shift dst = acc - a*src[r]; second member of a conjugate
// pair dst = acc - a*src[r] + b2*src2[r] (left to right, no contraction).
__device__ __forceinline__ double shift_epilogue(double acc, double a, double b2, double own,
                                                 double own2) {
    double r = __dsub_rn(acc, __dmul_rn(a, own));
    if (b2 != 0.0) r = __dadd_rn(r, __dmul_rn(b2, own2));
    return r;
}

}  // namespace mpkg_detail
