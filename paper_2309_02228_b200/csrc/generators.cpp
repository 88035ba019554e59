// Host-side matrix generators: the harness inputs of BASELINE.json's configs.
//
// The reference's own generators (proj/include/mpk/generators.hpp:35-146) build COO triplets and
// call from_coo (csr.hpp:72-110), which costs 16 B per triplet plus a stable-sort buffer (~30 GB
// transient at config C5).  These emit CSR directly in ascending column order and produce
// exactly the matrices from_coo would (checked against oracle/_ref in tests/test_generators.py).
// The 27-point stencil, the scramble and R-MAT have no reference implementation; they follow
// BASELINE.json configs C2-C4 as restated in SURVEY §7 step 1 and §8(d).
#include <omp.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <numeric>
#include <parallel/algorithm>
#include <random>
#include <unordered_set>
#include <utility>
#include <vector>

#include "common.h"
#include "host_csr.h"

using namespace mpkg_detail;

namespace {

using Csr = mpkg_host_csr_s;

// Two-pass CSR construction for stencil-like generators: count(r) returns the row length,
// fill(r, cols, vals) writes the row in ascending column order.
template <class Count, class Fill>
Csr* build_rows(uint32_t n, Count&& count, Fill&& fill) {
    auto* A = new Csr();
    A->n_rows = n;
    A->n_cols = n;
    A->row_ptr.reset(static_cast<uint64_t>(n) + 1);
#pragma omp parallel for schedule(static)
    for (int64_t r = 0; r < static_cast<int64_t>(n); ++r) A->row_ptr[r + 1] = count(static_cast<uint32_t>(r));
    A->row_ptr[0] = 0;
    uint64_t acc = 0;
    for (uint64_t r = 1; r <= n; ++r) {
        acc += A->row_ptr[r];
        if (acc >= (uint64_t{1} << 31)) {
            delete A;
            fail(MPKG_EINVAL, "generator: nnz exceeds the 32-bit index range (csr.hpp:74-76)");
        }
        A->row_ptr[r] = static_cast<uint32_t>(acc);
    }
    A->col_idx.reset(acc);
    A->values.reset(acc);
#pragma omp parallel for schedule(static)
    for (int64_t r = 0; r < static_cast<int64_t>(n); ++r) {
        const uint64_t o = A->row_ptr[r];
        fill(static_cast<uint32_t>(r), A->col_idx.p + o, A->values.p + o);
    }
    return A;
}

// generators.hpp:35-45
Csr* poisson1d(uint32_t n) {
    require(n > 0, "poisson1d: empty grid");
    return build_rows(
        n, [=](uint32_t i) { return 1u + (i > 0) + (i + 1 < n); },
        [=](uint32_t i, uint32_t* c, double* v) {
            int k = 0;
            if (i > 0) c[k] = i - 1, v[k++] = -1.0;
            c[k] = i, v[k++] = 2.0;
            if (i + 1 < n) c[k] = i + 1, v[k++] = -1.0;
        });
}

// generators.hpp:49-65, row i = y*nx + x
Csr* poisson2d(uint32_t nx, uint32_t ny) {
    require(nx > 0 && ny > 0, "poisson2d: empty grid");
    const uint64_t n64 = static_cast<uint64_t>(nx) * ny;
    require(n64 < (uint64_t{1} << 32), "poisson2d: grid too large");
    const uint32_t n = static_cast<uint32_t>(n64);
    return build_rows(
        n,
        [=](uint32_t i) {
            const uint32_t x = i % nx, y = i / nx;
            return 1u + (y > 0) + (x > 0) + (x + 1 < nx) + (y + 1 < ny);
        },
        [=](uint32_t i, uint32_t* c, double* v) {
            const uint32_t x = i % nx, y = i / nx;
            int k = 0;
            if (y > 0) c[k] = i - nx, v[k++] = -1.0;
            if (x > 0) c[k] = i - 1, v[k++] = -1.0;
            c[k] = i, v[k++] = 4.0;
            if (x + 1 < nx) c[k] = i + 1, v[k++] = -1.0;
            if (y + 1 < ny) c[k] = i + nx, v[k++] = -1.0;
        });
}

// generators.hpp:68-89, row i = (z*ny + y)*nx + x (configs C1 and C5)
Csr* poisson3d(uint32_t nx, uint32_t ny, uint32_t nz) {
    require(nx > 0 && ny > 0 && nz > 0, "poisson3d: empty grid");
    const uint64_t n64 = static_cast<uint64_t>(nx) * ny * nz;
    require(n64 < (uint64_t{1} << 32), "poisson3d: grid too large");
    const uint32_t n = static_cast<uint32_t>(n64);
    const uint32_t pl = nx * ny;
    return build_rows(
        n,
        [=](uint32_t i) {
            const uint32_t x = i % nx, y = (i / nx) % ny, z = i / pl;
            return 1u + (z > 0) + (y > 0) + (x > 0) + (x + 1 < nx) + (y + 1 < ny) + (z + 1 < nz);
        },
        [=](uint32_t i, uint32_t* c, double* v) {
            const uint32_t x = i % nx, y = (i / nx) % ny, z = i / pl;
            int k = 0;
            if (z > 0) c[k] = i - pl, v[k++] = -1.0;
            if (y > 0) c[k] = i - nx, v[k++] = -1.0;
            if (x > 0) c[k] = i - 1, v[k++] = -1.0;
            c[k] = i, v[k++] = 6.0;
            if (x + 1 < nx) c[k] = i + 1, v[k++] = -1.0;
            if (y + 1 < ny) c[k] = i + nx, v[k++] = -1.0;
            if (z + 1 < nz) c[k] = i + pl, v[k++] = -1.0;
        });
}

// 27-point stencil pattern: neighbours (dz,dy,dx) in lexicographic order == ascending column.
Csr* stencil27_pattern(uint32_t nx, uint32_t ny, uint32_t nz, double diag, double off) {
    require(nx > 0 && ny > 0 && nz > 0, "stencil27: empty grid");
    const uint64_t n64 = static_cast<uint64_t>(nx) * ny * nz;
    require(n64 < (uint64_t{1} << 32), "stencil27: grid too large");
    const uint32_t n = static_cast<uint32_t>(n64);
    const uint32_t pl = nx * ny;
    auto span = [](uint32_t a, uint32_t na) { return 1u + (a > 0) + (a + 1 < na); };
    return build_rows(
        n,
        [=](uint32_t i) {
            const uint32_t x = i % nx, y = (i / nx) % ny, z = i / pl;
            return span(x, nx) * span(y, ny) * span(z, nz);
        },
        [=](uint32_t i, uint32_t* c, double* v) {
            const int64_t x = i % nx, y = (i / nx) % ny, z = i / pl;
            int k = 0;
            for (int dz = -1; dz <= 1; ++dz) {
                if (z + dz < 0 || z + dz >= nz) continue;
                for (int dy = -1; dy <= 1; ++dy) {
                    if (y + dy < 0 || y + dy >= ny) continue;
                    for (int dx = -1; dx <= 1; ++dx) {
                        if (x + dx < 0 || x + dx >= nx) continue;
                        const int64_t j = i + static_cast<int64_t>(dz) * pl +
                                          static_cast<int64_t>(dy) * nx + dx;
                        c[k] = static_cast<uint32_t>(j);
                        v[k++] = (dz == 0 && dy == 0 && dx == 0) ? diag : off;
                    }
                }
            }
        });
}

// Config C2 before the scramble: off-diagonals -1 * U[0.9,1.1] drawn from mt19937_64(seed) in
// storage order (rows ascending, columns ascending; the diagonal draws nothing), then
// symmetrised as B = (A + A^T)/2 with b_ij = (a_ij + a_ji) * 0.5 (so b_ij == b_ji exactly).
Csr* stencil27_random_sym(uint32_t nx, uint32_t ny, uint32_t nz, uint64_t seed) {
    Csr* A = stencil27_pattern(nx, ny, nz, 26.0, -1.0);
    const uint32_t n = A->n_rows;
    std::mt19937_64 rng(seed);
    std::uniform_real_distribution<double> u(0.9, 1.1);
    HostArray<double> a(A->nnz());
    for (uint32_t r = 0; r < n; ++r)
        for (uint32_t k = A->row_ptr[r]; k < A->row_ptr[r + 1]; ++k)
            a[k] = A->col_idx[k] == r ? A->values[k] : -1.0 * u(rng);
#pragma omp parallel for schedule(static)
    for (int64_t r = 0; r < static_cast<int64_t>(n); ++r) {
        for (uint32_t k = A->row_ptr[r]; k < A->row_ptr[r + 1]; ++k) {
            const uint32_t c = A->col_idx[k];
            const uint32_t* b = A->col_idx.p + A->row_ptr[c];
            const uint32_t* e = A->col_idx.p + A->row_ptr[c + 1];
            const uint32_t* it = std::lower_bound(b, e, static_cast<uint32_t>(r));
            const double aji = a[static_cast<uint64_t>(it - A->col_idx.p)];
            A->values[k] = (a[k] + aji) * 0.5;
        }
    }
    return A;
}

// generators.hpp:96-122 — reproduced draw for draw (same engine and distributions).
Csr* random_csr(uint32_t n, uint32_t nnz_per_row, uint64_t seed) {
    require(n > 0, "random_csr: empty matrix");
    require(nnz_per_row > 0 && nnz_per_row <= n, "random_csr: bad nnz_per_row");
    std::mt19937_64 rng(seed);
    std::uniform_int_distribution<uint32_t> col_dist(0, n - 1);
    std::uniform_real_distribution<double> val_dist(-1.0, 1.0);
    auto* A = new Csr();
    A->n_rows = n;
    A->n_cols = n;
    const uint64_t nnz = static_cast<uint64_t>(n) * nnz_per_row;
    A->row_ptr.reset(static_cast<uint64_t>(n) + 1);
    A->col_idx.reset(nnz);
    A->values.reset(nnz);
    std::unordered_set<uint32_t> used;
    std::vector<std::pair<uint32_t, double>> row;
    uint64_t o = 0;
    A->row_ptr[0] = 0;
    for (uint32_t r = 0; r < n; ++r) {
        used.clear();
        used.insert(r);
        row.clear();
        double abs_sum = 0.0;
        for (uint32_t k = 1; k < nnz_per_row; ++k) {
            uint32_t c = col_dist(rng);
            while (used.count(c)) c = col_dist(rng);
            used.insert(c);
            const double v = val_dist(rng);
            abs_sum += std::abs(v);
            row.push_back({c, v});
        }
        row.push_back({r, abs_sum + 1.0});
        std::sort(row.begin(), row.end(),
                  [](const auto& x, const auto& y) { return x.first < y.first; });
        for (const auto& [c, v] : row) {
            A->col_idx[o] = c;
            A->values[o] = v;
            ++o;
        }
        A->row_ptr[r + 1] = static_cast<uint32_t>(o);
    }
    return A;
}

// generators.hpp:126-146 — (A + A^T)/2 with the diagonal re-boosted.  from_coo sums duplicate
// (r,c) entries in input order (A's entry first, then A^T's), starting from 0.0; the diagonal is
// 1 + the off-diagonal |.| sum accumulated over A's row then A^T's row.
Csr* random_spd(uint32_t n, uint32_t nnz_per_row, uint64_t seed) {
    Csr* A = random_csr(n, nnz_per_row, seed);
    // transpose (csr.hpp:207-227)
    std::vector<uint32_t> trp(static_cast<size_t>(n) + 1, 0), tci(A->nnz());
    std::vector<double> tv(A->nnz());
    for (uint64_t k = 0; k < A->nnz(); ++k) trp[A->col_idx[k] + 1]++;
    for (uint32_t r = 0; r < n; ++r) trp[r + 1] += trp[r];
    std::vector<uint32_t> cur(trp.begin(), trp.end() - 1);
    for (uint32_t r = 0; r < n; ++r)
        for (uint32_t k = A->row_ptr[r]; k < A->row_ptr[r + 1]; ++k) {
            const uint32_t pos = cur[A->col_idx[k]]++;
            tci[pos] = r;
            tv[pos] = A->values[k];
        }
    auto* B = new Csr();
    B->n_rows = n;
    B->n_cols = n;
    B->row_ptr.reset(static_cast<uint64_t>(n) + 1);
    std::vector<uint32_t> bc;
    std::vector<double> bv;
    bc.reserve(2 * A->nnz() + n);
    bv.reserve(2 * A->nnz() + n);
    B->row_ptr[0] = 0;
    for (uint32_t r = 0; r < n; ++r) {
        uint32_t a = A->row_ptr[r], ae = A->row_ptr[r + 1], b = trp[r], be = trp[r + 1];
        double off_sum = 0.0;
        for (uint32_t k = a; k < ae; ++k)
            if (A->col_idx[k] != r) off_sum += std::abs(0.5 * A->values[k]);
        for (uint32_t k = b; k < be; ++k)
            if (tci[k] != r) off_sum += std::abs(0.5 * tv[k]);
        bool diag_done = false;
        auto emit_diag = [&] {
            bc.push_back(r);
            bv.push_back(off_sum + 1.0);
            diag_done = true;
        };
        while (a < ae || b < be) {
            if (a < ae && A->col_idx[a] == r) { ++a; continue; }
            if (b < be && tci[b] == r) { ++b; continue; }
            uint32_t c;
            double s = 0.0;
            if (b >= be || (a < ae && A->col_idx[a] < tci[b])) {
                c = A->col_idx[a];
                s += 0.5 * A->values[a++];
            } else if (a >= ae || tci[b] < A->col_idx[a]) {
                c = tci[b];
                s += 0.5 * tv[b++];
            } else {
                c = A->col_idx[a];
                s += 0.5 * A->values[a++];
                s += 0.5 * tv[b++];
            }
            if (!diag_done && c > r) emit_diag();
            bc.push_back(c);
            bv.push_back(s);
        }
        if (!diag_done) emit_diag();
        B->row_ptr[r + 1] = static_cast<uint32_t>(bc.size());
    }
    B->col_idx.reset(bc.size());
    B->values.reset(bv.size());
    std::memcpy(B->col_idx.p, bc.data(), sizeof(uint32_t) * bc.size());
    std::memcpy(B->values.p, bv.data(), sizeof(double) * bv.size());
    delete A;
    return B;
}

uint64_t splitmix64(uint64_t x) {
    x += 0x9e3779b97f4a7c15ull;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
    return x ^ (x >> 31);
}

// Config C3: R-MAT(scale, edge_factor) with (a,b,c,d) = (.57,.19,.19,.05).  Edges are drawn in
// blocks of 2^16, block k from mt19937_64(splitmix64(seed ^ k)), one U[0,1) draw per level, so
// the matrix does not depend on the host thread count.  The pattern is symmetrised, self loops
// and duplicates removed; off-diagonal values are -U[0.1,1.0] from a counter hash of
// (seed, min(i,j), max(i,j)) (so a_ij == a_ji); the diagonal is 1 + the row's |off| sum
// (ascending column order).
Csr* rmat(uint32_t scale, uint32_t edge_factor, uint64_t seed) {
    require(scale >= 1 && scale <= 30, "rmat: scale out of range");
    require(edge_factor >= 1, "rmat: edge_factor must be >= 1");
    const uint32_t n = 1u << scale;
    const uint64_t m = static_cast<uint64_t>(edge_factor) << scale;
    const double A = 0.57, B = 0.19, C = 0.19;
    const uint64_t blk = uint64_t{1} << 16;
    const uint64_t nblk = (m + blk - 1) / blk;
    std::vector<uint64_t> keys(m);
#pragma omp parallel for schedule(dynamic, 4)
    for (int64_t bi = 0; bi < static_cast<int64_t>(nblk); ++bi) {
        std::mt19937_64 rng(splitmix64(seed ^ static_cast<uint64_t>(bi)));
        std::uniform_real_distribution<double> u(0.0, 1.0);
        const uint64_t e0 = bi * blk, e1 = std::min(m, e0 + blk);
        for (uint64_t e = e0; e < e1; ++e) {
            uint32_t r = 0, c = 0;
            for (uint32_t bit = scale; bit-- > 0;) {
                const double p = u(rng);
                if (p < A) {
                } else if (p < A + B) {
                    c |= 1u << bit;
                } else if (p < A + B + C) {
                    r |= 1u << bit;
                } else {
                    r |= 1u << bit;
                    c |= 1u << bit;
                }
            }
            const uint32_t lo = std::min(r, c), hi = std::max(r, c);
            keys[e] = lo == hi ? ~uint64_t{0} : (static_cast<uint64_t>(lo) << 32) | hi;
        }
    }
    __gnu_parallel::sort(keys.begin(), keys.end());
    keys.erase(std::unique(keys.begin(), keys.end()), keys.end());
    if (!keys.empty() && keys.back() == ~uint64_t{0}) keys.pop_back();
    const uint64_t ne = keys.size();
    std::vector<double> ev(ne);
#pragma omp parallel for schedule(static)
    for (int64_t e = 0; e < static_cast<int64_t>(ne); ++e) {
        const uint64_t h = splitmix64(splitmix64(seed * 0x9e3779b97f4a7c15ull + 1) ^ keys[e]);
        const double u01 = static_cast<double>(h >> 11) * 0x1.0p-53;
        ev[e] = -(0.1 + 0.9 * u01);
    }
    // row lengths: 1 (diag) + upper + lower
    std::vector<uint32_t> len(n, 1);
    for (uint64_t e = 0; e < ne; ++e) {
        len[keys[e] >> 32]++;
        len[keys[e] & 0xffffffffu]++;
    }
    auto* M = new Csr();
    M->n_rows = n;
    M->n_cols = n;
    M->row_ptr.reset(static_cast<uint64_t>(n) + 1);
    M->row_ptr[0] = 0;
    uint64_t acc = 0;
    for (uint32_t r = 0; r < n; ++r) {
        acc += len[r];
        M->row_ptr[r + 1] = static_cast<uint32_t>(acc);
    }
    M->col_idx.reset(acc);
    M->values.reset(acc);
    // lower entries (cols < r) come from edges (u, r) with u < r: edges are sorted by (u, v), so
    // a serial pass appends them in ascending u for every row.
    std::vector<uint32_t> cur(n);
    for (uint32_t r = 0; r < n; ++r) cur[r] = M->row_ptr[r];
    for (uint64_t e = 0; e < ne; ++e) {
        const uint32_t u = static_cast<uint32_t>(keys[e] >> 32), v = static_cast<uint32_t>(keys[e]);
        const uint32_t pos = cur[v]++;
        M->col_idx[pos] = u;
        M->values[pos] = ev[e];
    }
    // diagonal slot, then the upper entries (edges (r, v), v > r, contiguous and ascending).
#pragma omp parallel for schedule(dynamic, 1024)
    for (int64_t r = 0; r < static_cast<int64_t>(n); ++r) {
        uint32_t pos = cur[r];
        const uint32_t diag_pos = pos++;
        const uint64_t e0 = static_cast<uint64_t>(
            std::lower_bound(keys.begin(), keys.end(), static_cast<uint64_t>(r) << 32) - keys.begin());
        for (uint64_t e = e0; e < ne && (keys[e] >> 32) == static_cast<uint64_t>(r); ++e) {
            M->col_idx[pos] = static_cast<uint32_t>(keys[e]);
            M->values[pos] = ev[e];
            ++pos;
        }
        double s = 0.0;
        for (uint32_t k = M->row_ptr[r]; k < M->row_ptr[r + 1]; ++k)
            if (k != diag_pos) s += std::abs(M->values[k]);
        M->col_idx[diag_pos] = static_cast<uint32_t>(r);
        M->values[diag_pos] = 1.0 + s;
    }
    return M;
}

}  // namespace

extern "C" {

int mpkg_gen(int kind, uint32_t a, uint32_t b, uint32_t c, uint64_t seed, mpkg_host_csr_t* out) {
    return guarded([&] {
        require(out != nullptr, "mpkg_gen: null output");
        Csr* m = nullptr;
        switch (kind) {
            case 1: m = poisson1d(a); break;
            case 2: m = poisson2d(a, b); break;
            case 3: m = poisson3d(a, b, c); break;
            case 4: m = random_csr(a, b, seed); break;
            case 5: m = random_spd(a, b, seed); break;
            case 6: m = stencil27_pattern(a, b, c, 26.0, -1.0); break;
            case 7: m = stencil27_random_sym(a, b, c, seed); break;
            case 8: m = rmat(a, b, seed); break;
            default: fail(MPKG_EINVAL, "mpkg_gen: unknown generator kind");
        }
        *out = m;
    });
}

// Seeded symmetric scramble, B[perm[i], perm[j]] = A[i, j] (csr.hpp:159-188 semantics) with a
// Fisher-Yates shuffle: for i = n-1..1, j = floor(rng() * (i+1) / 2^64), swap(s[i], s[j]);
// perm = s.
int mpkg_host_csr_scramble(mpkg_host_csr_t A, uint64_t seed, uint32_t* perm_out,
                           mpkg_host_csr_t* out) {
    return guarded([&] {
        require(A && out, "scramble: null argument");
        require(A->n_rows == A->n_cols, "scramble: matrix must be square");
        const uint32_t n = A->n_rows;
        std::vector<uint32_t> s(n);
        std::iota(s.begin(), s.end(), 0u);
        std::mt19937_64 rng(seed);
        for (uint64_t i = n; i-- > 1;) {
            const uint64_t j =
                static_cast<uint64_t>((static_cast<unsigned __int128>(rng()) * (i + 1)) >> 64);
            std::swap(s[i], s[j]);
        }
        auto* B = new Csr();
        B->n_rows = n;
        B->n_cols = n;
        B->row_ptr.reset(static_cast<uint64_t>(n) + 1);
        std::vector<uint32_t> inv(n);
        for (uint32_t i = 0; i < n; ++i) inv[s[i]] = i;
        B->row_ptr[0] = 0;
        for (uint32_t i = 0; i < n; ++i) {
            const uint32_t old = inv[i];
            B->row_ptr[i + 1] = B->row_ptr[i] + (A->row_ptr[old + 1] - A->row_ptr[old]);
        }
        B->col_idx.reset(A->nnz());
        B->values.reset(A->nnz());
#pragma omp parallel
        {
            std::vector<std::pair<uint32_t, double>> tmp;
#pragma omp for schedule(dynamic, 4096)
            for (int64_t i = 0; i < static_cast<int64_t>(n); ++i) {
                const uint32_t old = inv[i];
                tmp.clear();
                for (uint32_t k = A->row_ptr[old]; k < A->row_ptr[old + 1]; ++k)
                    tmp.push_back({s[A->col_idx[k]], A->values[k]});
                std::sort(tmp.begin(), tmp.end(),
                          [](const auto& x, const auto& y) { return x.first < y.first; });
                uint64_t o = B->row_ptr[i];
                for (const auto& [cc, vv] : tmp) {
                    B->col_idx[o] = cc;
                    B->values[o] = vv;
                    ++o;
                }
            }
        }
        if (perm_out) std::memcpy(perm_out, s.data(), sizeof(uint32_t) * n);
        *out = B;
    });
}

int mpkg_host_csr_info(mpkg_host_csr_t h, uint32_t* n_rows, uint32_t* n_cols, uint64_t* nnz) {
    return guarded([&] {
        require(h != nullptr, "host_csr_info: null handle");
        if (n_rows) *n_rows = h->n_rows;
        if (n_cols) *n_cols = h->n_cols;
        if (nnz) *nnz = h->nnz();
    });
}

int mpkg_host_csr_arrays(mpkg_host_csr_t h, uint32_t** row_ptr, uint32_t** col_idx,
                         double** values) {
    return guarded([&] {
        require(h != nullptr, "host_csr_arrays: null handle");
        if (row_ptr) *row_ptr = h->row_ptr.p;
        if (col_idx) *col_idx = h->col_idx.p;
        if (values) *values = h->values.p;
    });
}

int mpkg_host_csr_destroy(mpkg_host_csr_t h) {
    delete h;
    return MPKG_OK;
}

// acceptance.cpp:84-90 random_vector
int mpkg_random_vector(uint64_t n, uint64_t seed, double* out) {
    return guarded([&] {
        require(out != nullptr || n == 0, "random_vector: null output");
        std::mt19937_64 rng(seed);
        std::uniform_real_distribution<double> u(-1.0, 1.0);
        for (uint64_t i = 0; i < n; ++i) out[i] = u(rng);
    });
}

}  // extern "C"
