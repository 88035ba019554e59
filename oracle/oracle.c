/*
 * TEST INFRASTRUCTURE ONLY — CPU oracle restating the reference's level-blocked MPK path.
 * See oracle.h for the contract and the pinning story.  Never linked by the product library.
 *
 * Build: cc -std=c99 -O2 (no -march: x86-64 baseline has no FMA, so `acc += v * x` is a mulsd
 * followed by an addsd, exactly like the reference build, proj/CMakeLists.txt:8-21).
 */
#include "oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ---------------------------------------------------------------------------------------------
 * csr.hpp:207-227 — transpose with sorted rows (walking A in row order writes each transposed
 * row in ascending original-row order).  Pattern only: build_levels never reads the values.
 * ------------------------------------------------------------------------------------------- */
static void transpose_pattern(uint32_t n, const uint32_t* rp, const uint32_t* ci, uint32_t* trp,
                              uint32_t* tci) {
    const uint32_t nnz = rp[n];
    memset(trp, 0, sizeof(uint32_t) * ((size_t)n + 1));
    for (uint32_t k = 0; k < nnz; ++k) trp[ci[k] + 1]++;
    for (uint32_t r = 0; r < n; ++r) trp[r + 1] += trp[r];
    uint32_t* cursor = (uint32_t*)malloc(sizeof(uint32_t) * ((size_t)n + 1));
    memcpy(cursor, trp, sizeof(uint32_t) * n);
    for (uint32_t r = 0; r < n; ++r)
        for (uint32_t k = rp[r]; k < rp[r + 1]; ++k) tci[cursor[ci[k]]++] = r;
    free(cursor);
}

static int cmp_u64(const void* a, const void* b) {
    const uint64_t x = *(const uint64_t*)a, y = *(const uint64_t*)b;
    return x < y ? -1 : (x > y ? 1 : 0);
}

/* levels.hpp:65-147 */
int orc_build_levels(uint32_t n, const uint32_t* rp, const uint32_t* ci, uint32_t* levels,
                     uint32_t* perm, uint32_t* inv_perm, uint32_t* level_ptr,
                     uint32_t* n_levels) {
    const uint32_t nnz = rp[n];
    uint32_t* trp = (uint32_t*)malloc(sizeof(uint32_t) * ((size_t)n + 1));
    uint32_t* tci = (uint32_t*)malloc(sizeof(uint32_t) * ((size_t)nnz + 1));
    transpose_pattern(n, rp, ci, trp, tci);

    /* levels.hpp:73-92 — per row the sorted union of the patterns of A and A^T, self-loops
     * dropped. */
    uint32_t* xadj = (uint32_t*)malloc(sizeof(uint32_t) * ((size_t)n + 1));
    uint32_t* adj = (uint32_t*)malloc(sizeof(uint32_t) * (2 * (size_t)nnz + 1));
    size_t m = 0;
    xadj[0] = 0;
    for (uint32_t r = 0; r < n; ++r) {
        uint32_t a = rp[r], ae = rp[r + 1], b = trp[r], be = trp[r + 1];
        while (a < ae || b < be) {
            uint32_t c;
            if (b >= be || (a < ae && ci[a] <= tci[b])) {
                c = ci[a];
                if (a < ae && b < be && ci[a] == tci[b]) ++b;
                ++a;
            } else {
                c = tci[b];
                ++b;
            }
            if (c != r) adj[m++] = c;
        }
        xadj[r + 1] = (uint32_t)m;
    }
    free(trp);
    free(tci);

    /* levels.hpp:101-107 — candidates in (degree, index) order. */
    uint64_t* order = (uint64_t*)malloc(sizeof(uint64_t) * ((size_t)n + 1));
    for (uint32_t i = 0; i < n; ++i)
        order[i] = ((uint64_t)(xadj[i + 1] - xadj[i]) << 32) | (uint64_t)i;
    qsort(order, n, sizeof(uint64_t), cmp_u64);

    /* levels.hpp:109-129 — the first unvisited candidate roots the next component; FIFO BFS. */
    char* visited = (char*)calloc((size_t)n + 1, 1);
    uint32_t* queue = (uint32_t*)malloc(sizeof(uint32_t) * ((size_t)n + 1));
    uint32_t max_level = 0;
    for (uint32_t i = 0; i < n; ++i) levels[i] = 0;
    for (uint32_t t = 0; t < n; ++t) {
        const uint32_t cand = (uint32_t)(order[t] & 0xffffffffu);
        if (visited[cand]) continue;
        visited[cand] = 1;
        levels[cand] = 0;
        uint32_t head = 0, tail = 0;
        queue[tail++] = cand;
        while (head < tail) {
            const uint32_t u = queue[head++];
            for (uint32_t k = xadj[u]; k < xadj[u + 1]; ++k) {
                const uint32_t v = adj[k];
                if (!visited[v]) {
                    visited[v] = 1;
                    levels[v] = levels[u] + 1;
                    if (levels[v] > max_level) max_level = levels[v];
                    queue[tail++] = v;
                }
            }
        }
    }
    free(order);
    free(visited);
    free(queue);
    free(xadj);
    free(adj);

    /* levels.hpp:131-145 — counting sort by (level, original index). */
    const uint32_t nl = n == 0 ? 0 : max_level + 1;
    memset(level_ptr, 0, sizeof(uint32_t) * ((size_t)nl + 1));
    for (uint32_t r = 0; r < n; ++r) level_ptr[levels[r] + 1]++;
    for (uint32_t l = 0; l < nl; ++l) level_ptr[l + 1] += level_ptr[l];
    uint32_t* cursor = (uint32_t*)malloc(sizeof(uint32_t) * ((size_t)nl + 1));
    memcpy(cursor, level_ptr, sizeof(uint32_t) * nl);
    for (uint32_t r = 0; r < n; ++r) {
        const uint32_t pos = cursor[levels[r]]++;
        perm[r] = pos;
        inv_perm[pos] = r;
    }
    free(cursor);
    *n_levels = nl;
    return ORC_OK;
}

/* csr.hpp:145-155 */
int orc_check_permutation(const uint32_t* perm, uint32_t n) {
    char* seen = (char*)calloc((size_t)n + 1, 1);
    int ok = ORC_OK;
    for (uint32_t i = 0; i < n; ++i) {
        if (perm[i] >= n || seen[perm[i]]) {
            ok = ORC_EINVAL;
            break;
        }
        seen[perm[i]] = 1;
    }
    free(seen);
    return ok;
}

typedef struct {
    uint32_t c;
    double v;
} entry_t;

static int cmp_entry(const void* a, const void* b) {
    const uint32_t x = ((const entry_t*)a)->c, y = ((const entry_t*)b)->c;
    return x < y ? -1 : (x > y ? 1 : 0);
}

/* csr.hpp:159-188 — B[perm[i], perm[j]] = A[i, j]; each row's (new col, value) pairs sorted.
 * Columns are unique within a row, so ordering by column alone equals std::sort on the pairs. */
int orc_permute(uint32_t n, const uint32_t* rp, const uint32_t* ci, const double* vals,
                const uint32_t* perm, uint32_t* orp, uint32_t* oci, double* ov) {
    if (orc_check_permutation(perm, n) != ORC_OK) return ORC_EINVAL;
    memset(orp, 0, sizeof(uint32_t) * ((size_t)n + 1));
    for (uint32_t r = 0; r < n; ++r) orp[perm[r] + 1] = rp[r + 1] - rp[r];
    for (uint32_t r = 0; r < n; ++r) orp[r + 1] += orp[r];
    size_t cap = 64;
    entry_t* scratch = (entry_t*)malloc(sizeof(entry_t) * cap);
    for (uint32_t r = 0; r < n; ++r) {
        const uint32_t len = rp[r + 1] - rp[r];
        if (len > cap) {
            cap = len;
            scratch = (entry_t*)realloc(scratch, sizeof(entry_t) * cap);
        }
        for (uint32_t k = 0; k < len; ++k) {
            scratch[k].c = perm[ci[rp[r] + k]];
            scratch[k].v = vals[rp[r] + k];
        }
        qsort(scratch, len, sizeof(entry_t), cmp_entry);
        uint32_t out = orp[perm[r]];
        for (uint32_t k = 0; k < len; ++k, ++out) {
            oci[out] = scratch[k].c;
            ov[out] = scratch[k].v;
        }
    }
    free(scratch);
    return ORC_OK;
}

/* csr.hpp:191-204 */
void orc_permute_vector(uint32_t n, const double* in, const uint32_t* perm, double* out) {
    for (uint32_t i = 0; i < n; ++i) out[perm[i]] = in[i];
}
void orc_unpermute_vector(uint32_t n, const double* in, const uint32_t* perm, double* out) {
    for (uint32_t i = 0; i < n; ++i) out[i] = in[perm[i]];
}

/* levels.hpp:151-164 */
int orc_validate_levels(uint32_t n, const uint32_t* rp, const uint32_t* ci, const uint32_t* levels,
                        const uint32_t* inv_perm) {
    uint32_t* lvl_new = (uint32_t*)malloc(sizeof(uint32_t) * ((size_t)n + 1));
    for (uint32_t i = 0; i < n; ++i) lvl_new[i] = levels[inv_perm[i]];
    int ok = 1;
    for (uint32_t r = 0; r < n && ok; ++r) {
        const uint32_t lr = lvl_new[r];
        for (uint32_t k = rp[r]; k < rp[r + 1]; ++k) {
            const uint32_t lc = lvl_new[ci[k]];
            const uint32_t d = lr > lc ? lr - lc : lc - lr;
            if (d > 1) {
                ok = 0;
                break;
            }
        }
    }
    free(lvl_new);
    return ok;
}

/* plan.hpp:59-64 */
uint64_t orc_row_range_footprint(const uint32_t* rp, uint32_t row_s, uint32_t row_e, int p_m) {
    const uint64_t nnz = (uint64_t)(rp[row_e] - rp[row_s]);
    const uint64_t rows = (uint64_t)(row_e - row_s);
    return 12 * nnz + 4 * rows + 8 * (uint64_t)(p_m + 1) * rows;
}

/* plan.hpp:70-85 */
uint32_t orc_greedy_group(const uint64_t* fp, uint32_t nl, uint64_t target, uint32_t* bounds) {
    uint32_t nb = 0;
    bounds[nb++] = 0;
    uint64_t acc = 0;
    for (uint32_t l = 0; l < nl; ++l) {
        if (l > bounds[nb - 1] && acc + fp[l] > target) {
            bounds[nb++] = l;
            acc = 0;
        }
        acc += fp[l];
    }
    if (nl > 0) bounds[nb++] = nl;
    return nb;
}

/* plan.hpp:88-115 */
int orc_group_levels(uint32_t n, const uint32_t* level_ptr, uint32_t nl, const uint32_t* rp_perm,
                     uint64_t cache_bytes, int p_m, uint32_t* group_rows,
                     uint32_t* group_level_ptr, uint64_t* group_fp, uint32_t* n_groups,
                     uint64_t* target_bytes) {
    (void)n;
    if (p_m < 1) return ORC_EINVAL;
    const uint64_t target = cache_bytes / (uint64_t)(p_m + 1);
    uint64_t* lfp = (uint64_t*)malloc(sizeof(uint64_t) * ((size_t)nl + 1));
    for (uint32_t l = 0; l < nl; ++l)
        lfp[l] = orc_row_range_footprint(rp_perm, level_ptr[l], level_ptr[l + 1], p_m);
    const uint32_t nb = orc_greedy_group(lfp, nl, target, group_level_ptr);
    for (uint32_t b = 0; b < nb; ++b) group_rows[b] = level_ptr[group_level_ptr[b]];
    for (uint32_t g = 0; g + 1 < nb; ++g) {
        uint64_t s = 0;
        for (uint32_t l = group_level_ptr[g]; l < group_level_ptr[g + 1]; ++l) s += lfp[l];
        group_fp[g] = s;
    }
    free(lfp);
    *n_groups = nb > 0 ? nb - 1 : 0;
    *target_bytes = target;
    return ORC_OK;
}

/* execute.hpp:59-72 */
uint64_t orc_wavefront_schedule(uint32_t ng, int stages, uint32_t* group, int* stage) {
    uint64_t cnt = 0;
    if (ng == 0 || stages <= 0) return 0;
    for (int64_t d = 0; d <= (int64_t)ng + stages - 2; ++d)
        for (int q = 1; q <= stages; ++q) {
            const int64_t g = d - (q - 1);
            if (g >= 0 && g < (int64_t)ng) {
                group[cnt] = (uint32_t)g;
                stage[cnt] = q;
                ++cnt;
            }
        }
    return cnt;
}

/* csr.hpp:115-123 */
void orc_spmv_rows(const uint32_t* rp, const uint32_t* ci, const double* vals, const double* x,
                   double* y, uint32_t row_s, uint32_t row_e) {
    for (uint32_t r = row_s; r < row_e; ++r) {
        double acc = 0.0;
        for (uint32_t k = rp[r]; k < rp[r + 1]; ++k) acc += vals[k] * x[ci[k]];
        y[r] = acc;
    }
}

/* mpk.hpp:59-75 */
int orc_baseline_mpk(uint32_t n, const uint32_t* rp, const uint32_t* ci, const double* vals,
                     const double* x, int p_m, double* block) {
    if (p_m < 1) return ORC_EINVAL;
    memcpy(block, x, sizeof(double) * n);
    for (int p = 1; p <= p_m; ++p)
        orc_spmv_rows(rp, ci, vals, block + (size_t)(p - 1) * n, block + (size_t)p * n, 0, n);
    return ORC_OK;
}

/* mpk.hpp:81-106 over execute.hpp:79-113 with a single worker: the cells run in wavefront
 * order, each over its whole group row range. */
int orc_mpk(uint32_t n, const uint32_t* rp, const uint32_t* ci, const double* vals,
            const uint32_t* group_rows, uint32_t ng, int plan_p_m, const double* x, int p_m,
            double* block) {
    if (p_m < 1 || p_m > plan_p_m) return ORC_EINVAL;
    memcpy(block, x, sizeof(double) * n);
    const uint64_t cells = (uint64_t)ng * (uint64_t)p_m;
    uint32_t* g = (uint32_t*)malloc(sizeof(uint32_t) * (cells + 1));
    int* q = (int*)malloc(sizeof(int) * (cells + 1));
    const uint64_t cnt = orc_wavefront_schedule(ng, p_m, g, q);
    for (uint64_t i = 0; i < cnt; ++i) {
        const int p = q[i];
        orc_spmv_rows(rp, ci, vals, block + (size_t)(p - 1) * n, block + (size_t)p * n,
                      group_rows[g[i]], group_rows[g[i] + 1]);
    }
    free(g);
    free(q);
    return ORC_OK;
}

/* mpk.hpp:111-127 */
int orc_check_shift_chain(const double* re, const double* im, int ns) {
    for (int i = 0; i < ns; ++i) {
        const double b = im[i];
        if (b == 0.0) continue;
        if (b < 0.0) return ORC_EINVAL;
        if (i + 1 == ns) return ORC_EINVAL;
        if (!(re[i + 1] == re[i] && im[i + 1] == -b)) return ORC_EINVAL;
        ++i;
    }
    return ORC_OK;
}

/* mpk.hpp:135-153 */
static void shifted_rows(const uint32_t* rp, const uint32_t* ci, const double* vals, double* dst,
                         const double* src, const double* src2, double a, double b2,
                         uint32_t row_s, uint32_t row_e) {
    for (uint32_t r = row_s; r < row_e; ++r) {
        double acc = 0.0;
        for (uint32_t k = rp[r]; k < rp[r + 1]; ++k) acc += vals[k] * src[ci[k]];
        if (b2 == 0.0)
            dst[r] = acc - a * src[r];
        else
            dst[r] = acc - a * src[r] + b2 * src2[r];
    }
}

static void shift_params(const double* re, const double* im, int p, double* a, double* b2) {
    const double bi = im[p - 1];
    *a = re[p - 1];
    *b2 = bi < 0.0 ? bi * bi : 0.0; /* mpk.hpp:171 / 201 */
}

/* mpk.hpp:160-180 */
int orc_baseline_mpk_shifted(uint32_t n, const uint32_t* rp, const uint32_t* ci,
                             const double* vals, const double* x, const double* re,
                             const double* im, int ns, double* block) {
    if (ns < 1) return ORC_EINVAL;
    if (orc_check_shift_chain(re, im, ns) != ORC_OK) return ORC_EINVAL;
    memcpy(block, x, sizeof(double) * n);
    for (int p = 1; p <= ns; ++p) {
        double a, b2;
        shift_params(re, im, p, &a, &b2);
        const double* src2 = p >= 2 ? block + (size_t)(p - 2) * n : NULL;
        shifted_rows(rp, ci, vals, block + (size_t)p * n, block + (size_t)(p - 1) * n, src2, a,
                     b2, 0, n);
    }
    return ORC_OK;
}

/* mpk.hpp:184-207 */
int orc_mpk_shifted(uint32_t n, const uint32_t* rp, const uint32_t* ci, const double* vals,
                    const uint32_t* group_rows, uint32_t ng, int plan_p_m, const double* x,
                    const double* re, const double* im, int ns, double* block) {
    if (ns < 1 || ns > plan_p_m) return ORC_EINVAL;
    if (orc_check_shift_chain(re, im, ns) != ORC_OK) return ORC_EINVAL;
    memcpy(block, x, sizeof(double) * n);
    const uint64_t cells = (uint64_t)ng * (uint64_t)ns;
    uint32_t* g = (uint32_t*)malloc(sizeof(uint32_t) * (cells + 1));
    int* q = (int*)malloc(sizeof(int) * (cells + 1));
    const uint64_t cnt = orc_wavefront_schedule(ng, ns, g, q);
    for (uint64_t i = 0; i < cnt; ++i) {
        const int p = q[i];
        double a, b2;
        shift_params(re, im, p, &a, &b2);
        const double* src2 = p >= 2 ? block + (size_t)(p - 2) * n : NULL;
        shifted_rows(rp, ci, vals, block + (size_t)p * n, block + (size_t)(p - 1) * n, src2, a,
                     b2, group_rows[g[i]], group_rows[g[i] + 1]);
    }
    free(g);
    free(q);
    return ORC_OK;
}

/* SURVEY §8(a) A23 restatement (coefficient form; the reference has none). */
void orc_poly_combine(uint32_t n, const double* block, const double* c, int d, double* z) {
    for (uint32_t r = 0; r < n; ++r) {
        double acc = c[0] * block[r];
        for (int k = 1; k <= d; ++k) acc += c[k] * block[(size_t)k * n + r];
        z[r] = acc;
    }
}

/* mpk.hpp:219-233 */
int orc_tune_select(const double* gflops, int p_lo, int p_hi) {
    int best_p = p_lo;
    double best = -1.0;
    for (int p = p_lo; p <= p_hi; ++p)
        if (gflops[p - p_lo] > best) {
            best = gflops[p - p_lo];
            best_p = p;
        }
    return best_p;
}

/* ---- Jacobi-preconditioned chains ------------------------------------------------------------ */

/* csr.hpp:233-243 + jacobi.hpp:48-64 */
int orc_diag_info(uint32_t n_rows, uint32_t n_cols, const uint32_t* rp, const uint32_t* ci,
                  const double* vals, uint32_t* pos, double* inv, uint32_t* bad_row) {
    if (n_rows != n_cols) return ORC_EINVAL;
    for (uint32_t r = 0; r < n_rows; ++r) {
        /* binary search for column r in the sorted row (lower_bound) */
        uint32_t lo = rp[r], hi = rp[r + 1];
        while (lo < hi) {
            const uint32_t mid = lo + (hi - lo) / 2;
            if (ci[mid] < r)
                lo = mid + 1;
            else
                hi = mid;
        }
        pos[r] = (lo < rp[r + 1] && ci[lo] == r) ? lo : ORC_NO_DIAG;
        if (pos[r] == ORC_NO_DIAG || vals[pos[r]] == 0.0) {
            if (bad_row) *bad_row = r;
            return ORC_ERUNTIME;
        }
        inv[r] = 1.0 / vals[pos[r]];
    }
    return ORC_OK;
}

/* jacobi.hpp:83-96 jacobi_sweep_rows: z_i = d_i v_i - d_i * sum_{k != diag} a_ik z_prev_k */
static void jacobi_sweep(const uint32_t* rp, const uint32_t* ci, const double* vals,
                         const uint32_t* pos, const double* inv, const double* v,
                         const double* z_prev, double* z_out, uint32_t n) {
    for (uint32_t r = 0; r < n; ++r) {
        double acc = 0.0;
        for (uint32_t k = rp[r]; k < rp[r + 1]; ++k) {
            if (k == pos[r]) continue;
            acc += vals[k] * z_prev[ci[k]];
        }
        z_out[r] = inv[r] * v[r] - inv[r] * acc;
    }
}

/* jacobi.hpp:155-174 */
void orc_jacobi_apply(uint32_t n, const uint32_t* rp, const uint32_t* ci, const double* vals,
                      const uint32_t* pos, const double* inv, int sweeps, const double* v,
                      double* z) {
    for (uint32_t r = 0; r < n; ++r) z[r] = inv[r] * v[r];
    if (sweeps <= 1) return;
    double* tmp = (double*)malloc(sizeof(double) * (n ? n : 1));
    for (int s = 2; s <= sweeps; ++s) {
        jacobi_sweep(rp, ci, vals, pos, inv, v, z, tmp, n);
        memcpy(z, tmp, sizeof(double) * n);
    }
    free(tmp);
}

/* jacobi.hpp:100-110 scaled_spmv_rows: y_r = sum_k a_rk * (d_c * x_c) */
static void scaled_spmv(const uint32_t* rp, const uint32_t* ci, const double* vals,
                        const double* inv, const double* x, double* y, uint32_t n) {
    for (uint32_t r = 0; r < n; ++r) {
        double acc = 0.0;
        for (uint32_t k = rp[r]; k < rp[r + 1]; ++k) acc += vals[k] * (inv[ci[k]] * x[ci[k]]);
        y[r] = acc;
    }
}

/* jacobi.hpp:120-149 chain stages, run in order (jacobi.hpp:177-192) */
void orc_jacobi_op(uint32_t n, const uint32_t* rp, const uint32_t* ci, const double* vals,
                   const uint32_t* pos, const double* inv, int sweeps, const double* v,
                   double* y) {
    if (sweeps <= 1) {
        scaled_spmv(rp, ci, vals, inv, v, y, n);
        return;
    }
    /* z^1 = D^{-1} v, z^{j+1} = sweep(z^j), y = A z^sweeps */
    double* z = (double*)malloc(sizeof(double) * (size_t)sweeps * (n ? n : 1));
    for (uint32_t r = 0; r < n; ++r) z[r] = inv[r] * v[r];
    for (int j = 1; j < sweeps; ++j)
        jacobi_sweep(rp, ci, vals, pos, inv, v, z + (size_t)(j - 1) * n, z + (size_t)j * n, n);
    orc_spmv_rows(rp, ci, vals, z + (size_t)(sweeps - 1) * n, y, 0, n);
    free(z);
}

/* sstep.hpp:68-157 (shifted_terminal_rows, scaled_shifted_spmv_rows, SstepJacobiChain) run by
 * run_chain_sequential (sstep.hpp:203-216) */
int orc_sstep_jacobi_block(uint32_t n, const uint32_t* rp, const uint32_t* ci,
                           const double* vals, const uint32_t* pos, const double* inv,
                           int sweeps, const double* re, const double* im, int ns,
                           double* block) {
    if (ns < 1) return ORC_EINVAL;
    if (orc_check_shift_chain(re, im, ns) != ORC_OK) return ORC_EINVAL;
    double* z = (double*)malloc(sizeof(double) * (size_t)(sweeps > 1 ? sweeps : 1) * (n ? n : 1));
    double* t = (double*)malloc(sizeof(double) * (n ? n : 1));
    for (int p = 1; p <= ns; ++p) {
        double a, b2;
        shift_params(re, im, p, &a, &b2);
        const double* src = block + (size_t)(p - 1) * n;
        const double* src2 = p >= 2 ? block + (size_t)(p - 2) * n : NULL;
        double* dst = block + (size_t)p * n;
        const double* zin;
        if (sweeps <= 1) {
            scaled_spmv(rp, ci, vals, inv, src, t, n); /* acc of scaled_shifted_spmv_rows */
            for (uint32_t r = 0; r < n; ++r)
                dst[r] = b2 == 0.0 ? t[r] - a * src[r] : t[r] - a * src[r] + b2 * src2[r];
            continue;
        }
        for (uint32_t r = 0; r < n; ++r) z[r] = inv[r] * src[r];
        for (int j = 1; j < sweeps; ++j)
            jacobi_sweep(rp, ci, vals, pos, inv, src, z + (size_t)(j - 1) * n, z + (size_t)j * n, n);
        zin = z + (size_t)(sweeps - 1) * n;
        orc_spmv_rows(rp, ci, vals, zin, t, 0, n);
        for (uint32_t r = 0; r < n; ++r)
            dst[r] = b2 == 0.0 ? t[r] - a * src[r] : t[r] - a * src[r] + b2 * src2[r];
    }
    free(z);
    free(t);
    return ORC_OK;
}

/* ---- GS2 (gs2.hpp) ------------------------------------------------------------------------------ */

/* gs2.hpp:70-82 gs2_stage0_rows */
static void gs2_stage0(const uint32_t* rp, const uint32_t* ci, const double* vals, const double* inv,
                       const double* v, const double* z_prev, double* g0, double* z_next, uint32_t n) {
    for (uint32_t r = 0; r < n; ++r) {
        double acc = 0.0;
        for (uint32_t k = rp[r]; k < rp[r + 1]; ++k) acc += vals[k] * z_prev[ci[k]];
        const double g = inv[r] * (v[r] - acc);
        g0[r] = g;
        if (z_next) z_next[r] = z_prev[r] + g;
    }
}

/* gs2.hpp:89-104 gs2_inner_rows */
static void gs2_inner(const uint32_t* rp, const uint32_t* ci, const double* vals, const uint32_t* pos,
                      const double* inv, const double* g0, const double* g_prev, double* g_out,
                      int forward, const double* z_prev, double* z_next, uint32_t n) {
    for (uint32_t r = 0; r < n; ++r) {
        const uint32_t ks = forward ? rp[r] : pos[r] + 1;
        const uint32_t ke = forward ? pos[r] : rp[r + 1];
        double acc = 0.0;
        for (uint32_t k = ks; k < ke; ++k) acc += vals[k] * g_prev[ci[k]];
        const double g = g0[r] - inv[r] * acc;
        g_out[r] = g;
        if (z_next) z_next[r] = z_prev[r] + g;
    }
}

/* gs2.hpp:108-116 residual_rows */
static void gs2_residual(const uint32_t* rp, const uint32_t* ci, const double* vals, const double* v,
                         const double* z, double* out, uint32_t n) {
    for (uint32_t r = 0; r < n; ++r) {
        double acc = 0.0;
        for (uint32_t k = rp[r]; k < rp[r + 1]; ++k) acc += vals[k] * z[ci[k]];
        out[r] = v[r] - acc;
    }
}

/* one K-sweep GS2 from z[0] (slices z[0..K], g[0..gamma]) : gs2.hpp:126-158 in chain order */
static void gs2_sweeps(uint32_t n, const uint32_t* rp, const uint32_t* ci, const double* vals,
                       const uint32_t* pos, const double* inv, int gamma, int sweeps, int forward,
                       const double* v, double* z, double* g) {
    for (int p = 1; p <= sweeps; ++p) {
        const double* z_prev = z + (size_t)(p - 1) * n;
        double* z_next = z + (size_t)p * n;
        gs2_stage0(rp, ci, vals, inv, v, z_prev, g, gamma == 0 ? z_next : NULL, n);
        for (int j = 1; j <= gamma; ++j)
            gs2_inner(rp, ci, vals, pos, inv, g, g + (size_t)(j - 1) * n, g + (size_t)j * n, forward,
                      z_prev, j == gamma ? z_next : NULL, n);
    }
}

void orc_gs2_chain(uint32_t n, const uint32_t* rp, const uint32_t* ci, const double* vals,
                   const uint32_t* pos, const double* inv, int gamma, int sweeps, int forward,
                   int terminal, const double* v, double* z_io, double* out) {
    const size_t nn = n ? n : 1;
    double* z = (double*)malloc(sizeof(double) * nn * (size_t)(sweeps + 1));
    double* g = (double*)malloc(sizeof(double) * nn * (size_t)(gamma + 1));
    memcpy(z, z_io, sizeof(double) * n);
    gs2_sweeps(n, rp, ci, vals, pos, inv, gamma, sweeps, forward, v, z, g);
    const double* zk = z + (size_t)sweeps * n;
    if (terminal == 1) orc_spmv_rows(rp, ci, vals, zk, out, 0, n);
    if (terminal == 2) gs2_residual(rp, ci, vals, v, zk, out, n);
    memcpy(z_io, zk, sizeof(double) * n);
    free(z);
    free(g);
}

int orc_sstep_gs2_block(uint32_t n, const uint32_t* rp, const uint32_t* ci, const double* vals,
                        const uint32_t* pos, const double* inv, int gamma, int sweeps, int forward,
                        const double* re, const double* im, int ns, double* block) {
    if (ns < 1) return ORC_EINVAL;
    if (orc_check_shift_chain(re, im, ns) != ORC_OK) return ORC_EINVAL;
    const size_t nn = n ? n : 1;
    double* z = (double*)calloc(nn * (size_t)(sweeps + 1), sizeof(double)); /* slice 0 stays 0 */
    double* g = (double*)malloc(sizeof(double) * nn * (size_t)(gamma + 1));
    double* t = (double*)malloc(sizeof(double) * nn);
    for (int p = 1; p <= ns; ++p) {
        double a, b2;
        shift_params(re, im, p, &a, &b2);
        const double* src = block + (size_t)(p - 1) * n;
        const double* src2 = p >= 2 ? block + (size_t)(p - 2) * n : NULL;
        double* dst = block + (size_t)p * n;
        gs2_sweeps(n, rp, ci, vals, pos, inv, gamma, sweeps, forward, src, z, g);
        orc_spmv_rows(rp, ci, vals, z + (size_t)sweeps * n, t, 0, n);
        for (uint32_t r = 0; r < n; ++r)
            dst[r] = b2 == 0.0 ? t[r] - a * src[r] : t[r] - a * src[r] + b2 * src2[r];
    }
    free(z);
    free(g);
    free(t);
    return ORC_OK;
}

/* ---- from_coo (csr.hpp:72-110) --------------------------------------------------------------- */
static const uint32_t* g_sort_rows;
static const uint32_t* g_sort_cols;

/* (row, col, input index): a total order, so any sort is the stable sort of csr.hpp:86-89 */
static int coo_cmp(const void* a, const void* b) {
    const uint64_t i = *(const uint64_t*)a, j = *(const uint64_t*)b;
    if (g_sort_rows[i] != g_sort_rows[j]) return g_sort_rows[i] < g_sort_rows[j] ? -1 : 1;
    if (g_sort_cols[i] != g_sort_cols[j]) return g_sort_cols[i] < g_sort_cols[j] ? -1 : 1;
    return i < j ? -1 : (i > j ? 1 : 0);
}

int orc_from_coo(uint32_t n_rows, uint32_t n_cols, uint64_t nnz, const uint32_t* rows,
                 const uint32_t* cols, const double* vals, uint32_t* row_ptr, uint32_t* col_idx,
                 double* values, uint64_t* out_nnz, uint64_t* bad) {
    if (nnz >= ((uint64_t)1 << 31)) return ORC_EINVAL;
    for (uint64_t i = 0; i < nnz; ++i)
        if (rows[i] >= n_rows || cols[i] >= n_cols) {
            if (bad) *bad = i;
            return ORC_EINVAL;
        }
    uint64_t* idx = (uint64_t*)malloc(sizeof(uint64_t) * (nnz ? nnz : 1));
    for (uint64_t i = 0; i < nnz; ++i) idx[i] = i;
    g_sort_rows = rows;
    g_sort_cols = cols;
    qsort(idx, nnz, sizeof(uint64_t), coo_cmp);
    memset(row_ptr, 0, sizeof(uint32_t) * ((size_t)n_rows + 1));
    uint64_t u = 0;
    for (uint64_t i = 0; i < nnz;) {
        const uint32_t r = rows[idx[i]], c = cols[idx[i]];
        double sum = 0.0;
        for (; i < nnz && rows[idx[i]] == r && cols[idx[i]] == c; ++i) sum += vals[idx[i]];
        col_idx[u] = c;
        values[u] = sum;
        ++u;
        row_ptr[r + 1] = (uint32_t)u;
    }
    for (uint32_t r = 0; r < n_rows; ++r)
        if (row_ptr[r + 1] < row_ptr[r]) row_ptr[r + 1] = row_ptr[r];
    *out_nnz = u;
    free(idx);
    return ORC_OK;
}

/* ---- product-form polynomial (poly.hpp:77-93, 146-281) -------------------------------------- */
int orc_poly_apply(uint32_t n, const uint32_t* rp, const uint32_t* ci, const double* vals,
                   const uint32_t* pos, const double* inv, int inner, int sweeps, int gamma,
                   int forward, const double* re, const double* im, int degree, const double* v,
                   double* z) {
    if (degree < 1) return ORC_EINVAL;
    unsigned char* role = (unsigned char*)malloc((size_t)degree);
    for (int i = 0; i < degree;) { /* poly_roles: 0 real, 1 pair first, 2 pair second */
        if (im[i] == 0.0) {
            role[i++] = 0;
            continue;
        }
        if (i + 1 >= degree || re[i + 1] != re[i] || im[i + 1] != -im[i]) {
            free(role);
            return ORC_EINVAL;
        }
        role[i] = 1, role[i + 1] = 2;
        i += 2;
    }
    const size_t nn = n ? n : 1;
    double* w = (double*)malloc(sizeof(double) * nn * (size_t)degree);
    double* zb = (double*)calloc(nn * (size_t)(sweeps > 2 ? sweeps : 2), sizeof(double));
    double* gb = (double*)malloc(sizeof(double) * nn * (size_t)(gamma + 1));
    double* t = (double*)malloc(sizeof(double) * nn);
    memcpy(w, v, sizeof(double) * n);
    for (uint32_t r = 0; r < n; ++r) z[r] = 0.0;
    for (int pw = 1; pw <= degree - 1; ++pw) {
        const double* w_in = w + (size_t)(pw - 1) * n;
        const double* z_src = w_in;
        int fused = 0;
        if (inner == 1) {
            if (sweeps == 1) {
                fused = 1;
            } else { /* stage 0 + sweeps (jacobi.hpp:83-117) into zb slices */
                for (uint32_t r = 0; r < n; ++r) zb[r] = inv[r] * w_in[r];
                for (int j = 1; j < sweeps; ++j)
                    jacobi_sweep(rp, ci, vals, pos, inv, w_in, zb + (size_t)(j - 1) * n, zb + (size_t)j * n, n);
                z_src = zb + (size_t)(sweeps - 1) * n;
            }
        } else if (inner == 2) { /* single GS2 sweep from the zero guess zb[0] into zb[1] */
            double* z0 = zb;
            double* z1 = zb + n;
            for (uint32_t r = 0; r < n; ++r) z0[r] = 0.0;
            gs2_stage0(rp, ci, vals, inv, w_in, z0, gb, gamma == 0 ? z1 : NULL, n);
            for (int j = 1; j <= gamma; ++j)
                gs2_inner(rp, ci, vals, pos, inv, gb, gb + (size_t)(j - 1) * n, gb + (size_t)j * n, forward,
                          z0, j == gamma ? z1 : NULL, n);
            z_src = z1;
        }
        if (fused)
            scaled_spmv(rp, ci, vals, inv, z_src, t, n);
        else
            orc_spmv_rows(rp, ci, vals, z_src, t, 0, n);
        const double th_re = re[pw - 1];
        const double mod = th_re * th_re + im[pw - 1] * im[pw - 1];
        double* w_out = w + (size_t)pw * n;
        for (uint32_t r = 0; r < n; ++r) {
            if (role[pw - 1] == 0) {
                z[r] += w_in[r] / th_re;
                w_out[r] = w_in[r] - t[r] / th_re;
            } else if (role[pw - 1] == 1) {
                const double u = 2.0 * th_re * w_in[r] - t[r];
                w_out[r] = u;
                z[r] += u / mod;
            } else {
                w_out[r] = w[(size_t)(pw - 2) * n + r] - t[r] / mod;
            }
        }
    }
    if (role[degree - 1] == 0) { /* trailing real root (poly.hpp:271-278) */
        const double th = re[degree - 1];
        const double* wl = w + (size_t)(degree - 1) * n;
        for (uint32_t r = 0; r < n; ++r) z[r] += wl[r] / th;
    }
    free(role);
    free(w);
    free(zb);
    free(gb);
    free(t);
    return ORC_OK;
}

/* ---- block orthogonalisation (ortho.hpp) ------------------------------------------------ */

void orc_block_dots(const double* q, const double* v, uint64_t rows, uint32_t qcols,
                    uint32_t vcols, double* c) {
    /* ortho.hpp:49-62: entry e = (k = e % qcols, j = e / qcols), serial over the rows */
    for (uint64_t e = 0; e < (uint64_t)qcols * vcols; ++e) {
        const double* qk = q + (e % qcols) * rows;
        const double* vj = v + (e / qcols) * rows;
        double acc = 0.0;
        for (uint64_t i = 0; i < rows; ++i) acc += qk[i] * vj[i];
        c[e] = acc;
    }
}

void orc_block_update(const double* q, const double* c, uint64_t rows, uint32_t qcols,
                      uint32_t vcols, double* v) {
    /* ortho.hpp:80-90 with one thread: for j, for k ascending, for i */
    for (uint32_t j = 0; j < vcols; ++j) {
        double* vj = v + (uint64_t)j * rows;
        for (uint32_t k = 0; k < qcols; ++k) {
            const double ck = c[(uint64_t)j * qcols + k];
            const double* qk = q + (uint64_t)k * rows;
            for (uint64_t i = 0; i < rows; ++i) vj[i] -= ck * qk[i];
        }
    }
}

int orc_icgs(const double* q, uint64_t rows, uint32_t qcols, double* v, uint32_t vcols,
             int sweeps, double* coeff) {
    const uint64_t ne = (uint64_t)qcols * vcols;
    if (ne == 0) return ORC_OK;             /* ortho.hpp:102-104 */
    if (sweeps < 1) return ORC_EINVAL;      /* ortho.hpp:105-107 */
    double* c = (double*)malloc(sizeof(double) * ne);
    for (uint64_t e = 0; e < ne; ++e) coeff[e] = 0.0;
    for (int sw = 0; sw < sweeps; ++sw) {   /* ortho.hpp:110-115 */
        orc_block_dots(q, v, rows, qcols, vcols, c);
        orc_block_update(q, c, rows, qcols, vcols, v);
        for (uint64_t e = 0; e < ne; ++e) coeff[e] += c[e];
    }
    free(c);
    return ORC_OK;
}

int orc_tsqr(double* v, uint64_t rows, uint32_t cols, double* r) {
    if (cols == 0) return ORC_OK;           /* ortho.hpp:148-150 */
    if (rows < cols) return ORC_EINVAL;     /* ortho.hpp:151-153 */
    const uint64_t c = cols;
    double* tau = (double*)malloc(sizeof(double) * c);
    double* a = v; /* factor in place: reflectors below the diagonal */
    for (uint64_t j = 0; j < c; ++j) {
        double* aj = a + j * rows;
        double sigma = 0.0;
        for (uint64_t i = j + 1; i < rows; ++i) sigma += aj[i] * aj[i];
        const double alpha = aj[j];
        double t = 0.0, beta = alpha;
        if (sigma != 0.0) {
            const double nrm = sqrt(alpha * alpha + sigma);
            beta = alpha >= 0.0 ? -nrm : nrm;
            t = (beta - alpha) / beta;
            const double s = 1.0 / (alpha - beta);
            for (uint64_t i = j + 1; i < rows; ++i) aj[i] *= s;
        } else {
            for (uint64_t i = j + 1; i < rows; ++i) aj[i] = 0.0;
        }
        aj[j] = beta;
        tau[j] = t;
        for (uint64_t l = j + 1; l < c && t != 0.0; ++l) {
            double* al = a + l * rows;
            double w = al[j];
            for (uint64_t i = j + 1; i < rows; ++i) w += aj[i] * al[i];
            w *= t;
            al[j] -= w;
            for (uint64_t i = j + 1; i < rows; ++i) al[i] -= w * aj[i];
        }
    }
    /* R with the sign fix (ortho.hpp:204-212, 221-226) */
    double* sg = (double*)malloc(sizeof(double) * c);
    for (uint64_t j = 0; j < c; ++j) sg[j] = a[j * rows + j] < 0.0 ? -1.0 : 1.0;
    for (uint64_t l = 0; l < c; ++l)
        for (uint64_t i = 0; i < c; ++i) r[l * c + i] = i <= l ? sg[i] * a[l * rows + i] : 0.0;
    /* explicit Q D = H_0 ... H_{c-1} [D; 0], applied right to left into a scratch block */
    double* y = (double*)malloc(sizeof(double) * rows * c);
    for (uint64_t l = 0; l < c; ++l)
        for (uint64_t i = 0; i < rows; ++i) y[l * rows + i] = i == l ? sg[l] : 0.0;
    for (uint64_t jj = c; jj-- > 0;) {
        if (tau[jj] == 0.0) continue;
        const double* h = a + jj * rows;
        for (uint64_t l = 0; l < c; ++l) {
            double* yl = y + l * rows;
            double w = yl[jj];
            for (uint64_t i = jj + 1; i < rows; ++i) w += h[i] * yl[i];
            w *= tau[jj];
            yl[jj] -= w;
            for (uint64_t i = jj + 1; i < rows; ++i) yl[i] -= w * h[i];
        }
    }
    memcpy(v, y, sizeof(double) * rows * c);
    free(y);
    free(sg);
    free(tau);
    return ORC_OK;
}
