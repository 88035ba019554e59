/*
 * TEST INFRASTRUCTURE ONLY — the CPU oracle for the level-blocked MPK path.
 *
 * A plain-C99 restatement of the reference algorithm (the mpk headers under /root/reference/proj/include),
 * each function citing the reference file:line it follows.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load this library, and only as the
 * checker or the CPU baseline.  The product path (paper_2309_02228_b200/libmpkg.so) never links
 * or calls it.
 *
 * Pinning: the restatement is checked bit-for-bit against (a) oracle/_ref/libmpkref.so, the
 * reference's own headers compiled in place with the reference flags (no -march => no FMA), and
 * (b) the golden fixtures in tests/golden/ generated from that library by
 * tests/golden/make_golden.py.
 *
 * Floating point contract (proj/include/mpk/mpk.hpp:68-73): each row is summed sequentially in
 * stored column order starting from 0.0 as `acc += v * x[c]` (a multiply then an add; this file
 * is compiled without -march so no FMA contraction is possible on x86-64).
 */
#ifndef MPK_ORACLE_H
#define MPK_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Return codes mirror the reference's exception classes. */
#define ORC_OK 0
#define ORC_EINVAL 1 /* std::invalid_argument */

/* levels.hpp:65-147.  level_ptr must hold n+1 entries; *n_levels receives the level count. */
int orc_build_levels(uint32_t n, const uint32_t* row_ptr, const uint32_t* col_idx,
                     uint32_t* levels, uint32_t* perm, uint32_t* inv_perm,
                     uint32_t* level_ptr, uint32_t* n_levels);

/* csr.hpp:145-155 (returns ORC_EINVAL if perm is not a permutation of [0,n)). */
int orc_check_permutation(const uint32_t* perm, uint32_t n);

/* csr.hpp:159-188.  Output arrays sized n+1 / nnz / nnz. */
int orc_permute(uint32_t n, const uint32_t* row_ptr, const uint32_t* col_idx,
                const double* values, const uint32_t* perm, uint32_t* out_row_ptr,
                uint32_t* out_col_idx, double* out_values);

/* csr.hpp:191-204. */
void orc_permute_vector(uint32_t n, const double* in, const uint32_t* perm, double* out);
void orc_unpermute_vector(uint32_t n, const double* in, const uint32_t* perm, double* out);

/* levels.hpp:151-164: 1 if every nonzero of A_perm couples levels at most one apart. */
int orc_validate_levels(uint32_t n, const uint32_t* row_ptr, const uint32_t* col_idx,
                        const uint32_t* levels, const uint32_t* inv_perm);

/* plan.hpp:59-64. */
uint64_t orc_row_range_footprint(const uint32_t* row_ptr, uint32_t row_s, uint32_t row_e, int p_m);

/* plan.hpp:70-85.  bounds must hold n_levels+1 entries; returns the number of bounds. */
uint32_t orc_greedy_group(const uint64_t* level_fp, uint32_t n_levels, uint64_t target,
                          uint32_t* bounds);

/* plan.hpp:88-115.  group arrays sized n_levels+1 (group_fp: n_levels). */
int orc_group_levels(uint32_t n, const uint32_t* level_ptr, uint32_t n_levels,
                     const uint32_t* row_ptr_perm, uint64_t cache_bytes, int p_m,
                     uint32_t* group_rows, uint32_t* group_level_ptr, uint64_t* group_fp,
                     uint32_t* n_groups, uint64_t* target_bytes);

/* execute.hpp:59-72.  Arrays sized n_groups*stages; returns the cell count. */
uint64_t orc_wavefront_schedule(uint32_t n_groups, int stages, uint32_t* group, int* stage);

/* csr.hpp:115-123. */
void orc_spmv_rows(const uint32_t* row_ptr, const uint32_t* col_idx, const double* values,
                   const double* x, double* y, uint32_t row_s, uint32_t row_e);

/* mpk.hpp:59-75.  block is slice-major (p_m+1)*n. */
int orc_baseline_mpk(uint32_t n, const uint32_t* row_ptr, const uint32_t* col_idx,
                     const double* values, const double* x, int p_m, double* block);

/* mpk.hpp:81-106 driven by execute.hpp:79-113 (serial wavefront). */
int orc_mpk(uint32_t n, const uint32_t* row_ptr, const uint32_t* col_idx, const double* values,
            const uint32_t* group_rows, uint32_t n_groups, int plan_p_m, const double* x,
            int p_m, double* block);

/* mpk.hpp:111-127: ORC_OK or ORC_EINVAL. */
int orc_check_shift_chain(const double* re, const double* im, int n_shifts);

/* mpk.hpp:160-180. */
int orc_baseline_mpk_shifted(uint32_t n, const uint32_t* row_ptr, const uint32_t* col_idx,
                             const double* values, const double* x, const double* re,
                             const double* im, int n_shifts, double* block);

/* mpk.hpp:184-207. */
int orc_mpk_shifted(uint32_t n, const uint32_t* row_ptr, const uint32_t* col_idx,
                    const double* values, const uint32_t* group_rows, uint32_t n_groups,
                    int plan_p_m, const double* x, const double* re, const double* im,
                    int n_shifts, double* block);

/* SURVEY §8(a) A23 (not in the reference): z = c_0*y_0, then z += c_k*y_k for
 * k = 1..d ascending, each a multiply then an add, over a power block from orc_baseline_mpk. */
void orc_poly_combine(uint32_t n, const double* block, const double* c, int d, double* z);

/* ---- Jacobi-preconditioned chains ------------------------------------ */
#define ORC_ERUNTIME 2 /* std::runtime_error (missing / zero diagonal) */
#define ORC_NO_DIAG 0xffffffffu /* csr.hpp:231 kNoDiag */

/* csr.hpp:233-243 diagonal_positions + jacobi.hpp:48-64 build_diag_info: pos[r] = index of
 * A(r,r) in col_idx (ORC_NO_DIAG if absent), inv[r] = 1.0 / A(r,r).  ORC_EINVAL if not square,
 * ORC_ERUNTIME (row in *bad_row) if a diagonal is missing or zero. */
int orc_diag_info(uint32_t n_rows, uint32_t n_cols, const uint32_t* row_ptr,
                  const uint32_t* col_idx, const double* values, uint32_t* pos, double* inv,
                  uint32_t* bad_row);

/* jacobi.hpp:155-174 jacobi_apply: z = M^{-1} v with `sweeps` zero-guess Jacobi sweeps. */
void orc_jacobi_apply(uint32_t n, const uint32_t* row_ptr, const uint32_t* col_idx,
                      const double* values, const uint32_t* pos, const double* inv, int sweeps,
                      const double* v, double* z);

/* jacobi.hpp:177-192 jacobi_op (== jacobi_op_blocked, jacobi.hpp:196-209): y = A (M^{-1} v)
 * through the chain stages of JacobiOpChain (jacobi.hpp:120-149). */
void orc_jacobi_op(uint32_t n, const uint32_t* row_ptr, const uint32_t* col_idx,
                   const double* values, const uint32_t* pos, const double* inv, int sweeps,
                   const double* v, double* y);

/* sstep.hpp:122-157 SstepJacobiChain run in order (sstep.hpp:203-216 run_chain_sequential,
 * the ordered twin of the blocked executor): w_p = (A M^{-1} - a_p) w_{p-1} (+ b2_p w_{p-2}),
 * p = 1..ns; block slice 0 holds the start vector on entry.  ORC_EINVAL for a bad shift chain.
 * sstep.hpp needs Eigen (absent here), so this chain is pinned by composition: with zero shifts
 * it is jacobi_op applied ns times (pinned against the compiled jacobi.hpp) and its terminal is
 * mpk.hpp's shifted row formula (pinned through orc_baseline_mpk_shifted). */
int orc_sstep_jacobi_block(uint32_t n, const uint32_t* row_ptr, const uint32_t* col_idx,
                           const double* values, const uint32_t* pos, const double* inv,
                           int sweeps, const double* re, const double* im, int ns,
                           double* block);

/* gs2.hpp:123-196 run_gs2_chain (K-sweep two-stage Gauss-Seidel: stage 0 scaled residual,
 * gamma inner Jacobi-Richardson iterations over the strict lower (forward) / upper (backward)
 * part, optional terminal on the last sweep).  terminal: 0 none, 1 apply_a (out = A z),
 * 2 residual (out = v - A z).  z_io holds the initial guess in and the iterate out. */
void orc_gs2_chain(uint32_t n, const uint32_t* row_ptr, const uint32_t* col_idx,
                   const double* values, const uint32_t* pos, const double* inv, int gamma,
                   int sweeps, int forward, int terminal, const double* v, double* z_io,
                   double* out);

/* sstep.hpp:160-198 SstepGs2Chain run in order (plan power q = (p-1)*K + sweep): every basis
 * power applies the full K-sweep zero-guess GS2 to w_{p-1}, the last sweep's terminal emits
 * w_p = A z - a_p w_{p-1} (+ b2_p w_{p-2}).  Pinned by composition like the Jacobi chain: with
 * zero shifts it is gs2_op applied ns times (gs2_op pinned against the compiled gs2.hpp). */
int orc_sstep_gs2_block(uint32_t n, const uint32_t* row_ptr, const uint32_t* col_idx,
                        const double* values, const uint32_t* pos, const double* inv, int gamma,
                        int sweeps, int forward, const double* re, const double* im, int ns,
                        double* block);

/* poly.hpp:146-281 run_poly_chain (product-form GMRES polynomial):
 * z = p(A M^{-1}) v for the given roots theta (re, im; conjugate pairs adjacent, + imaginary part
 * first), inner: 0 none, 1 Jacobi (sweeps), 2 GS2 (gamma, forward; single sweep).  ORC_EINVAL if
 * a conjugate pair is not adjacent (poly.hpp:77-93).  poly.hpp needs Eigen (absent here), so
 * this restatement is checked by the polynomial identity A z = v - prod_i (I - A/theta_i) v on
 * exactly-known spectra and by composition with the pinned Jacobi / GS2 stages. */
int orc_poly_apply(uint32_t n, const uint32_t* row_ptr, const uint32_t* col_idx,
                   const double* values, const uint32_t* pos, const double* inv, int inner,
                   int sweeps, int gamma, int forward, const double* re, const double* im,
                   int degree, const double* v, double* z);

/* csr.hpp:72-110 from_coo: stable (row, col) sort, duplicates summed in input order starting
 * from 0.0, empty rows filled.  Outputs sized n_rows+1 / nnz / nnz; *out_nnz = unique entries.
 * ORC_EINVAL (first offending entry in *bad) when an index is out of range. */
int orc_from_coo(uint32_t n_rows, uint32_t n_cols, uint64_t nnz, const uint32_t* rows,
                 const uint32_t* cols, const double* vals, uint32_t* row_ptr, uint32_t* col_idx,
                 double* values, uint64_t* out_nnz, uint64_t* bad);

/* ---- block orthogonalisation (ortho.hpp) ----------------------------
 * ortho.hpp needs Eigen (absent here), so these restatements are pinned by the reference's own
 * known-answer tests (test_ortho.cpp: exactly-orthogonal input untouched, coefficients that
 * reconstruct a known projection, duplicates projecting to zero, tsqr bounds / identity R /
 * rank deficiency / panel-tree agreement), restated in tests/test_oracle.py.
 * Blocks are column-major with leading dimension rows. */
/* ortho.hpp:46-63: c[j*qcols+k] = serial ascending sum of q_k[i] * v_j[i] from 0.0. */
void orc_block_dots(const double* q, const double* v, uint64_t rows, uint32_t qcols,
                    uint32_t vcols, double* c);
/* ortho.hpp:67-92: v_j[i] -= c[j*qcols+k] * q_k[i] for k ascending. */
void orc_block_update(const double* q, const double* c, uint64_t rows, uint32_t qcols,
                      uint32_t vcols, double* v);
/* ortho.hpp:97-117: `sweeps` x (dots, update), coeff accumulated from 0.0.  ORC_EINVAL if
 * sweeps < 1 with a non-empty block; an empty one returns ORC_OK untouched. */
int orc_icgs(const double* q, uint64_t rows, uint32_t qcols, double* v, uint32_t vcols,
             int sweeps, double* coeff);
/* ortho.hpp:136-229 tsqr, restated as one Householder QR of the whole block (LAPACK
 * convention: beta = -sign(alpha) |x|, tau = (beta - alpha) / beta), then the sign fix to a
 * non-negative R diagonal (ortho.hpp:204-212).  (Q, R) is unique for a full-rank block, so
 * this equals the reference's panel tree to roundoff.  ORC_EINVAL if rows < cols. */
int orc_tsqr(double* v, uint64_t rows, uint32_t cols, double* r);

/* mpk.hpp:219-233: argmax over the table, ties toward the smaller p. */
int orc_tune_select(const double* gflops, int p_lo, int p_hi);

#ifdef __cplusplus
}
#endif

#endif
