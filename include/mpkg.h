/*
 * mpkg — B200-native level-blocked matrix power kernel (MPK), C ABI.
 *
 * This is the drop-in boundary for the reference's C++ MPK interface (namespace mpk, header-only,
 * /root/reference/proj/include/mpk/).  Every entry point below names the reference symbol it
 * replaces (file:line).  The C++ facade in include/mpkg.hpp restores the reference's types,
 * names and exceptions on top of these functions, so a reference call site switches with
 * `namespace mpk = mpkg;`.
 *
 * Conventions
 *  - Every function returns an int status (MPKG_OK on success).  No exception crosses the ABI;
 *    the facade maps MPKG_EINVAL -> std::invalid_argument, MPKG_ERANGE -> std::out_of_range,
 *    everything else -> std::runtime_error.  mpkg_last_error() holds a thread-local message.
 *  - Indices are uint32 (reference index_t, csr.hpp:41); values are IEEE fp64.
 *  - Power workspaces ("blocks") are slice-major: slice p of a block with `rows` rows starts at
 *    block + p*rows (reference VectorBlock, vector_block.hpp:38-57).  Slice 0 receives x.
 *  - Functions without a suffix take HOST pointers and are synchronous (they mirror the
 *    reference's synchronous calls).  `_dev` variants take DEVICE pointers and enqueue on the
 *    context's stream without synchronising.
 *  - Handles are not thread-safe; use one context per device ("safe to call from
 *    one thread at a time per plan").  Immutable objects (csr, levels, plan) may be shared.
 *  - There is no CPU fallback: with no usable CUDA device every compute entry point fails with
 *    MPKG_ECUDA.
 */
#ifndef MPKG_H
#define MPKG_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MPKG_ABI_VERSION 1

/* Status codes. */
#define MPKG_OK 0
#define MPKG_EINVAL 1    /* reference: std::invalid_argument */
#define MPKG_ERANGE 2    /* reference: std::out_of_range (VectorBlock::slice) */
#define MPKG_ECUDA 3     /* CUDA runtime failure / no device */
#define MPKG_ENOMEM 4    /* device or host allocation failed */
#define MPKG_EINTERNAL 5 /* anything else */

/* Arithmetic modes (mpkg_ctx_set_mode). */
#define MPKG_MODE_BITWISE 0 /* one sequential accumulator per row in stored column order,
                               __dmul_rn + __dadd_rn: bit-identical to the reference CPU build */
#define MPKG_MODE_FAST 1    /* mpk / mpk_shifted / mpk_poly only: rows longer than the SELL
                               long-row cap (1024) are reduced in parallel (fixed-shape tree,
                               deterministic) instead of in stored order, so power-law hubs no
                               longer serialise a power; every other row and every baseline_*
                               result stays bitwise.  Checked to the north star's 1e-12
                               inf-norm relative bound per basis vector. */

typedef struct mpkg_ctx_s* mpkg_ctx_t;
typedef struct mpkg_csr_s* mpkg_csr_t;
typedef struct mpkg_levels_s* mpkg_levels_t;
typedef struct mpkg_plan_s* mpkg_plan_t;
typedef struct mpkg_jacobi_s* mpkg_jacobi_t;
typedef struct mpkg_gs2_s* mpkg_gs2_t;
typedef struct mpkg_host_csr_s* mpkg_host_csr_t;
typedef struct mpkg_dist_s* mpkg_dist_t;

/* ---- errors / version ------------------------------------------------------------------- */
const char* mpkg_last_error(void);
int mpkg_abi_version(void);

/* ---- context (replaces threading.hpp:34-46 resolve_threads: device + stream selection) --- */
int mpkg_ctx_create(int device, mpkg_ctx_t* out);
int mpkg_ctx_destroy(mpkg_ctx_t ctx);
int mpkg_ctx_stream(mpkg_ctx_t ctx, void** cuda_stream);
int mpkg_ctx_synchronize(mpkg_ctx_t ctx);
int mpkg_ctx_set_mode(mpkg_ctx_t ctx, int mode);
/* Device facts the planner uses: SM count, L2 bytes, max persisting-L2 bytes. */
int mpkg_ctx_device_info(mpkg_ctx_t ctx, int* sm_count, size_t* l2_bytes, size_t* persist_max);
/* Executor tuning knobs: "slack" (tickets between a dependency and its
 * consumer in the list schedule; -1 = auto), "order" (0: A_perm order, 1: Cuthill-McKee inside
 * levels), "pass" (force powers per fused pass; 0 = auto from the L2 budget), "l2_budget" (live
 * window bytes; 0 = 0.6 x L2), "tile_rows" (fixed 256); "kernel_timing" = 1 records a CUDA event
 * pair around every power-kernel launch on the context stream; "schedule" (0 auto, 1 fused
 * tile-DAG kernel, 2 one launch per power, 3 the wave: passes of p' powers with cross-power L2
 * reuse); "trace" (1: per (tile, power) device timestamps, mpkg_plan_exec_trace); "graphs" (replay the per-power launches as one CUDA
 * graph, default 1); "pdl" (default 1: programmatic dependent launch between consecutive
 * powers, hiding the launch gap); "resident" (default 0; 1: a matrix that fits half the L2 together with its p+1
 * working vectors runs all powers of a device-pointer call in one cooperative launch);
 * "ortho_fused" (fast-mode ICGS: 0 unfused, 1 update fused with the next dots re-reading Q from
 * L1/L2, 2 the same with Q staged in shared memory, default); "sweep_variant" (0..5) and
 * "coop_variant" (0..3) select row-loop variants for experiments. */
int mpkg_ctx_set_param(mpkg_ctx_t ctx, const char* key, int64_t value);
/* Reads (and clears) the event pairs recorded with "kernel_timing": sum, count and max of the
 * per-launch device durations in milliseconds.  Synchronises on the recorded events. */
int mpkg_ctx_kernel_times(mpkg_ctx_t ctx, double* total_ms, uint64_t* count, double* max_ms);
/* Kernel launches issued by this context since creation (instrumentation for bench.py). */
int mpkg_ctx_launch_count(mpkg_ctx_t ctx, uint64_t* launches);

/* ---- device CSR (csr.hpp:57-65 CsrMatrix) ------------------------------------------------- */
/* Uploads a square or rectangular CSR (row_ptr[n_rows+1], col_idx[nnz], values[nnz]).
 * Validates the csr.hpp:53-56 invariants (row_ptr monotone from 0, columns in range, strictly
 * ascending within each row) and fails with MPKG_EINVAL otherwise. */
int mpkg_csr_create(mpkg_ctx_t ctx, uint32_t n_rows, uint32_t n_cols, const uint32_t* row_ptr,
                    const uint32_t* col_idx, const double* values, mpkg_csr_t* out);
int mpkg_csr_create_from_host(mpkg_ctx_t ctx, mpkg_host_csr_t h, mpkg_csr_t* out);
int mpkg_csr_info(mpkg_csr_t A, uint32_t* n_rows, uint32_t* n_cols, uint32_t* nnz);
int mpkg_csr_download(mpkg_csr_t A, uint32_t* row_ptr, uint32_t* col_idx, double* values);
int mpkg_csr_destroy(mpkg_csr_t A);

/* csr.hpp:126-142 spmv: y = A x (bitwise row formula of csr.hpp:115-123). */
int mpkg_spmv(mpkg_ctx_t ctx, mpkg_csr_t A, const double* x, double* y);
int mpkg_spmv_dev(mpkg_ctx_t ctx, mpkg_csr_t A, const double* d_x, double* d_y);

/* ---- level engine (levels.hpp) ------------------------------------------------------------ */
/* levels.hpp:65-147 build_levels: GPU BFS, bit-exact levels / perm / inv_perm / level_ptr. */
int mpkg_build_levels(mpkg_ctx_t ctx, mpkg_csr_t A, mpkg_levels_t* out);
/* Build a level structure from host arrays (used to hand an externally built structure, e.g. a
 * reference LevelStructure, to group_levels / validate_levels). level_ptr has n_levels+1. */
int mpkg_levels_create(mpkg_ctx_t ctx, uint32_t n_rows, uint32_t n_levels,
                       const uint32_t* levels, const uint32_t* perm, const uint32_t* inv_perm,
                       const uint32_t* level_ptr, mpkg_levels_t* out);
int mpkg_levels_info(mpkg_levels_t L, uint32_t* n_rows, uint32_t* n_levels);
/* Any output pointer may be NULL.  level_ptr receives n_levels+1 entries. */
int mpkg_levels_get(mpkg_levels_t L, uint32_t* levels, uint32_t* perm, uint32_t* inv_perm,
                    uint32_t* level_ptr);
int mpkg_levels_destroy(mpkg_levels_t L);
/* levels.hpp:151-164 validate_levels: *ok = 1 iff every nonzero couples levels <= 1 apart. */
int mpkg_validate_levels(mpkg_ctx_t ctx, mpkg_csr_t A_perm, mpkg_levels_t L, int* ok);

/* ---- permutation (csr.hpp:145-204) -------------------------------------------------------- */
/* csr.hpp:159-188 permute with a host permutation (old -> new).  MPKG_EINVAL if not square or
 * perm is not a permutation (csr.hpp:145-155). */
int mpkg_permute(mpkg_ctx_t ctx, mpkg_csr_t A, const uint32_t* perm, mpkg_csr_t* out);
/* Same, with the device-resident perm of a level structure (no host round trip). */
/* csr.hpp:72-110 from_coo on the GPU: stable (row, col) sort, duplicates
 * summed in input order from 0.0, empty rows filled; bit-identical to the reference.  EINVAL:
 * nnz >= 2^31 or an index out of range (the first offending entry, in input order). */
int mpkg_csr_from_coo(mpkg_ctx_t ctx, uint32_t n_rows, uint32_t n_cols, uint64_t nnz,
                      const uint32_t* rows, const uint32_t* cols, const double* vals,
                      mpkg_csr_t* out);
int mpkg_csr_from_coo_dev(mpkg_ctx_t ctx, uint32_t n_rows, uint32_t n_cols, uint64_t nnz,
                          const uint32_t* d_rows, const uint32_t* d_cols, const double* d_vals,
                          mpkg_csr_t* out);
/* matrix_market.hpp:48-113 read_matrix_market: the reference's format
 * rules and messages (EINTERNAL = std::runtime_error); text parsed on the host, assembled by the
 * GPU from_coo. */
int mpkg_read_matrix_market(mpkg_ctx_t ctx, const char* path, mpkg_csr_t* out);

/* Shard support (multi-GPU level ranges): B = A[r0:r1, c0:c1] on the device,
 * column indices shifted by -c0, kept entries in stored order. */
int mpkg_csr_block(mpkg_ctx_t ctx, mpkg_csr_t A, uint32_t r0, uint32_t r1, uint32_t c0,
                   uint32_t c1, mpkg_csr_t* out);
int mpkg_permute_levels(mpkg_ctx_t ctx, mpkg_csr_t A, mpkg_levels_t L, mpkg_csr_t* out);
/* csr.hpp:191-204: out[perm[i]] = in[i] / out[i] = in[perm[i]] (host arrays). */
int mpkg_permute_vector(mpkg_ctx_t ctx, uint32_t n, const double* in, const uint32_t* perm,
                        double* out);
int mpkg_unpermute_vector(mpkg_ctx_t ctx, uint32_t n, const double* in, const uint32_t* perm,
                          double* out);

/* ---- plan (plan.hpp) ----------------------------------------------------------------------- */
/* plan.hpp:59-64 row_range_footprint over a device CSR. */
int mpkg_row_range_footprint(mpkg_csr_t A_perm, uint32_t row_s, uint32_t row_e, int p_m,
                             uint64_t* bytes);
/* plan.hpp:70-85 greedy_group (pure host function).  bounds holds n_levels+1 entries. */
int mpkg_greedy_group(const uint64_t* level_fp, uint32_t n_levels, uint64_t target,
                      uint32_t* bounds, uint32_t* n_bounds);
/* plan.hpp:88-115 group_levels. */
int mpkg_group_levels(mpkg_ctx_t ctx, mpkg_levels_t L, mpkg_csr_t A_perm, uint64_t cache_bytes,
                      int p_m, mpkg_plan_t* out);
/* Builds a plan from host fields (plan.hpp:41-54 ExecutionPlan), e.g. one made by hand as in
 * the reference's schedule tests.  level_ptr (n_levels+1 entries) may be NULL: the executor
 * then derives dependencies without level buckets (still exact, coarser). */
int mpkg_plan_create(int p_m, int sub_powers, uint32_t n_rows, uint64_t cache_bytes,
                     uint64_t target_bytes, uint32_t n_groups, const uint32_t* group_rows,
                     const uint32_t* group_level_ptr, const uint64_t* group_footprint,
                     uint32_t n_levels, const uint32_t* level_ptr, mpkg_plan_t* out);
int mpkg_plan_info(mpkg_plan_t P, int* p_m, int* sub_powers, uint32_t* n_rows,
                   uint64_t* cache_bytes, uint64_t* target_bytes, uint32_t* n_groups);
/* Any output may be NULL: group_rows / group_level_ptr have n_groups+1, footprint n_groups. */
int mpkg_plan_get(mpkg_plan_t P, uint32_t* group_rows, uint32_t* group_level_ptr,
                  uint64_t* group_footprint);
int mpkg_plan_destroy(mpkg_plan_t P);
/* Executor statistics for the GPU schedule attached to a plan (after the first mpkg_mpk):
 * tiles, tickets, dependency ranges. */
int mpkg_plan_exec_info(mpkg_plan_t P, uint32_t* n_tiles, uint64_t* n_tickets,
                        uint64_t* n_dep_tiles, uint32_t* pass_powers);
/* How the last mpkg_mpk* on this plan ran: private row order (0 A_perm, 1 Cuthill-McKee inside
 * levels, 2 longest rows first), schedule (1: one launch per power, 2: the wave schedule, one
 * persistent launch per pass of p' powers; 0: one fused tile-DAG launch), fused kernel variant,
 * rows handled outside the SELL arrays (long rows). */
int mpkg_plan_exec_mode(mpkg_plan_t P, int* order, int* sweeps, int* kernel, uint64_t* long_rows);
/* The wave schedule's private matrix copy (chunk records of 32 rows): record format (0 plain, 1
 * value dictionary), chunks, chunks stored as affine records (diagonal pieces: 8 column bases and 8
 * values for the whole chunk), chunks stored as banded records (rows that are sub-sequences of two
 * such templates), and the bytes of all records.  Zeros when the plan has no wave. */
int mpkg_plan_exec_wave(mpkg_plan_t P, int* format, uint64_t* n_chunks, uint64_t* n_affine,
                        uint64_t* n_banded, uint64_t* record_bytes);
/* Schedule audit (ctx knob "trace" = 1): after an mpkg_mpk* on the fused or wave schedule, the
 * 2 * n_tiles * (p+1) globaltimer stamps of the last call, [2 (q n_tiles + T)] = tile T's inputs for
 * power q complete, [.. + 1] = its results about to be stored / published; out may be NULL to
 * query n_stamps and the tile size.  The acceptance.cpp:188-251 predecessor audit replays on it. */
int mpkg_plan_exec_trace(mpkg_plan_t P, uint64_t* out, uint64_t capacity, uint64_t* n_stamps,
                         uint32_t* tile_rows);

/* execute.hpp:59-72 wavefront_schedule (pure host function; arrays hold n_groups*stages). */
int mpkg_wavefront_schedule(uint32_t n_groups, int stages, uint32_t* group, int* stage,
                            uint64_t* n_cells);

/* ---- power kernels (mpk.hpp) --------------------------------------------------------------- */
/* mpk.hpp:59-75 baseline_mpk: p_m back-to-back SpMV launches.  block has block_rows x
 * block_slices; MPKG_EINVAL unless A square, p_m >= 1, block_rows == n and
 * block_slices >= p_m+1 (mpk.hpp:44-53). */
int mpkg_baseline_mpk(mpkg_ctx_t ctx, mpkg_csr_t A, const double* x, int p_m, double* block,
                      uint64_t block_rows, uint64_t block_slices);
int mpkg_baseline_mpk_dev(mpkg_ctx_t ctx, mpkg_csr_t A, const double* d_x, int p_m,
                          double* d_block, uint64_t block_rows, uint64_t block_slices);

/* mpk.hpp:81-106 mpk.  The executor picks the schedule (mpkg_ctx_set_param "schedule", 0 = auto):
 * the wave -- one persistent launch per pass of p' powers with cross-power L2 reuse, tickets
 * synchronised by value -- for large matrices whose rows have at most 8 entries, otherwise one
 * launch per power replayed as a CUDA graph; the fused tile-DAG kernel (device-side completion
 * flags) on request.  mpkg_plan_exec_info reports which ran.
 * A_perm must be level-permuted, x in permuted order; p_m <= the plan's p_m (execute.hpp:81-83).
 * Bitwise equal to mpkg_baseline_mpk on A_perm in MPKG_MODE_BITWISE. */
int mpkg_mpk(mpkg_ctx_t ctx, mpkg_plan_t P, mpkg_csr_t A_perm, const double* x, int p_m,
             double* block, uint64_t block_rows, uint64_t block_slices);
int mpkg_mpk_dev(mpkg_ctx_t ctx, mpkg_plan_t P, mpkg_csr_t A_perm, const double* d_x, int p_m,
                 double* d_block, uint64_t block_rows, uint64_t block_slices);

/* mpk.hpp:111-127 check_shift_chain over shifts re[i] + i*im[i]. */
int mpkg_check_shift_chain(const double* re, const double* im, int n_shifts);

/* mpk.hpp:160-180 baseline_mpk_shifted / mpk.hpp:184-207 mpk_shifted (Newton basis
 * y_p = (A - lambda_p I) y_{p-1}; conjugate pairs via the two-step real formulation). */
int mpkg_baseline_mpk_shifted(mpkg_ctx_t ctx, mpkg_csr_t A, const double* x, const double* re,
                              const double* im, int n_shifts, double* block, uint64_t block_rows,
                              uint64_t block_slices);
int mpkg_baseline_mpk_shifted_dev(mpkg_ctx_t ctx, mpkg_csr_t A, const double* d_x,
                                  const double* re, const double* im, int n_shifts,
                                  double* d_block, uint64_t block_rows, uint64_t block_slices);
int mpkg_mpk_shifted(mpkg_ctx_t ctx, mpkg_plan_t P, mpkg_csr_t A_perm, const double* x,
                     const double* re, const double* im, int n_shifts, double* block,
                     uint64_t block_rows, uint64_t block_slices);
int mpkg_mpk_shifted_dev(mpkg_ctx_t ctx, mpkg_plan_t P, mpkg_csr_t A_perm, const double* d_x,
                         const double* re, const double* im, int n_shifts, double* d_block,
                         uint64_t block_rows, uint64_t block_slices);

/* Coefficient-form polynomial z = sum_{k=0..d} c_k A^k x (the reference has
 * no such API).  Accumulated inside the fused kernel in ascending k, each term a
 * multiply then an add.  block may be NULL (then an internal workspace holds y_1..y_d). */
int mpkg_mpk_poly(mpkg_ctx_t ctx, mpkg_plan_t P, mpkg_csr_t A_perm, const double* x,
                  const double* c, int d, double* z, double* block, uint64_t block_rows,
                  uint64_t block_slices);
int mpkg_mpk_poly_dev(mpkg_ctx_t ctx, mpkg_plan_t P, mpkg_csr_t A_perm, const double* d_x,
                      const double* c, int d, double* d_z, double* d_block, uint64_t block_rows,
                      uint64_t block_slices);

/* mpk.hpp:211-258 tune_p: plan per p, one warm-up, median of max(reps,3) CUDA-event-timed runs,
 * GF/s = 2*nnz*p/t; argmax with ties toward the smaller p.  gflops_table has p_hi-p_lo+1. */
int mpkg_tune_p(mpkg_ctx_t ctx, mpkg_levels_t L, mpkg_csr_t A_perm, uint64_t cache_bytes,
                int p_lo, int p_hi, int reps, int* p_opt, double* gflops_table);
/* mpk.hpp:219-233 tune_p(trial) selection rule over a given throughput table. */
int mpkg_tune_select(const double* gflops_table, int p_lo, int p_hi, int* p_opt);

/* ---- Jacobi-preconditioned chains (jacobi.hpp, sstep.hpp:68-157) ------
 * Bitwise equal to the reference's sequential and cache-blocked paths (same per-row formulas,
 * stored-order sums, no FMA). */
/* jacobi.hpp:48-76 build_diag_info + jacobi_setup: EINVAL (not square, sweeps < 1),
 * EINTERNAL = std::runtime_error (missing / zero diagonal: first failing row in the message). */
int mpkg_jacobi_setup(mpkg_ctx_t ctx, mpkg_csr_t A, int sweeps, mpkg_jacobi_t* out);
int mpkg_jacobi_info(mpkg_jacobi_t J, uint32_t* n, int* sweeps);
/* DiagInfo (jacobi.hpp:41-44): pos[n] (0xffffffff = kNoDiag), inv[n]; either may be NULL. */
int mpkg_jacobi_get(mpkg_jacobi_t J, uint32_t* pos, double* inv);
int mpkg_jacobi_destroy(mpkg_jacobi_t J);
/* jacobi.hpp:155-174 jacobi_apply: z = M^{-1} v. */
int mpkg_jacobi_apply(mpkg_ctx_t ctx, mpkg_jacobi_t J, mpkg_csr_t A, const double* v, double* z);
int mpkg_jacobi_apply_dev(mpkg_ctx_t ctx, mpkg_jacobi_t J, mpkg_csr_t A, const double* d_v,
                          double* d_z);
/* jacobi.hpp:177-192 jacobi_op: y = A (M^{-1} v). */
int mpkg_jacobi_op(mpkg_ctx_t ctx, mpkg_jacobi_t J, mpkg_csr_t A, const double* v, double* y);
int mpkg_jacobi_op_dev(mpkg_ctx_t ctx, mpkg_jacobi_t J, mpkg_csr_t A, const double* d_v,
                       double* d_y);
/* jacobi.hpp:196-209 jacobi_op_blocked: the plan must match A_perm and carry
 * sub_powers == (sweeps == 1 ? 1 : sweeps + 1) (EINVAL otherwise). */
int mpkg_jacobi_op_blocked(mpkg_ctx_t ctx, mpkg_jacobi_t J, mpkg_plan_t P, mpkg_csr_t A_perm,
                           const double* v, double* y);
int mpkg_jacobi_op_blocked_dev(mpkg_ctx_t ctx, mpkg_jacobi_t J, mpkg_plan_t P,
                               mpkg_csr_t A_perm, const double* d_v, double* d_y);
/* sstep.hpp:356-385 sstep_generate_block, Jacobi case: block slice 0 holds the start vector on
 * entry; slices 1..s receive w_p = (A M^{-1} - a_p) w_{p-1} (+ b2_p w_{p-2}), b2_p = im_p^2 for
 * the second member of a conjugate pair.  P may be NULL (sequential form); otherwise it must
 * match A, carry the chain's sub_powers and a power budget >= s (execute.hpp:81-83). */
int mpkg_sstep_jacobi(mpkg_ctx_t ctx, mpkg_jacobi_t J, mpkg_plan_t P, mpkg_csr_t A,
                      const double* re, const double* im, int s, double* block,
                      uint64_t block_rows, uint64_t block_slices);
int mpkg_sstep_jacobi_dev(mpkg_ctx_t ctx, mpkg_jacobi_t J, mpkg_plan_t P, mpkg_csr_t A,
                          const double* re, const double* im, int s, double* d_block,
                          uint64_t block_rows, uint64_t block_slices);

/* ---- GS2 (K-sweep two-stage Gauss-Seidel) chains (gs2.hpp; sstep.hpp:160-198) ---------------
 * direction: 0 forward (strict lower part), 1 backward (strict upper part).  P may be NULL (the
 * sequential form) or must match A, carry sub_powers == gamma + 2 and a power budget >= sweeps
 * (the cache-blocked twins, bitwise equal to the sequential form). */
int mpkg_gs2_setup(mpkg_ctx_t ctx, mpkg_csr_t A, int gamma, int sweeps, int direction,
                   mpkg_gs2_t* out);                                       /* gs2.hpp:55-62 */
int mpkg_gs2_info(mpkg_gs2_t G, uint32_t* n, int* gamma, int* sweeps, int* direction);
int mpkg_gs2_get(mpkg_gs2_t G, uint32_t* pos, double* inv);
int mpkg_gs2_destroy(mpkg_gs2_t G);
/* gs2.hpp:200-204 gs2_smooth (z in/out) / 207-212 gs2_apply (zero guess) / 215-220
 * gs2_smooth_residual (z in/out, r = v - A z) / 223-228 gs2_op (y = A M^{-1} v) and their
 * *_blocked twins (gs2.hpp:233-275) when P != NULL.  Host pointers. */
int mpkg_gs2_smooth(mpkg_ctx_t ctx, mpkg_gs2_t G, mpkg_plan_t P, mpkg_csr_t A, const double* v,
                    double* z);
int mpkg_gs2_apply(mpkg_ctx_t ctx, mpkg_gs2_t G, mpkg_plan_t P, mpkg_csr_t A, const double* v,
                   double* z);
int mpkg_gs2_smooth_residual(mpkg_ctx_t ctx, mpkg_gs2_t G, mpkg_plan_t P, mpkg_csr_t A,
                             const double* v, double* z, double* r);
int mpkg_gs2_op(mpkg_ctx_t ctx, mpkg_gs2_t G, mpkg_plan_t P, mpkg_csr_t A, const double* v,
                double* y);
/* Device-pointer form of the four: mode 0 smooth, 1 apply, 2 smooth_residual, 3 op; d_z is
 * in/out (ignored on input for apply / op), d_out receives r or y. */
int mpkg_gs2_run_dev(mpkg_ctx_t ctx, mpkg_gs2_t G, mpkg_plan_t P, mpkg_csr_t A, int mode,
                     const double* d_v, double* d_z, double* d_out);
/* sstep.hpp:356-398 sstep_generate_block, GS2 case (P: sub_powers == gamma + 2, power budget
 * >= s * sweeps). */
int mpkg_sstep_gs2(mpkg_ctx_t ctx, mpkg_gs2_t G, mpkg_plan_t P, mpkg_csr_t A, const double* re,
                   const double* im, int s, double* block, uint64_t block_rows,
                   uint64_t block_slices);
int mpkg_sstep_gs2_dev(mpkg_ctx_t ctx, mpkg_gs2_t G, mpkg_plan_t P, mpkg_csr_t A,
                       const double* re, const double* im, int s, double* d_block,
                       uint64_t block_rows, uint64_t block_slices);

/* ---- product-form GMRES polynomial (poly.hpp:146-281) ------------------
 * z = p(A M^{-1}) v for the given roots (re, im: degree entries, Leja-ordered by the caller,
 * conjugate pairs adjacent); M^{-1} = J (Jacobi), G (GS2, one sweep) or none (both NULL).  P may
 * be NULL (sequential form) or carry sub_powers == the inner chain's stages + terminal
 * (poly.hpp:132-144); roots beyond its power budget are processed in further passes, bitwise
 * equal.  The roots themselves come from an Arnoldi/harmonic-Ritz setup that needs Eigen in the
 * reference (poly_setup_gmres) and is not part of this library. */
int mpkg_poly_apply(mpkg_ctx_t ctx, mpkg_csr_t A, mpkg_jacobi_t J, mpkg_gs2_t G, const double* re,
                    const double* im, int degree, mpkg_plan_t P, const double* v, double* z);
int mpkg_poly_apply_dev(mpkg_ctx_t ctx, mpkg_csr_t A, mpkg_jacobi_t J, mpkg_gs2_t G,
                        const double* re, const double* im, int degree, mpkg_plan_t P,
                        const double* d_v, double* d_z);

/* ---- multi-GPU level-range shards (csrc/dist.cu) -----------------------------
 * No reference counterpart (the reference is single-node OpenMP); this is the C++ caller's view of
 * multi.py.  Rank r owns the BFS levels [bounds[r], bounds[r+1]) of A_perm (balanced by nnz) and
 * holds p ghost levels on each side; one halo exchange of x per MPK call, then the local MPK of its
 * block A_perm[g0:g1, g0:g1]; own rows are bit-identical to the single-GPU result.
 *
 * Pure host functions (no GPU, no NCCL): nnz_before[L] = nonzeros in levels < L (n_levels+1
 * entries); bounds has world+1 entries.  own / local: [first, end) global rows; send / recv:
 * 2*world entries, the row range this rank sends to / receives from each rank (empty: lo == hi). */
int mpkg_dist_partition(const uint32_t* level_ptr, uint32_t n_levels, const uint64_t* nnz_before,
                        int world, uint32_t* bounds);
int mpkg_dist_halo(const uint32_t* level_ptr, uint32_t n_levels, const uint32_t* bounds, int world,
                   int rank, int p, uint32_t* own, uint32_t* local, uint32_t* send, uint32_t* recv);
/* NCCL communicator (libnccl.so.2 loaded at run time; MPKG_EINTERNAL if absent).  The 128-byte id
 * comes from mpkg_dist_unique_id on one rank and reaches the others by the caller's bootstrap. */
int mpkg_dist_unique_id(void* id128);
int mpkg_dist_create(mpkg_ctx_t ctx, const void* id128, int world, int rank, mpkg_dist_t* out);
int mpkg_dist_destroy(mpkg_dist_t D);
/* Broadcast of a host buffer from root (e.g. level_ptr and bounds before mpkg_dist_set_plan). */
int mpkg_dist_bcast_host(mpkg_dist_t D, void* buf, uint64_t bytes, int root);
/* The rank's halo plan for p powers; preallocates the local x buffer. */
int mpkg_dist_set_plan(mpkg_dist_t D, const uint32_t* level_ptr, uint32_t n_levels,
                       const uint32_t* bounds, int p);
int mpkg_dist_info(mpkg_dist_t D, uint32_t* own, uint32_t* local, uint64_t* send_bytes,
                   uint64_t* recv_bytes);
/* One-time setup from a root that holds A_perm (and a device vector in A_perm order): every rank
 * receives its local block / its own rows. */
int mpkg_dist_scatter_blocks(mpkg_dist_t D, int root, mpkg_csr_t A_perm, mpkg_csr_t* A_local);
int mpkg_dist_scatter_rows(mpkg_dist_t D, int root, const double* d_full, double* d_own);
/* Per step: the halo exchange (grouped ncclSend / ncclRecv on the context's stream into the
 * preallocated local x, whose device pointer is returned), and exchange + local mpkg_mpk_dev of
 * the block (block_rows >= local rows; the own rows sit at own[0] - local[0]). */
int mpkg_dist_exchange(mpkg_dist_t D, const double* d_x_own, double** d_x_local);
int mpkg_dist_mpk(mpkg_dist_t D, mpkg_plan_t P, mpkg_csr_t A_local, const double* d_x_own, int p,
                  double* d_block, uint64_t block_rows, uint64_t block_slices);

/* ---- block orthogonalisation (ortho.hpp) --------------------------------
 * Blocks are column-major with leading dimension `rows` (consecutive VectorBlock slices).  The
 * plain names take host pointers (synchronous, as the reference); _dev take device pointers and
 * run on the context's stream.
 *
 * ortho.hpp:46-63 block_dots: C (qcols x vcols, column-major) = Q^T V.  MPKG_MODE_BITWISE: every
 * entry is the reference's serial ascending-row sum (bit-identical); MPKG_MODE_FAST: fp64 tensor
 * cores with a fixed-order reduction (deterministic, roundoff-level difference). */
int mpkg_block_dots(mpkg_ctx_t ctx, const double* q, const double* v, uint64_t rows, uint32_t qcols,
                    uint32_t vcols, double* c);
int mpkg_block_dots_dev(mpkg_ctx_t ctx, const double* d_q, const double* d_v, uint64_t rows,
                        uint32_t qcols, uint32_t vcols, double* d_c);
/* ortho.hpp:67-92 block_update: V <- V - Q C, every element updated in ascending k with mul then
 * sub (bit-identical in both modes). */
int mpkg_block_update(mpkg_ctx_t ctx, const double* q, const double* c, uint64_t rows,
                      uint32_t qcols, uint32_t vcols, double* v);
int mpkg_block_update_dev(mpkg_ctx_t ctx, const double* d_q, const double* d_c, uint64_t rows,
                          uint32_t qcols, uint32_t vcols, double* d_v);
/* ortho.hpp:97-117 icgs_block_orthogonalize: `sweeps` rounds of dots + update; coeff
 * (qcols x vcols, column-major) receives the accumulated coefficients.  qcols == 0 or vcols == 0
 * returns at once (nothing written); otherwise MPKG_EINVAL if sweeps < 1. */
int mpkg_icgs_block_orthogonalize(mpkg_ctx_t ctx, const double* q, uint64_t rows, uint32_t qcols,
                                  double* v, uint32_t vcols, int sweeps, double* coeff);
int mpkg_icgs_block_orthogonalize_dev(mpkg_ctx_t ctx, const double* d_q, uint64_t rows,
                                      uint32_t qcols, double* d_v, uint32_t vcols, int sweeps,
                                      double* d_coeff);
/* ortho.hpp:136-229 tsqr: V (rows x cols) is overwritten with Q (orthonormal columns), r
 * (cols x cols, column-major) with the upper-triangular R (non-negative diagonal, zero below),
 * Q R = V_in.  Panels are chosen by the library (shared-memory sized); the factorisation is
 * unique for a full-rank block, so it agrees with the reference's panel tree to roundoff.
 * MPKG_EINVAL if rows < cols or cols > 64; cols == 0 returns at once. */
int mpkg_tsqr(mpkg_ctx_t ctx, double* v, uint64_t rows, uint32_t cols, double* r);
int mpkg_tsqr_dev(mpkg_ctx_t ctx, double* d_v, uint64_t rows, uint32_t cols, double* d_r);
/* sstep.hpp:539-545: icgs_block_orthogonalize(q, ..., v, ..., sweeps) then tsqr(v, ..., r) in one
 * call; for s-step blocks (vcols <= 8, qcols <= 64) ICGS's last update runs inside TSQR's first
 * factor kernel and the updated block is never stored.  Every output is bit-identical to the two
 * calls in sequence.  Same arguments and errors as those two. */
int mpkg_ortho_block(mpkg_ctx_t ctx, const double* q, uint64_t rows, uint32_t qcols, double* v, uint32_t vcols,
                     int sweeps, double* coeff, double* r);
int mpkg_ortho_block_dev(mpkg_ctx_t ctx, const double* d_q, uint64_t rows, uint32_t qcols, double* d_v,
                         uint32_t vcols, int sweeps, double* d_coeff, double* d_r);

/* ---- host-side matrix generators (harness inputs; generators.hpp + SURVEY §7 step 1) ------- */
/* kinds: 1 poisson1d(a) 2 poisson2d(a,b) 3 poisson3d(a,b,c) [generators.hpp:35-89]
 *        4 random_csr(a=n, b=nnz_per_row, seed) 5 random_spd(a, b, seed) [generators.hpp:96-146]
 *        6 stencil27(a,b,c; diag 26, off -1) [config C4]
 *        7 stencil27 with off-diagonal -U[0.9,1.1] (seeded), then (A+A^T)/2 [config C2, before
 *          the scramble]
 *        8 rmat(scale=a, edge_factor=b, seed) with a,b,c,d = .57,.19,.19,.05, symmetrised,
 *          self loops / duplicates removed, off-diagonal -U[0.1,1], diag 1+sum|off| [config C3] */
int mpkg_gen(int kind, uint32_t a, uint32_t b, uint32_t c, uint64_t seed, mpkg_host_csr_t* out);
/* Seeded symmetric scramble B = P A P^T (same semantics as permute) with a Fisher-Yates
 * permutation drawn from mt19937_64(seed); perm_out (n entries, may be NULL) receives it. */
int mpkg_host_csr_scramble(mpkg_host_csr_t A, uint64_t seed, uint32_t* perm_out,
                           mpkg_host_csr_t* out);
int mpkg_host_csr_info(mpkg_host_csr_t h, uint32_t* n_rows, uint32_t* n_cols, uint64_t* nnz);
/* Borrowed pointers into the handle's arrays (valid until mpkg_host_csr_destroy). */
int mpkg_host_csr_arrays(mpkg_host_csr_t h, uint32_t** row_ptr, uint32_t** col_idx,
                         double** values);
int mpkg_host_csr_destroy(mpkg_host_csr_t h);
/* x_i ~ U[-1,1] from std::mt19937_64(seed) (acceptance.cpp:84-90 random_vector). */
int mpkg_random_vector(uint64_t n, uint64_t seed, double* out);

#ifdef __cplusplus
}
#endif

#endif /* MPKG_H */
