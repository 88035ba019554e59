// TEST INFRASTRUCTURE ONLY — extern "C" shim over the reference's own hot-path headers.
//
// Compiled by oracle/Makefile *in place* against /root/reference/proj/include (read-only, never
// copied) with the reference's flags (proj/CMakeLists.txt:8-21: -O3 -DNDEBUG, OpenMP, no -march),
// producing oracle/_ref/libmpkref.so.  Used (1) to pin the C restatement in oracle/oracle.c,
// (2) by tests/golden/make_golden.py to generate the committed fixtures, and (3) as bench.py's
// `--impl reference` / cpu_baseline arm (the reference's OpenMP CPU path, timed on host cores).
// The product library never links it.
#include <cstdint>
#include <cstring>
#include <complex>
#include <exception>
#include <random>
#include <stdexcept>
#include <vector>

#include "mpk/csr.hpp"
#include "mpk/execute.hpp"
#include "mpk/generators.hpp"
#include "mpk/gs2.hpp"
#include "mpk/jacobi.hpp"
#include "mpk/matrix_market.hpp"
#include "mpk/levels.hpp"
#include "mpk/mpk.hpp"
#include "mpk/plan.hpp"
#include "mpk/vector_block.hpp"

using mpk::index_t;

namespace {

thread_local std::string g_err;

mpk::CsrMatrix wrap(uint32_t n, const uint32_t* rp, const uint32_t* ci, const double* v) {
    mpk::CsrMatrix A;
    A.n_rows = n;
    A.n_cols = n;
    A.row_ptr.assign(rp, rp + n + 1);
    A.col_idx.assign(ci, ci + rp[n]);
    A.values.assign(v, v + rp[n]);
    return A;
}

mpk::ExecutionPlan plan_from(uint32_t n, const uint32_t* group_rows, uint32_t ng, int p_m) {
    mpk::ExecutionPlan plan;
    plan.p_m = p_m;
    plan.n_rows = n;
    plan.group_rows.assign(group_rows, group_rows + ng + 1);
    plan.group_level_ptr.assign(ng + 1, 0);
    plan.group_footprint.assign(ng, 0);
    return plan;
}

template <class F>
int guard(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const std::out_of_range& e) {
        g_err = e.what();
        return 2;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 3;
    }
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// ---- generators (proj/include/mpk/generators.hpp) -------------------------------------------
void* ref_gen(int kind, uint32_t a, uint32_t b, uint32_t c, uint64_t seed) {
    auto* m = new mpk::CsrMatrix();
    int rc = guard([&] {
        switch (kind) {
            case 1: *m = mpk::poisson1d(a); break;
            case 2: *m = mpk::poisson2d(a, b); break;
            case 3: *m = mpk::poisson3d(a, b, c); break;
            case 4: *m = mpk::random_csr(a, b, seed); break;
            case 5: *m = mpk::random_spd(a, b, seed); break;
            default: throw std::invalid_argument("ref_gen: unknown kind");
        }
    });
    if (rc) {
        delete m;
        return nullptr;
    }
    return m;
}
void ref_csr_info(void* h, uint32_t* n, uint32_t* nnz) {
    auto* m = static_cast<mpk::CsrMatrix*>(h);
    *n = m->n_rows;
    *nnz = m->nnz();
}
void ref_csr_copy(void* h, uint32_t* rp, uint32_t* ci, double* v) {
    auto* m = static_cast<mpk::CsrMatrix*>(h);
    std::memcpy(rp, m->row_ptr.data(), sizeof(uint32_t) * m->row_ptr.size());
    std::memcpy(ci, m->col_idx.data(), sizeof(uint32_t) * m->col_idx.size());
    std::memcpy(v, m->values.data(), sizeof(double) * m->values.size());
}
void ref_csr_free(void* h) { delete static_cast<mpk::CsrMatrix*>(h); }

// acceptance.cpp:84-90 random_vector
void ref_random_vector(uint64_t n, uint64_t seed, double* out) {
    std::mt19937_64 rng(seed);
    std::uniform_real_distribution<double> u(-1.0, 1.0);
    for (uint64_t i = 0; i < n; ++i) out[i] = u(rng);
}

// ---- level engine -------------------------------------------------------------------------------
int ref_build_levels(uint32_t n, const uint32_t* rp, const uint32_t* ci, const double* v,
                     uint32_t* levels, uint32_t* perm, uint32_t* inv_perm, uint32_t* level_ptr,
                     uint32_t* n_levels) {
    return guard([&] {
        const auto A = wrap(n, rp, ci, v);
        const auto ls = mpk::build_levels(A);
        std::memcpy(levels, ls.levels.data(), sizeof(uint32_t) * n);
        std::memcpy(perm, ls.perm.data(), sizeof(uint32_t) * n);
        std::memcpy(inv_perm, ls.inv_perm.data(), sizeof(uint32_t) * n);
        std::memcpy(level_ptr, ls.level_ptr.data(), sizeof(uint32_t) * ls.level_ptr.size());
        *n_levels = ls.n_levels();
    });
}

// Handle forms for full-size inputs (C5: 11.8 GB of CSR): no second host copy per call.
int ref_build_levels_h(void* h, uint32_t* levels, uint32_t* perm, uint32_t* inv_perm,
                       uint32_t* level_ptr, uint32_t* n_levels) {
    return guard([&] {
        const auto& A = *static_cast<mpk::CsrMatrix*>(h);
        const auto ls = mpk::build_levels(A);
        const std::size_t n = A.n_rows;
        std::memcpy(levels, ls.levels.data(), sizeof(uint32_t) * n);
        std::memcpy(perm, ls.perm.data(), sizeof(uint32_t) * n);
        std::memcpy(inv_perm, ls.inv_perm.data(), sizeof(uint32_t) * n);
        std::memcpy(level_ptr, ls.level_ptr.data(), sizeof(uint32_t) * ls.level_ptr.size());
        *n_levels = ls.n_levels();
    });
}
void* ref_permute_h(void* h, const uint32_t* perm) {
    void* out = nullptr;
    guard([&] {
        const auto& A = *static_cast<mpk::CsrMatrix*>(h);
        out = new mpk::CsrMatrix(mpk::permute(A, std::vector<index_t>(perm, perm + A.n_rows)));
    });
    return out;
}
// Borrowed views of a handle's arrays (valid until ref_csr_free).
void ref_csr_views(void* h, uint32_t** rp, uint32_t** ci, double** v) {
    auto* m = static_cast<mpk::CsrMatrix*>(h);
    *rp = m->row_ptr.data();
    *ci = m->col_idx.data();
    *v = m->values.data();
}

int ref_permute(uint32_t n, const uint32_t* rp, const uint32_t* ci, const double* v,
                const uint32_t* perm, uint32_t* orp, uint32_t* oci, double* ov) {
    return guard([&] {
        const auto A = wrap(n, rp, ci, v);
        const auto B = mpk::permute(A, std::vector<index_t>(perm, perm + n));
        std::memcpy(orp, B.row_ptr.data(), sizeof(uint32_t) * (n + 1));
        std::memcpy(oci, B.col_idx.data(), sizeof(uint32_t) * B.nnz());
        std::memcpy(ov, B.values.data(), sizeof(double) * B.nnz());
    });
}

int ref_validate_levels(uint32_t n, const uint32_t* rp, const uint32_t* ci, const double* v,
                        const uint32_t* levels, const uint32_t* perm, const uint32_t* inv_perm,
                        const uint32_t* level_ptr, uint32_t n_levels) {
    int ok = 0;
    guard([&] {
        const auto A = wrap(n, rp, ci, v);
        mpk::LevelStructure ls;
        ls.n_rows = n;
        ls.levels.assign(levels, levels + n);
        ls.perm.assign(perm, perm + n);
        ls.inv_perm.assign(inv_perm, inv_perm + n);
        ls.level_ptr.assign(level_ptr, level_ptr + n_levels + 1);
        ok = mpk::validate_levels(A, ls) ? 1 : 0;
    });
    return ok;
}

int ref_group_levels(uint32_t n, const uint32_t* rp, const uint32_t* ci, const double* v,
                     const uint32_t* level_ptr, uint32_t n_levels, uint64_t cache_bytes, int p_m,
                     uint32_t* group_rows, uint32_t* group_level_ptr, uint64_t* group_fp,
                     uint32_t* n_groups, uint64_t* target) {
    return guard([&] {
        const auto A = wrap(n, rp, ci, v);
        mpk::LevelStructure ls;
        ls.n_rows = n;
        ls.level_ptr.assign(level_ptr, level_ptr + n_levels + 1);
        const auto plan = mpk::group_levels(ls, A, cache_bytes, p_m);
        std::memcpy(group_rows, plan.group_rows.data(), sizeof(uint32_t) * plan.group_rows.size());
        std::memcpy(group_level_ptr, plan.group_level_ptr.data(),
                    sizeof(uint32_t) * plan.group_level_ptr.size());
        for (std::size_t g = 0; g < plan.group_footprint.size(); ++g)
            group_fp[g] = plan.group_footprint[g];
        *n_groups = plan.n_groups();
        *target = plan.target_bytes;
    });
}

uint32_t ref_greedy_group(const uint64_t* fp, uint32_t nl, uint64_t target, uint32_t* bounds) {
    std::vector<std::size_t> f(fp, fp + nl);
    const auto b = mpk::greedy_group(f, target);
    std::memcpy(bounds, b.data(), sizeof(uint32_t) * b.size());
    return static_cast<uint32_t>(b.size());
}

uint64_t ref_wavefront_schedule(uint32_t ng, int stages, uint32_t* group, int* stage) {
    const auto order = mpk::wavefront_schedule(ng, stages);
    for (std::size_t i = 0; i < order.size(); ++i) {
        group[i] = order[i].group;
        stage[i] = order[i].stage;
    }
    return order.size();
}

// ---- power kernels (proj/include/mpk/mpk.hpp) ---------------------------------------------------
// The CSR is wrapped once per handle so that timed calls measure only the kernel.
void* ref_csr_wrap(uint32_t n, const uint32_t* rp, const uint32_t* ci, const double* v) {
    return new mpk::CsrMatrix(wrap(n, rp, ci, v));
}

int ref_baseline_mpk_h(void* h, const double* x, int p_m, double* block, int threads) {
    return guard([&] {
        const auto& A = *static_cast<mpk::CsrMatrix*>(h);
        mpk::VectorBlock blk(A.n_rows, static_cast<std::size_t>(p_m) + 1);
        mpk::baseline_mpk(A, std::vector<double>(x, x + A.n_rows), p_m, blk, threads);
        std::memcpy(block, blk.data.data(), sizeof(double) * blk.data.size());
    });
}

int ref_mpk_h(void* h, const uint32_t* group_rows, uint32_t ng, int plan_p_m, const double* x,
              int p_m, double* block, int threads) {
    return guard([&] {
        const auto& A = *static_cast<mpk::CsrMatrix*>(h);
        const auto plan = plan_from(A.n_rows, group_rows, ng, plan_p_m);
        mpk::VectorBlock blk(A.n_rows, static_cast<std::size_t>(p_m) + 1);
        mpk::mpk(plan, A, std::vector<double>(x, x + A.n_rows), p_m, blk, threads);
        std::memcpy(block, blk.data.data(), sizeof(double) * blk.data.size());
    });
}

// Timed variants keep a caller-owned VectorBlock so the timing excludes allocation/copies.
void* ref_block_new(uint64_t rows, uint64_t slices) { return new mpk::VectorBlock(rows, slices); }
void ref_block_free(void* b) { delete static_cast<mpk::VectorBlock*>(b); }
double* ref_block_data(void* b) { return static_cast<mpk::VectorBlock*>(b)->data.data(); }
void* ref_vec_new(const double* x, uint64_t n) { return new std::vector<double>(x, x + n); }
void ref_vec_free(void* v) { delete static_cast<std::vector<double>*>(v); }
void* ref_plan_new(uint32_t n, const uint32_t* group_rows, uint32_t ng, int p_m) {
    return new mpk::ExecutionPlan(plan_from(n, group_rows, ng, p_m));
}
void ref_plan_free(void* p) { delete static_cast<mpk::ExecutionPlan*>(p); }

int ref_baseline_mpk_t(void* h, void* x, int p_m, void* blk, int threads) {
    return guard([&] {
        mpk::baseline_mpk(*static_cast<mpk::CsrMatrix*>(h), *static_cast<std::vector<double>*>(x),
                          p_m, *static_cast<mpk::VectorBlock*>(blk), threads);
    });
}
int ref_mpk_t(void* plan, void* h, void* x, int p_m, void* blk, int threads) {
    return guard([&] {
        mpk::mpk(*static_cast<mpk::ExecutionPlan*>(plan), *static_cast<mpk::CsrMatrix*>(h),
                 *static_cast<std::vector<double>*>(x), p_m, *static_cast<mpk::VectorBlock*>(blk),
                 threads);
    });
}

static std::vector<std::complex<double>> shifts_from(const double* re, const double* im, int ns) {
    std::vector<std::complex<double>> s(ns);
    for (int i = 0; i < ns; ++i) s[i] = {re[i], im[i]};
    return s;
}

int ref_baseline_mpk_shifted_h(void* h, const double* x, const double* re, const double* im,
                               int ns, double* block, int threads) {
    return guard([&] {
        const auto& A = *static_cast<mpk::CsrMatrix*>(h);
        mpk::VectorBlock blk(A.n_rows, static_cast<std::size_t>(ns) + 1);
        mpk::baseline_mpk_shifted(A, std::vector<double>(x, x + A.n_rows),
                                  shifts_from(re, im, ns), blk, threads);
        std::memcpy(block, blk.data.data(), sizeof(double) * blk.data.size());
    });
}

int ref_mpk_shifted_h(void* h, const uint32_t* group_rows, uint32_t ng, int plan_p_m,
                      const double* x, const double* re, const double* im, int ns, double* block,
                      int threads) {
    return guard([&] {
        const auto& A = *static_cast<mpk::CsrMatrix*>(h);
        const auto plan = plan_from(A.n_rows, group_rows, ng, plan_p_m);
        mpk::VectorBlock blk(A.n_rows, static_cast<std::size_t>(ns) + 1);
        mpk::mpk_shifted(plan, A, std::vector<double>(x, x + A.n_rows), shifts_from(re, im, ns),
                         blk, threads);
        std::memcpy(block, blk.data.data(), sizeof(double) * blk.data.size());
    });
}

// Timed shifted variants (bench --impl reference, C4): the shift list, the plan, x and the block
// are built once outside the timed loop, as ref_mpk_t does for the plain MPK.
void* ref_shifts_new(const double* re, const double* im, int ns) {
    return new std::vector<std::complex<double>>(shifts_from(re, im, ns));
}
void ref_shifts_free(void* s) { delete static_cast<std::vector<std::complex<double>>*>(s); }
int ref_baseline_mpk_shifted_t(void* h, void* x, void* shifts, void* blk, int threads) {
    return guard([&] {
        mpk::baseline_mpk_shifted(*static_cast<mpk::CsrMatrix*>(h), *static_cast<std::vector<double>*>(x),
                                  *static_cast<std::vector<std::complex<double>>*>(shifts),
                                  *static_cast<mpk::VectorBlock*>(blk), threads);
    });
}
int ref_mpk_shifted_t(void* plan, void* h, void* x, void* shifts, void* blk, int threads) {
    return guard([&] {
        mpk::mpk_shifted(*static_cast<mpk::ExecutionPlan*>(plan), *static_cast<mpk::CsrMatrix*>(h),
                         *static_cast<std::vector<double>*>(x),
                         *static_cast<std::vector<std::complex<double>>*>(shifts),
                         *static_cast<mpk::VectorBlock*>(blk), threads);
    });
}

int ref_check_shift_chain(const double* re, const double* im, int ns) {
    return guard([&] { mpk::check_shift_chain(shifts_from(re, im, ns), "ref"); });
}

int ref_tune_select(const double* table, int p_lo, int p_hi) {
    const auto r = mpk::tune_p(p_lo, p_hi, [&](int p) { return table[p - p_lo]; });
    return r.p_opt;
}

int ref_resolve_threads(int requested) { return mpk::resolve_threads(requested); }

// jacobi.hpp: setup, preconditioner apply, A M^{-1} v sequential and
// cache-blocked (plan with sub_powers = JacobiOpChain::stages(sweeps)).
int ref_jacobi_setup(uint32_t n, const uint32_t* rp, const uint32_t* ci, const double* v,
                     int sweeps, uint32_t* pos, double* inv) {
    return guard([&] {
        const auto A = wrap(n, rp, ci, v);
        const mpk::JacobiPrecon P = mpk::jacobi_setup(A, sweeps);
        std::memcpy(pos, P.diag.pos.data(), sizeof(uint32_t) * n);
        std::memcpy(inv, P.diag.inv.data(), sizeof(double) * n);
    });
}

int ref_jacobi_apply(uint32_t n, const uint32_t* rp, const uint32_t* ci, const double* v,
                     int sweeps, const double* x, double* z) {
    return guard([&] {
        const auto A = wrap(n, rp, ci, v);
        const mpk::JacobiPrecon P = mpk::jacobi_setup(A, sweeps);
        std::vector<double> out;
        mpk::jacobi_apply(P, A, std::vector<double>(x, x + n), out, 1);
        std::memcpy(z, out.data(), sizeof(double) * n);
    });
}

int ref_jacobi_op(uint32_t n, const uint32_t* rp, const uint32_t* ci, const double* v,
                  int sweeps, const double* x, double* y) {
    return guard([&] {
        const auto A = wrap(n, rp, ci, v);
        const mpk::JacobiPrecon P = mpk::jacobi_setup(A, sweeps);
        std::vector<double> out;
        mpk::jacobi_op(P, A, std::vector<double>(x, x + n), out, 1);
        std::memcpy(y, out.data(), sizeof(double) * n);
    });
}

int ref_jacobi_op_blocked(uint32_t n, const uint32_t* rp, const uint32_t* ci, const double* v,
                          int sweeps, const uint32_t* group_rows, uint32_t ng, const double* x,
                          double* y, int threads) {
    return guard([&] {
        const auto A = wrap(n, rp, ci, v);
        const mpk::JacobiPrecon P = mpk::jacobi_setup(A, sweeps);
        auto plan = plan_from(n, group_rows, ng, 1);
        plan.sub_powers = mpk::detail::JacobiOpChain::stages(sweeps);
        std::vector<double> out;
        mpk::jacobi_op_blocked(P, A, plan, std::vector<double>(x, x + n), out, threads);
        std::memcpy(y, out.data(), sizeof(double) * n);
    });
}

// gs2.hpp: mode 0 smooth (z in/out), 1 apply (zero guess), 2 smooth_residual, 3 op; plan
// (group_rows) NULL = sequential form, otherwise the blocked twin (sub_powers = gamma + 2).
int ref_gs2(uint32_t n, const uint32_t* rp, const uint32_t* ci, const double* v, int gamma,
            int sweeps, int forward, int mode, const uint32_t* group_rows, uint32_t ng, int plan_p_m,
            const double* vin, double* z_io, double* out, int threads) {
    return guard([&] {
        const auto A = wrap(n, rp, ci, v);
        const mpk::Gs2Precon P = mpk::gs2_setup(A, gamma, sweeps,
                                                forward ? mpk::SweepDirection::forward
                                                        : mpk::SweepDirection::backward);
        const std::vector<double> vv(vin, vin + n);
        std::vector<double> z(z_io, z_io + n), o;
        mpk::ExecutionPlan plan;
        if (group_rows) {
            plan = plan_from(n, group_rows, ng, plan_p_m);
            plan.sub_powers = gamma + 2;
        }
        switch (mode) {
            case 0: group_rows ? mpk::gs2_smooth_blocked(P, A, plan, vv, z, threads) : mpk::gs2_smooth(P, A, vv, z, threads); break;
            case 1: group_rows ? mpk::gs2_apply_blocked(P, A, plan, vv, z, threads) : mpk::gs2_apply(P, A, vv, z, threads); break;
            case 2: group_rows ? mpk::gs2_smooth_residual_blocked(P, A, plan, vv, z, o, threads) : mpk::gs2_smooth_residual(P, A, vv, z, o, threads); break;
            default: group_rows ? mpk::gs2_op_blocked(P, A, plan, vv, o, threads) : mpk::gs2_op(P, A, vv, o, threads); break;
        }
        std::memcpy(z_io, z.data(), sizeof(double) * n);
        if (out && !o.empty()) std::memcpy(out, o.data(), sizeof(double) * n);
    });
}

// csr.hpp:72-110 from_coo and matrix_market.hpp read_matrix_market; results through ref_csr_*.
void* ref_from_coo(uint32_t n_rows, uint32_t n_cols, uint64_t nnz, const uint32_t* rows,
                   const uint32_t* cols, const double* vals) {
    void* out = nullptr;
    const int rc = guard([&] {
        std::vector<mpk::Triplet> t(nnz);
        for (uint64_t i = 0; i < nnz; ++i) t[i] = {rows[i], cols[i], vals[i]};
        out = new mpk::CsrMatrix(mpk::from_coo(n_rows, n_cols, std::move(t)));
    });
    return rc ? nullptr : out;
}

void ref_csr_shape(void* h, uint32_t* n_rows, uint32_t* n_cols) {
    auto* m = static_cast<mpk::CsrMatrix*>(h);
    *n_rows = m->n_rows;
    *n_cols = m->n_cols;
}

void* ref_read_matrix_market(const char* path) {
    void* out = nullptr;
    const int rc = guard([&] { out = new mpk::CsrMatrix(mpk::read_matrix_market(path)); });
    return rc ? nullptr : out;
}

}  // extern "C"
