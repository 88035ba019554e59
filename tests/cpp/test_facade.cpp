// The reference's hot-path tests (proj/tests/test_levels.cpp, test_mpk.cpp, acceptance.cpp
// C1-C3) restated against the C++ facade include/mpkg.hpp, with a minimal assertion harness
// (GTest is not available here).  A reference call site switches with `namespace mpk = mpkg;`
// -- this file does exactly that, so the test bodies read like the reference's own.
// Built by __graft_entry__.build(); run by tests/test_gpu_facade.py on the GPU.
#include <array>
#include <cmath>
#include <complex>
#include <cstdio>
#include <cstring>
#include <random>
#include <vector>

#include "mpkg.hpp"

namespace mpk = mpkg;
using mpk::CsrMatrix;
using mpk::ExecutionPlan;
using mpk::index_t;
using mpk::LevelStructure;
using mpk::VectorBlock;
using cplx = std::complex<double>;

static int g_fail = 0, g_checks = 0;
#define EXPECT(c)                                                                  \
    do {                                                                           \
        ++g_checks;                                                                \
        if (!(c)) {                                                                \
            ++g_fail;                                                              \
            std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #c);               \
        }                                                                          \
    } while (0)
#define EXPECT_THROW(stmt, E)                                                      \
    do {                                                                           \
        bool thrown_ = false;                                                      \
        try {                                                                      \
            stmt;                                                                  \
        } catch (const E&) {                                                       \
            thrown_ = true;                                                        \
        }                                                                          \
        EXPECT(thrown_);                                                           \
    } while (0)

static bool bitwise_equal(const std::vector<double>& a, const std::vector<double>& b) {
    return a.size() == b.size() && std::memcmp(a.data(), b.data(), a.size() * 8) == 0;
}

static std::vector<double> random_vector(std::size_t n, std::uint64_t seed) {
    std::mt19937_64 rng(seed);
    std::uniform_real_distribution<double> u(-1.0, 1.0);
    std::vector<double> v(n);
    for (double& x : v) x = u(rng);
    return v;
}

static ExecutionPlan synthetic_plan(index_t n_groups, int p_m, int sub_powers = 1) {
    ExecutionPlan plan;
    plan.p_m = p_m;
    plan.sub_powers = sub_powers;
    plan.n_rows = n_groups;
    plan.group_rows.resize(n_groups + 1);
    for (index_t g = 0; g <= n_groups; ++g) plan.group_rows[g] = g;
    plan.group_level_ptr = plan.group_rows;
    plan.group_footprint.assign(n_groups, 0);
    return plan;
}

static void test_levels() {
    // test_levels.cpp:15-24
    {
        const CsrMatrix A = mpk::poisson1d(5);
        const LevelStructure ls = mpk::build_levels(A);
        EXPECT(ls.n_levels() == 5u);
        for (index_t r = 0; r < 5; ++r) EXPECT(ls.perm[r] == r);
    }
    // test_levels.cpp:26-33
    {
        const LevelStructure ls = mpk::build_levels(mpk::poisson2d(3, 3));
        const std::vector<index_t> sizes = {1, 2, 3, 2, 1};
        EXPECT(ls.n_levels() == 5u);
        for (index_t l = 0; l < 5; ++l) EXPECT(ls.level_ptr[l + 1] - ls.level_ptr[l] == sizes[l]);
    }
    // test_levels.cpp:35-46
    {
        const CsrMatrix A = mpk::from_coo(
            6, 6, {{0, 0, 1.0}, {1, 1, 2.0}, {2, 2, 3.0}, {3, 3, 4.0}, {4, 4, 5.0}, {5, 5, 6.0}});
        const LevelStructure ls = mpk::build_levels(A);
        EXPECT(ls.n_levels() == 1u);
        EXPECT(ls.level_ptr[1] == 6u);
    }
    // test_levels.cpp:58-72
    {
        const CsrMatrix A = mpk::from_coo(
            5, 5, {{0, 1, 1.0}, {1, 0, 1.0}, {1, 2, 1.0}, {2, 1, 1.0}, {3, 4, 1.0}, {4, 3, 1.0}});
        const LevelStructure ls = mpk::build_levels(A);
        EXPECT(ls.n_levels() == 3u);
        EXPECT(ls.level_ptr[1] - ls.level_ptr[0] == 2u);
        EXPECT(ls.level_ptr[2] - ls.level_ptr[1] == 2u);
        EXPECT(ls.level_ptr[3] - ls.level_ptr[2] == 1u);
    }
    // test_levels.cpp:74-84
    {
        const LevelStructure ls = mpk::build_levels(mpk::random_spd(200, 5, 77));
        for (index_t i = 0; i + 1 < ls.n_rows; ++i) {
            const index_t a = ls.inv_perm[i], b = ls.inv_perm[i + 1];
            EXPECT(ls.levels[a] < ls.levels[b] || (ls.levels[a] == ls.levels[b] && a < b));
            EXPECT(ls.perm[a] == i);
        }
    }
    // test_levels.cpp:86-93
    for (const CsrMatrix& A :
         {mpk::poisson2d(20, 17), mpk::poisson3d(7, 8, 9), mpk::random_csr(300, 5, 11)}) {
        const LevelStructure ls = mpk::build_levels(A);
        EXPECT(mpk::validate_levels(mpk::permute(A, ls.perm), ls));
    }
    // test_levels.cpp:95-107
    {
        const CsrMatrix A =
            mpk::from_coo(4, 4, {{0, 3, 1.0}, {0, 0, 1.0}, {1, 1, 1.0}, {2, 2, 1.0}, {3, 3, 1.0}});
        LevelStructure fake;
        fake.n_rows = 4;
        fake.levels = {0, 1, 2, 3};
        fake.perm = {0, 1, 2, 3};
        fake.inv_perm = {0, 1, 2, 3};
        fake.level_ptr = {0, 1, 2, 3, 4};
        EXPECT(!mpk::validate_levels(A, fake));
    }
    // test_levels.cpp:109-122
    EXPECT((mpk::greedy_group(std::vector<std::size_t>(10, 1000), 2500) ==
            std::vector<index_t>{0, 2, 4, 6, 8, 10}));
    EXPECT((mpk::greedy_group({1000, 5000, 1000, 1000}, 2500) == std::vector<index_t>{0, 1, 2, 4}));
    EXPECT((mpk::greedy_group({10, 10, 10}, 0) == std::vector<index_t>{0, 1, 2, 3}));
    // test_levels.cpp:124-147
    {
        const CsrMatrix A = mpk::poisson2d(64, 64);
        const LevelStructure ls = mpk::build_levels(A);
        const CsrMatrix P = mpk::permute(A, ls.perm);
        const ExecutionPlan plan = mpk::group_levels(ls, P, 100 * 1024, 4);
        EXPECT(plan.target_bytes == 100 * 1024 / 5);
        EXPECT(plan.group_rows.front() == 0u && plan.group_rows.back() == A.n_rows);
        EXPECT(plan.group_level_ptr.back() == ls.n_levels());
        for (index_t g = 0; g < plan.n_groups(); ++g) {
            EXPECT(plan.group_rows[g] < plan.group_rows[g + 1]);
            EXPECT(plan.group_footprint[g] ==
                   mpk::row_range_footprint(P, plan.group_rows[g], plan.group_rows[g + 1], 4));
            if (plan.group_footprint[g] > plan.target_bytes)
                EXPECT(plan.group_level_ptr[g + 1] - plan.group_level_ptr[g] == 1u);
        }
    }
    // test_levels.cpp:149-155
    {
        const CsrMatrix A = mpk::poisson1d(10);
        const LevelStructure ls = mpk::build_levels(A);
        EXPECT_THROW(mpk::group_levels(ls, A, 1024, 0), std::invalid_argument);
        const CsrMatrix B = mpk::poisson1d(11);
        EXPECT_THROW(mpk::group_levels(ls, B, 1024, 2), std::invalid_argument);
    }
}

static void test_wavefront() {
    // test_mpk.cpp:47-58
    const auto order = mpk::wavefront_schedule(3, 2);
    const std::vector<std::pair<index_t, int>> expect = {{0, 1}, {1, 1}, {0, 2}, {2, 1}, {1, 2}, {2, 2}};
    EXPECT(order.size() == expect.size());
    for (std::size_t i = 0; i < order.size() && i < expect.size(); ++i)
        EXPECT(order[i].group == expect[i].first && order[i].stage == expect[i].second);
    // test_mpk.cpp:72-102 / acceptance.cpp C3 dependency audit (host execute hook)
    for (index_t ng = 1; ng <= 10; ++ng)
        for (int p_m = 1; p_m <= 8; ++p_m) {
            const ExecutionPlan plan = synthetic_plan(ng, p_m);
            std::vector<int> done(ng * (p_m + 1), 0);
            std::size_t cells = 0;
            mpk::execute(plan, [&](index_t rs, index_t, int p, int) {
                const int q = p;
                if (q > 1) {
                    if (rs > 0) EXPECT(done[(rs - 1) * (p_m + 1) + q - 1]);
                    EXPECT(done[rs * (p_m + 1) + q - 1]);
                    if (rs + 1 < ng) EXPECT(done[(rs + 1) * (p_m + 1) + q - 1]);
                }
                done[rs * (p_m + 1) + q] = 1;
                ++cells;
            });
            EXPECT(cells == static_cast<std::size_t>(ng) * p_m);
        }
}

static void test_mpk() {
    // test_mpk.cpp:125-139 dense oracle
    {
        const CsrMatrix A = mpk::poisson2d(12, 9);
        std::vector<double> x(A.n_rows);
        for (std::size_t i = 0; i < x.size(); ++i) x[i] = std::sin(0.37 * i) + 0.5;
        VectorBlock block(A.n_rows, 6);
        mpk::baseline_mpk(A, x, 5, block);
        std::vector<double> y = x, z(x.size());
        for (int p = 1; p <= 5; ++p) {
            for (index_t r = 0; r < A.n_rows; ++r) {
                double acc = 0.0;
                for (index_t k = A.row_ptr[r]; k < A.row_ptr[r + 1]; ++k) acc += A.values[k] * y[A.col_idx[k]];
                z[r] = acc;
            }
            y = z;
            double scale = 0.0;
            for (double v : y) scale = std::max(scale, std::abs(v));
            for (index_t r = 0; r < A.n_rows; ++r) EXPECT(std::abs(block.slice(p)[r] - y[r]) <= 1e-13 * scale);
        }
    }
    // test_mpk.cpp:141-159 blocked == baseline, bitwise
    for (const CsrMatrix& A :
         {mpk::poisson2d(48, 37), mpk::poisson3d(9, 10, 11), mpk::random_csr(2000, 5, 3)}) {
        const auto ls = mpk::build_levels(A);
        const CsrMatrix P = mpk::permute(A, ls.perm);
        std::vector<double> x(A.n_rows);
        for (std::size_t i = 0; i < x.size(); ++i) x[i] = std::cos(0.11 * i);
        for (int p_m : {1, 3, 6}) {
            const ExecutionPlan plan = mpk::group_levels(ls, P, 64 * 1024, p_m);
            VectorBlock base(P.n_rows, p_m + 1), blk(P.n_rows, p_m + 1);
            mpk::baseline_mpk(P, x, p_m, base);
            mpk::mpk(plan, P, x, p_m, blk);
            EXPECT(bitwise_equal(base.data, blk.data));
        }
    }
    // test_mpk.cpp:176-206 shifted
    {
        const CsrMatrix A = mpk::poisson2d(30, 30);
        const auto ls = mpk::build_levels(A);
        const CsrMatrix P = mpk::permute(A, ls.perm);
        std::vector<double> x(A.n_rows);
        for (std::size_t i = 0; i < x.size(); ++i) x[i] = 1.0 / (1.0 + i % 17);
        const std::vector<cplx> shifts = {{2.0, 0.0}, {3.5, 1.5}, {3.5, -1.5}, {4.0, 0.0}, {1.0, 0.0}};
        const ExecutionPlan plan = mpk::group_levels(ls, P, 16 * 1024, 5);
        VectorBlock base(P.n_rows, 6), blk(P.n_rows, 6);
        mpk::baseline_mpk_shifted(P, x, shifts, base);
        mpk::mpk_shifted(plan, P, x, shifts, blk);
        EXPECT(bitwise_equal(base.data, blk.data));
    }
    // test_mpk.cpp:208-222
    {
        const CsrMatrix A = mpk::poisson1d(8);
        std::vector<double> x(8, 1.0);
        VectorBlock block(8, 4);
        EXPECT_THROW(mpk::baseline_mpk_shifted(A, x, {{1.0, 0.0}, {2.0, 1.0}}, block), std::invalid_argument);
        EXPECT_THROW(mpk::baseline_mpk_shifted(A, x, {{2.0, 1.0}, {0.5, 0.0}, {2.0, -1.0}}, block),
                     std::invalid_argument);
        EXPECT_THROW(mpk::baseline_mpk_shifted(A, x, {{2.0, -1.0}, {2.0, 1.0}, {0.0, 0.0}}, block),
                     std::invalid_argument);
    }
    // test_mpk.cpp:224-245
    {
        const std::vector<double> table = {1.0, 1.8, 2.1, 2.0};
        auto res = mpk::tune_p(1, 4, [&](int p) { return table[p - 1]; });
        EXPECT(res.p_opt == 3 && res.table.size() == 4u);
        const std::vector<double> tied = {1.0, 2.1, 1.5, 2.1};
        EXPECT(mpk::tune_p(1, 4, [&](int p) { return tied[p - 1]; }).p_opt == 2);
        const CsrMatrix A = mpk::poisson2d(48, 48);
        const auto ls = mpk::build_levels(A);
        const CsrMatrix P = mpk::permute(A, ls.perm);
        const auto measured = mpk::tune_p(ls, P, 256 * 1024, 1, 3);
        EXPECT(measured.p_opt >= 1 && measured.p_opt <= 3 && measured.table.size() == 3u);
        for (const auto& pg : measured.table) EXPECT(pg.second > 0.0);
    }
    // test_mpk.cpp:247-259
    {
        const CsrMatrix A = mpk::poisson1d(10);
        const auto ls = mpk::build_levels(A);
        const CsrMatrix P = mpk::permute(A, ls.perm);
        const ExecutionPlan plan = mpk::group_levels(ls, P, 1024, 2);
        std::vector<double> x(10, 1.0);
        VectorBlock small(10, 2);
        EXPECT_THROW(mpk::mpk(plan, P, x, 2, small), std::invalid_argument);
        VectorBlock ok(10, 4);
        EXPECT_THROW(mpk::mpk(plan, P, x, 3, ok), std::invalid_argument);
        std::vector<double> bad(9, 1.0);
        EXPECT_THROW(mpk::baseline_mpk(A, bad, 2, ok), std::invalid_argument);
        EXPECT_THROW(ok.slice(4), std::out_of_range);
    }
    // acceptance.cpp C1 (a subset: corpus x p 1..8, 1 MiB budget, x = random_vector(n, 42))
    for (const CsrMatrix& A : {mpk::poisson2d(256, 256), mpk::poisson3d(32, 32, 32), mpk::random_spd(50000, 5, 777)}) {
        const auto ls = mpk::build_levels(A);
        const CsrMatrix P = mpk::permute(A, ls.perm);
        const std::vector<double> x = random_vector(P.n_rows, 42);
        for (int p = 1; p <= 8; ++p) {
            const ExecutionPlan plan = mpk::group_levels(ls, P, std::size_t{1} << 20, p);
            VectorBlock base(P.n_rows, p + 1), blk(P.n_rows, p + 1);
            mpk::baseline_mpk(P, x, p, base);
            mpk::mpk(plan, P, x, p, blk);
            EXPECT(bitwise_equal(base.data, blk.data));
        }
    }
}

// csr.hpp:207-227 transpose and threading.hpp:34-46 resolve_threads (host helpers).
static void test_host_helpers() {
    const CsrMatrix A = mpk::random_csr(300, 5, 11);  // nonsymmetric pattern
    const CsrMatrix T = mpk::transpose(A);
    EXPECT(T.n_rows == A.n_cols && T.n_cols == A.n_rows && T.nnz() == A.nnz());
    bool sorted = true, match = true;
    for (index_t r = 0; r < T.n_rows; ++r)
        for (index_t k = T.row_ptr[r]; k < T.row_ptr[r + 1]; ++k) {
            if (k + 1 < T.row_ptr[r + 1] && T.col_idx[k] >= T.col_idx[k + 1]) sorted = false;
            const index_t c = T.col_idx[k];  // A(c, r) must hold the same value
            bool found = false;
            for (index_t j = A.row_ptr[c]; j < A.row_ptr[c + 1]; ++j)
                if (A.col_idx[j] == r) found = std::memcmp(&A.values[j], &T.values[k], 8) == 0;
            match = match && found;
        }
    EXPECT(sorted);
    EXPECT(match);
    const CsrMatrix TT = mpk::transpose(T);
    EXPECT(TT.row_ptr == A.row_ptr && TT.col_idx == A.col_idx);
    EXPECT(mpk::resolve_threads(7) == 7);
    {  // matrix_market.hpp through the GPU reader: a symmetric file with a duplicate entry
        const char* path = "/tmp/mpkg_facade_test.mtx";
        FILE* f = std::fopen(path, "w");
        std::fputs("%%MatrixMarket matrix coordinate real symmetric\n% c\n3 3 4\n1 1 2.0\n2 1 -1.5\n"
                   "3 3 4.0\n2 1 0.25\n", f);
        std::fclose(f);
        const CsrMatrix M = mpk::read_matrix_market(path);
        const CsrMatrix R = mpk::from_coo(3, 3, {{0, 0, 2.0}, {1, 0, -1.5}, {0, 1, -1.5}, {2, 2, 4.0},
                                                {1, 0, 0.25}, {0, 1, 0.25}});
        EXPECT(M.row_ptr == R.row_ptr && M.col_idx == R.col_idx && bitwise_equal(M.values, R.values));
        EXPECT_THROW(mpk::read_matrix_market("/tmp/does_not_exist.mtx"), std::runtime_error);
    }
    EXPECT(mpk::resolve_threads() >= 1);
}

// proj/tests/test_relax.cpp:112-206 (Jacobi), with a small dense recurrence standing in for the
// Eigen oracle of MultiSweepMatchesDenseOracle.
static std::vector<double> dense_jacobi(const CsrMatrix& a, const std::vector<double>& v, int sweeps) {
    const std::size_t n = a.n_rows;
    std::vector<double> d(n), z(n), t(n);
    for (index_t r = 0; r < a.n_rows; ++r)
        for (index_t k = a.row_ptr[r]; k < a.row_ptr[r + 1]; ++k)
            if (a.col_idx[k] == r) d[r] = a.values[k];
    for (std::size_t r = 0; r < n; ++r) z[r] = v[r] / d[r];
    for (int s = 2; s <= sweeps; ++s) {
        for (index_t r = 0; r < a.n_rows; ++r) {
            long double acc = 0.0L;
            for (index_t k = a.row_ptr[r]; k < a.row_ptr[r + 1]; ++k)
                if (a.col_idx[k] != r) acc += (long double)a.values[k] * z[a.col_idx[k]];
            t[r] = (double)(((long double)v[r] - acc) / d[r]);
        }
        z.swap(t);
    }
    return z;
}

static void test_jacobi() {
    {  // SetupRejectsBadInput
        CsrMatrix a = mpk::poisson1d(4);
        EXPECT_THROW(mpk::jacobi_setup(a, 0), std::invalid_argument);
        CsrMatrix zd = mpk::from_coo(2, 2, {{0, 0, 0.0}, {0, 1, 1.0}, {1, 0, 1.0}, {1, 1, 2.0}});
        EXPECT_THROW(mpk::jacobi_setup(zd, 1), std::runtime_error);
        CsrMatrix md = mpk::from_coo(2, 2, {{0, 1, 1.0}, {1, 0, 1.0}, {1, 1, 2.0}});
        EXPECT_THROW(mpk::jacobi_setup(md, 1), std::runtime_error);
    }
    {  // IdentityAndDiagonalExamples
        CsrMatrix i2 = mpk::from_coo(2, 2, {{0, 0, 1.0}, {1, 1, 1.0}});
        mpk::JacobiPrecon p = mpk::jacobi_setup(i2, 1);
        std::vector<double> z;
        mpk::jacobi_apply(p, i2, {5.0, -7.0}, z);
        EXPECT(z[0] == 5.0 && z[1] == -7.0);
        CsrMatrix d = mpk::from_coo(2, 2, {{0, 0, 2.0}, {1, 1, 4.0}});
        mpk::JacobiPrecon pd = mpk::jacobi_setup(d, 1);
        mpk::jacobi_apply(pd, d, {2.0, 4.0}, z);
        EXPECT(z[0] == 1.0 && z[1] == 1.0);
    }
    {  // TwoSweepExample: A = [[2,1],[1,2]], v = (1,1), two sweeps -> (0.25, 0.25)
        CsrMatrix a = mpk::from_coo(2, 2, {{0, 0, 2.0}, {0, 1, 1.0}, {1, 0, 1.0}, {1, 1, 2.0}});
        mpk::JacobiPrecon p = mpk::jacobi_setup(a, 2);
        std::vector<double> z;
        mpk::jacobi_apply(p, a, {1.0, 1.0}, z);
        EXPECT(z[0] == 0.25 && z[1] == 0.25);
        EXPECT(p.diag.pos == mpk::diagonal_positions(a));
    }
    {  // MultiSweepMatchesDenseOracle
        const CsrMatrix a = mpk::random_spd(40, 4, 123);
        const std::vector<double> v = random_vector(40, 7);
        for (int sweeps : {1, 2, 3, 4}) {
            mpk::JacobiPrecon p = mpk::jacobi_setup(a, sweeps);
            std::vector<double> z;
            mpk::jacobi_apply(p, a, v, z);
            const std::vector<double> want = dense_jacobi(a, v, sweeps);
            double err = 0.0, scale = 0.0;
            for (std::size_t i = 0; i < z.size(); ++i) {
                err = std::max(err, std::fabs(z[i] - want[i]));
                scale = std::max(scale, std::fabs(want[i]));
            }
            EXPECT(err <= 1e-14 * scale);
        }
    }
    {  // OpEqualsApplyThenSpmvBitwise
        const CsrMatrix a = mpk::random_spd(60, 5, 9);
        const std::vector<double> v = random_vector(60, 11);
        for (int sweeps : {1, 2, 3}) {
            mpk::JacobiPrecon p = mpk::jacobi_setup(a, sweeps);
            std::vector<double> z, want(a.n_rows), y;
            mpk::jacobi_apply(p, a, v, z);
            mpk::spmv(a, z, want);
            mpk::jacobi_op(p, a, v, y);
            EXPECT(bitwise_equal(want, y));
        }
    }
    {  // BlockedOpBitwiseEqualsSequential
        const CsrMatrix a = mpk::poisson2d(32, 32);
        const std::vector<double> v = random_vector(a.n_rows, 21);
        const LevelStructure ls = mpk::build_levels(a);
        const CsrMatrix ap = mpk::permute(a, ls.perm);
        for (int sweeps : {1, 3}) {
            ExecutionPlan plan = mpk::group_levels(ls, ap, 64 * 1024, 1);
            plan.sub_powers = mpk::jacobi_stages(sweeps);
            plan.invalidate();
            EXPECT(plan.n_groups() > 2u);
            mpk::JacobiPrecon p = mpk::jacobi_setup(ap, sweeps);
            std::vector<double> y_seq, y_blk;
            mpk::jacobi_op(p, ap, v, y_seq);
            mpk::jacobi_op_blocked(p, ap, plan, v, y_blk);
            EXPECT(bitwise_equal(y_seq, y_blk));
            ExecutionPlan bad = plan;
            bad.sub_powers = 7;
            bad.invalidate();
            EXPECT_THROW(mpk::jacobi_op_blocked(p, ap, bad, v, y_blk), std::invalid_argument);
        }
    }
}

// proj/tests/test_relax.cpp:208-406 (GS2).  The Eigen dense solves of NilpotentExactness /
// BackwardDirectionSolvesUpperTriangular are restated as plain triangular substitutions.
static CsrMatrix random_lower(std::size_t n, unsigned seed) {
    std::mt19937_64 rng(seed);
    std::uniform_real_distribution<double> u(0.5, 1.5);
    std::vector<mpk::Triplet> t;
    for (std::size_t i = 0; i < n; ++i) {
        t.push_back({(index_t)i, (index_t)i, 2.0 + u(rng)});
        for (std::size_t j = 0; j < i; ++j)
            if ((rng() & 1u) == 0) t.push_back({(index_t)i, (index_t)j, u(rng) - 1.0});
    }
    return mpk::from_coo((index_t)n, (index_t)n, t);
}

static std::vector<double> tri_solve(const CsrMatrix& a, const std::vector<double>& v, bool lower) {
    const std::size_t n = a.n_rows;
    std::vector<double> z(n, 0.0);
    for (std::size_t s = 0; s < n; ++s) {
        const index_t r = (index_t)(lower ? s : n - 1 - s);
        long double acc = v[r];
        double d = 0.0;
        for (index_t k = a.row_ptr[r]; k < a.row_ptr[r + 1]; ++k) {
            if (a.col_idx[k] == r) d = a.values[k];
            else acc -= (long double)a.values[k] * z[a.col_idx[k]];
        }
        z[r] = (double)(acc / d);
    }
    return z;
}

static double max_err(const std::vector<double>& a, const std::vector<double>& b) {
    double e = 0.0;
    for (std::size_t i = 0; i < a.size(); ++i) e = std::max(e, std::fabs(a[i] - b[i]));
    return e;
}

static double max_abs(const std::vector<double>& a) {
    double m = 0.0;
    for (double v : a) m = std::max(m, std::fabs(v));
    return m;
}

static void test_gs2() {
    {  // SetupRejectsBadInput
        CsrMatrix a = mpk::poisson1d(4);
        EXPECT_THROW(mpk::gs2_setup(a, -1), std::invalid_argument);
        EXPECT_THROW(mpk::gs2_setup(a, 1, 0), std::invalid_argument);
        CsrMatrix zd = mpk::from_coo(2, 2, {{0, 0, 0.0}, {1, 1, 2.0}});
        EXPECT_THROW(mpk::gs2_setup(zd, 1), std::runtime_error);
    }
    {  // DiagonalMatrixIsExactForAnyGamma
        CsrMatrix a = mpk::from_coo(3, 3, {{0, 0, 2.0}, {1, 1, -4.0}, {2, 2, 0.5}});
        for (int gamma : {0, 1, 3}) {
            mpk::Gs2Precon p = mpk::gs2_setup(a, gamma);
            std::vector<double> z;
            mpk::gs2_apply(p, a, {2.0, 8.0, 1.0}, z);
            EXPECT(z[0] == 1.0 && z[1] == -2.0 && z[2] == 2.0);
        }
    }
    {  // LowerTriangularExampleEqualsExactSolve: A = [[2,0],[1,2]], v = (2,2) -> (1, 0.5)
        CsrMatrix a = mpk::from_coo(2, 2, {{0, 0, 2.0}, {1, 0, 1.0}, {1, 1, 2.0}});
        mpk::Gs2Precon p = mpk::gs2_setup(a, 1);
        std::vector<double> z;
        mpk::gs2_apply(p, a, {2.0, 2.0}, z);
        EXPECT(z[0] == 1.0 && z[1] == 0.5);
    }
    {  // GammaZeroIsDiagonalScaling
        const CsrMatrix a = mpk::random_spd(20, 3, 31);
        mpk::Gs2Precon p = mpk::gs2_setup(a, 0);
        const std::vector<double> v = random_vector(20, 33);
        std::vector<double> z;
        mpk::gs2_apply(p, a, v, z);
        bool ok = true;
        for (std::size_t i = 0; i < 20; ++i) ok = ok && z[i] == p.diag.inv[i] * v[i];
        EXPECT(ok);
    }
    for (unsigned seed : {1u, 2u, 3u, 4u, 5u}) {  // NilpotentExactness
        const std::size_t n = 6;
        const CsrMatrix a = random_lower(n, seed);
        const std::vector<double> v = random_vector(n, seed + 100);
        mpk::Gs2Precon p = mpk::gs2_setup(a, (int)n - 1);
        std::vector<double> z;
        mpk::gs2_apply(p, a, v, z);
        const std::vector<double> want = tri_solve(a, v, true);
        EXPECT(max_err(z, want) <= 1e-14 * max_abs(want));
    }
    {  // BackwardDirectionSolvesUpperTriangular
        const CsrMatrix a = mpk::transpose(random_lower(6, 77));
        const std::vector<double> v = random_vector(6, 78);
        mpk::Gs2Precon p = mpk::gs2_setup(a, 5, 1, mpk::SweepDirection::backward);
        std::vector<double> z;
        mpk::gs2_apply(p, a, v, z);
        const std::vector<double> want = tri_solve(a, v, false);
        EXPECT(max_err(z, want) <= 1e-14 * max_abs(want));
    }
    {  // OpAndResidualShareKernelsBitwise
        const CsrMatrix a = mpk::random_spd(50, 5, 51);
        const std::vector<double> v = random_vector(50, 53);
        mpk::Gs2Precon p = mpk::gs2_setup(a, 1);
        std::vector<double> z, y_manual(a.n_rows), y;
        mpk::gs2_apply(p, a, v, z);
        mpk::spmv(a, z, y_manual);
        mpk::gs2_op(p, a, v, y);
        EXPECT(bitwise_equal(y_manual, y));
        std::vector<double> r_manual(50), z2(50, 0.0), r;
        for (std::size_t i = 0; i < 50; ++i) r_manual[i] = v[i] - y_manual[i];
        mpk::gs2_smooth_residual(p, a, v, z2, r);
        EXPECT(bitwise_equal(z, z2));
        EXPECT(bitwise_equal(r_manual, r));
    }
    {  // BlockedVariantsBitwiseEqualSequential + PlanShapeMismatchRejected
        const CsrMatrix a = mpk::poisson2d(20, 20);
        const std::vector<double> v = random_vector(a.n_rows, 61);
        const std::vector<double> guess = random_vector(a.n_rows, 62);
        const LevelStructure ls = mpk::build_levels(a);
        const CsrMatrix ap = mpk::permute(a, ls.perm);
        for (int gamma : {0, 1, 2})
            for (int sweeps : {1, 2})
                for (auto dir : {mpk::SweepDirection::forward, mpk::SweepDirection::backward}) {
                    ExecutionPlan plan = mpk::group_levels(ls, ap, 8 * 1024, sweeps);
                    plan.sub_powers = gamma + 2;
                    plan.invalidate();
                    mpk::Gs2Precon p = mpk::gs2_setup(ap, gamma, sweeps, dir);
                    std::vector<double> z_seq = guess, z_blk = guess;
                    mpk::gs2_smooth(p, ap, v, z_seq);
                    mpk::gs2_smooth_blocked(p, ap, plan, v, z_blk);
                    EXPECT(bitwise_equal(z_seq, z_blk));
                    std::vector<double> y_seq, y_blk;
                    mpk::gs2_op(p, ap, v, y_seq);
                    mpk::gs2_op_blocked(p, ap, plan, v, y_blk);
                    EXPECT(bitwise_equal(y_seq, y_blk));
                    std::vector<double> zr_seq(a.n_rows, 0.0), zr_blk(a.n_rows, 0.0), r_seq, r_blk;
                    mpk::gs2_smooth_residual(p, ap, v, zr_seq, r_seq);
                    mpk::gs2_smooth_residual_blocked(p, ap, plan, v, zr_blk, r_blk);
                    EXPECT(bitwise_equal(zr_seq, zr_blk) && bitwise_equal(r_seq, r_blk));
                }
        ExecutionPlan plan = mpk::group_levels(ls, ap, 4 * 1024, 1);
        plan.sub_powers = 3;
        plan.invalidate();
        mpk::Gs2Precon p = mpk::gs2_setup(ap, 2);  // needs sub_powers 4
        std::vector<double> y;
        EXPECT_THROW(mpk::gs2_op_blocked(p, ap, plan, v, y), std::invalid_argument);
    }
}

// proj/tests/test_poly.cpp with the roots given (the reference's Eigen-based setup is not part of
// this library): ScaledIdentityDegreeOne, exactness on a known spectrum (real and complex pair),
// blocked == sequential with root slicing, plan shape mismatch.
static void test_poly() {
    using cplx = std::complex<double>;
    {
        CsrMatrix a = mpk::from_coo(2, 2, {{0, 0, 2.0}, {1, 1, 2.0}});
        mpk::PolyPrecon exact;
        exact.theta = {cplx(2.0, 0.0)};
        exact.degree = 1;
        std::vector<double> z;
        mpk::poly_apply(exact, a, {4.0, 6.0}, z);
        EXPECT(z[0] == 2.0 && z[1] == 3.0);
    }
    {  // eigenvalues 1 +- 2i and 3: A z = v when the roots are the spectrum
        const CsrMatrix a = mpk::from_coo(3, 3, {{0, 0, 1.0}, {0, 1, -2.0}, {1, 0, 2.0}, {1, 1, 1.0}, {2, 2, 3.0}});
        mpk::PolyPrecon p;
        p.theta = {cplx(3.0, 0.0), cplx(1.0, 2.0), cplx(1.0, -2.0)};
        p.degree = 3;
        const std::vector<double> v = {0.3, -0.7, 1.1};
        std::vector<double> z, az(3);
        mpk::poly_apply(p, a, v, z);
        mpk::spmv(a, z, az);
        EXPECT(max_err(az, v) <= 1e-10);
    }
    {
        const CsrMatrix a = mpk::poisson2d(48, 48);
        const std::vector<double> v = random_vector(a.n_rows, 95);
        const LevelStructure ls = mpk::build_levels(a);
        const CsrMatrix ap = mpk::permute(a, ls.perm);
        mpk::PolyPrecon p;
        p.theta = {cplx(7.5, 0), cplx(0.3, 0), cplx(4.0, 1.0), cplx(4.0, -1.0), cplx(2.0, 0), cplx(6.0, 0),
                   cplx(1.0, 0.5), cplx(1.0, -0.5)};
        p.degree = 8;
        ExecutionPlan plan = mpk::group_levels(ls, ap, 16 * 1024, 3);  // p_m 3 < 7 powers: slicing
        plan.sub_powers = mpk::poly_sub_powers(p);
        plan.invalidate();
        std::vector<double> z_seq, z_blk;
        mpk::poly_apply(p, ap, v, z_seq);
        mpk::poly_apply_blocked(p, ap, plan, v, z_blk);
        EXPECT(bitwise_equal(z_seq, z_blk));
        plan.sub_powers = 3;
        plan.invalidate();
        EXPECT_THROW(mpk::poly_apply_blocked(p, ap, plan, v, z_blk), std::invalid_argument);
    }
}

// proj/tests/test_ortho.cpp (Tsqr / Icgs suites) through the facade; defects computed with
// plain loops instead of Eigen.
static double ortho_defect(const std::vector<double>& q, std::size_t rows, std::size_t cols) {
    double m = 0.0;
    for (std::size_t a = 0; a < cols; ++a)
        for (std::size_t b = 0; b < cols; ++b) {
            double s = 0.0;
            for (std::size_t i = 0; i < rows; ++i) s += q[a * rows + i] * q[b * rows + i];
            m = std::max(m, std::abs(s - (a == b ? 1.0 : 0.0)));
        }
    return m;
}

static double factorization_defect(const std::vector<double>& v, const std::vector<double>& q,
                                   const std::vector<double>& r, std::size_t rows, std::size_t cols) {
    double m = 0.0;
    for (std::size_t j = 0; j < cols; ++j)
        for (std::size_t i = 0; i < rows; ++i) {
            double s = 0.0;
            for (std::size_t k = 0; k < cols; ++k) s += q[k * rows + i] * r[j * cols + k];
            m = std::max(m, std::abs(s - v[j * rows + i]));
        }
    return m;
}

static void test_ortho() {
    {  // Tsqr.RandomBlockBounds
        const std::size_t rows = 1000, cols = 4;
        const std::vector<double> v_in = random_vector(rows * cols, 17);
        std::vector<double> q = v_in, r(cols * cols);
        mpk::tsqr(q.data(), rows, cols, r.data());
        EXPECT(ortho_defect(q, rows, cols) <= 1e-13);
        EXPECT(factorization_defect(v_in, q, r, rows, cols) <= 1e-13 * max_abs(v_in));
        for (std::size_t j = 0; j < cols; ++j) {
            EXPECT(r[j * cols + j] >= 0.0);
            for (std::size_t i = j + 1; i < cols; ++i) EXPECT(r[j * cols + i] == 0.0);
        }
    }
    {  // Tsqr.OrthonormalInputGivesIdentityR
        const std::size_t rows = 600, cols = 5;
        std::vector<double> q = random_vector(rows * cols, 3), r(cols * cols);
        mpk::tsqr(q.data(), rows, cols, r.data());
        mpk::tsqr(q.data(), rows, cols, r.data());
        for (std::size_t j = 0; j < cols; ++j)
            for (std::size_t i = 0; i < cols; ++i) EXPECT(std::abs(r[j * cols + i] - (i == j ? 1.0 : 0.0)) <= 1e-13);
    }
    {  // Tsqr.DuplicateColumnsFlagRankDeficiency
        const std::size_t rows = 500, cols = 3;
        std::vector<double> v = random_vector(rows * cols, 5);
        std::copy_n(v.begin(), rows, v.begin() + rows);
        const double vmax = max_abs(v);
        std::vector<double> r(cols * cols);
        mpk::tsqr(v.data(), rows, cols, r.data());
        EXPECT(mpk::tsqr_rank_deficient(r.data(), cols, 1e-14 * vmax * std::sqrt(double(rows))));
        const std::vector<double> full = {2.0, 0.0, 0.0, 1.0};
        EXPECT(!mpk::tsqr_rank_deficient(full.data(), 2, 1e-14));
    }
    {  // Tsqr.PanelTreeMatchesSinglePanelToRoundoff
        const std::size_t rows = 10000, cols = 5;
        const std::vector<double> v_in = random_vector(rows * cols, 29);
        std::vector<double> q_one = v_in, r_one(cols * cols), q_many = v_in, r_many(cols * cols);
        mpk::tsqr(q_one.data(), rows, cols, r_one.data(), rows);
        mpk::tsqr(q_many.data(), rows, cols, r_many.data(), 64);
        EXPECT(ortho_defect(q_many, rows, cols) <= 1e-13);
        EXPECT(factorization_defect(v_in, q_many, r_many, rows, cols) <= 1e-13 * max_abs(v_in));
        double d = 0.0;
        for (std::size_t e = 0; e < r_one.size(); ++e) d = std::max(d, std::abs(r_one[e] - r_many[e]));
        EXPECT(d <= 1e-10 * max_abs(v_in));
    }
    {  // Tsqr.ThreadCountDoesNotChangeBits
        const std::size_t rows = 8192, cols = 6;
        const std::vector<double> v_in = random_vector(rows * cols, 41);
        std::vector<double> q1 = v_in, r1(cols * cols);
        mpk::tsqr(q1.data(), rows, cols, r1.data(), 1024, 1);
        for (int threads : {2, 4, 8}) {
            std::vector<double> q = v_in, r(cols * cols);
            mpk::tsqr(q.data(), rows, cols, r.data(), 1024, threads);
            EXPECT(bitwise_equal(q1, q) && bitwise_equal(r1, r));
        }
    }
    {  // Tsqr.RejectsWideBlocks
        std::vector<double> v(6, 1.0), r(9);
        EXPECT_THROW(mpk::tsqr(v.data(), 2, 3, r.data()), std::invalid_argument);
    }
    {  // Icgs.ExactlyOrthogonalInputIsUntouched
        const std::size_t rows = 64, qcols = 4, vcols = 2;
        std::vector<double> q(rows * qcols, 0.0);
        for (std::size_t k = 0; k < qcols; ++k) q[k * rows + k] = 1.0;
        std::vector<double> v = random_vector(rows * vcols, 7);
        for (std::size_t j = 0; j < vcols; ++j)
            for (std::size_t k = 0; k < qcols; ++k) v[j * rows + k] = 0.0;
        const std::vector<double> v_in = v;
        auto coeff = mpk::icgs_block_orthogonalize(q.data(), rows, qcols, v.data(), vcols, 2);
        for (double c : coeff) EXPECT(c == 0.0);
        EXPECT(bitwise_equal(v, v_in));
    }
    {  // Icgs.DuplicateOfBasisColumnProjectsToZero
        const std::size_t rows = 1000, qcols = 5;
        std::vector<double> q = random_vector(rows * qcols, 11), r(qcols * qcols);
        mpk::tsqr(q.data(), rows, qcols, r.data());
        std::vector<double> v(q.begin(), q.begin() + rows);
        auto coeff = mpk::icgs_block_orthogonalize(q.data(), rows, qcols, v.data(), 1, 1);
        EXPECT(max_abs(v) <= 1e-13);
        EXPECT(std::abs(coeff[0] - 1.0) <= 1e-12);
        for (std::size_t k = 1; k < qcols; ++k) EXPECT(std::abs(coeff[k]) <= 1e-12);
    }
    {  // Icgs.CrossProductsAfterSweeps
        const std::size_t rows = 1000, qcols = 8, vcols = 4;
        std::vector<double> q = random_vector(rows * qcols, 13), rq(qcols * qcols);
        mpk::tsqr(q.data(), rows, qcols, rq.data());
        const std::vector<double> v_in = random_vector(rows * vcols, 19);
        for (int sweeps : {1, 2}) {
            std::vector<double> v = v_in, cross(qcols * vcols);
            mpk::icgs_block_orthogonalize(q.data(), rows, qcols, v.data(), vcols, sweeps);
            mpk::block_dots(q.data(), v.data(), rows, qcols, vcols, cross.data());
            EXPECT(max_abs(cross) <= (sweeps == 1 ? 1e-10 : 1e-12));
        }
    }
    {  // Icgs.CoefficientsReconstructTheProjection
        const std::size_t rows = 128, qcols = 3, vcols = 2;
        std::vector<double> q(rows * qcols, 0.0);
        for (std::size_t k = 0; k < qcols; ++k) q[k * rows + k] = 1.0;
        const std::vector<double> c0 = {0.5, -2.0, 1.25, 3.0, 0.0, -0.75};
        std::vector<double> w = random_vector(rows * vcols, 23);
        for (std::size_t j = 0; j < vcols; ++j)
            for (std::size_t k = 0; k < qcols; ++k) w[j * rows + k] = 0.0;
        std::vector<double> v = w;
        for (std::size_t j = 0; j < vcols; ++j)
            for (std::size_t k = 0; k < qcols; ++k) v[j * rows + k] = c0[j * qcols + k];
        auto coeff = mpk::icgs_block_orthogonalize(q.data(), rows, qcols, v.data(), vcols, 2);
        double dc = 0.0, dv = 0.0;
        for (std::size_t e = 0; e < c0.size(); ++e) dc = std::max(dc, std::abs(coeff[e] - c0[e]));
        for (std::size_t e = 0; e < w.size(); ++e) dv = std::max(dv, std::abs(v[e] - w[e]));
        EXPECT(dc <= 1e-15 && dv <= 1e-15);
    }
    {  // Icgs.ThreadCountDoesNotChangeBits
        const std::size_t rows = 4096, qcols = 7, vcols = 3;
        std::vector<double> q = random_vector(rows * qcols, 31), rq(qcols * qcols);
        mpk::tsqr(q.data(), rows, qcols, rq.data());
        const std::vector<double> v_in = random_vector(rows * vcols, 37);
        std::vector<double> v1 = v_in;
        auto c1 = mpk::icgs_block_orthogonalize(q.data(), rows, qcols, v1.data(), vcols, 2, 1);
        for (int threads : {2, 4, 8}) {
            std::vector<double> v = v_in;
            auto c = mpk::icgs_block_orthogonalize(q.data(), rows, qcols, v.data(), vcols, 2, threads);
            EXPECT(bitwise_equal(v1, v) && bitwise_equal(c1, c));
        }
    }
    {  // s-step block step (sstep.hpp:539-545): ortho_block == icgs_block_orthogonalize then tsqr
        const std::size_t rows = 100000, qcols = 25, vcols = 8;
        std::vector<double> q = random_vector(rows * qcols, 51), rq(qcols * qcols);
        mpk::tsqr(q.data(), rows, qcols, rq.data());
        const std::vector<double> v_in = random_vector(rows * vcols, 53);
        std::vector<double> v1 = v_in, r1(vcols * vcols), v2 = v_in, r2(vcols * vcols);
        auto c1 = mpk::icgs_block_orthogonalize(q.data(), rows, qcols, v1.data(), vcols, 2);
        mpk::tsqr(v1.data(), rows, vcols, r1.data());
        auto c2 = mpk::ortho_block(q.data(), rows, qcols, v2.data(), vcols, 2, r2.data());
        EXPECT(bitwise_equal(c1, c2) && bitwise_equal(v1, v2) && bitwise_equal(r1, r2));
    }
    {  // Icgs.RejectsNonPositiveSweeps / EmptyBasisReturnsEmptyCoefficients
        std::vector<double> q(8, 0.0), v(8, 1.0);
        EXPECT_THROW(mpk::icgs_block_orthogonalize(q.data(), 8, 1, v.data(), 1, 0), std::invalid_argument);
        std::vector<double> e = random_vector(64, 43);
        const std::vector<double> e_in = e;
        auto coeff = mpk::icgs_block_orthogonalize(nullptr, 32, 0, e.data(), 2, 1);
        EXPECT(coeff.empty() && bitwise_equal(e, e_in));
    }
}

int main() {
    test_ortho();
    test_host_helpers();
    test_jacobi();
    test_gs2();
    test_poly();
    test_levels();
    test_wavefront();
    test_mpk();
    std::printf("%s: %d checks, %d failures\n", g_fail ? "FAILED" : "PASSED", g_checks, g_fail);
    return g_fail ? 1 : 0;
}
