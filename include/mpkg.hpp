// mpkg.hpp — C++ facade with the reference's interface over the mpkg C ABI.
//
// Mirrors namespace `mpk` of the reference (proj/include/mpk/{csr,levels,plan,execute,mpk,
// vector_block,generators}.hpp) name for name, type for type and exception for exception, so a
// reference call site switches with `namespace mpk = mpkg;` and links libmpkg.so.  All compute
// (build_levels, permute, validate_levels, spmv, baseline_mpk, mpk, *_shifted, tune_p) runs on
// the GPU through include/mpkg.h; status codes come back as the reference's exceptions:
// MPKG_EINVAL -> std::invalid_argument, MPKG_ERANGE -> std::out_of_range, else runtime_error.
//
// Host-side types own host arrays exactly like the reference; device copies are made on first
// use and cached per object (the reference treats these structures as immutable after
// construction).  Call `invalidate()` after mutating one in place.
//
// Exception: `execute(plan, kernel)` (execute.hpp:79-113) takes an arbitrary host callback and
// therefore cannot cross to the GPU; it runs the callback in the reference's wavefront order on
// the calling thread.  The GPU power kernels never use it.
#pragma once

#include <algorithm>
#include <complex>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <new>
#include <stdexcept>
#include <string>
#include <thread>
#include <utility>
#include <vector>

#include "mpkg.h"

namespace mpkg {

using index_t = std::uint32_t;  // csr.hpp:41

namespace detail {

inline void check(int rc) {
    if (rc == MPKG_OK) return;
    const std::string msg = mpkg_last_error();
    if (rc == MPKG_EINVAL) throw std::invalid_argument(msg);
    if (rc == MPKG_ERANGE) throw std::out_of_range(msg);
    if (rc == MPKG_ENOMEM) throw std::bad_alloc();
    throw std::runtime_error(msg);
}

struct CtxHolder {
    mpkg_ctx_t h = nullptr;
    explicit CtxHolder(int device) { check(mpkg_ctx_create(device, &h)); }
    ~CtxHolder() { mpkg_ctx_destroy(h); }
};

struct CsrHolder {
    mpkg_csr_t h = nullptr;
    const void *rp = nullptr, *ci = nullptr, *v = nullptr;
    std::size_t nnz = 0;
    ~CsrHolder() { mpkg_csr_destroy(h); }
};
struct LevelsHolder {
    mpkg_levels_t h = nullptr;
    ~LevelsHolder() { mpkg_levels_destroy(h); }
};
struct PlanHolder {
    mpkg_plan_t h = nullptr;
    ~PlanHolder() { mpkg_plan_destroy(h); }
};
struct JacobiHolder {
    mpkg_jacobi_t h = nullptr;
    ~JacobiHolder() { mpkg_jacobi_destroy(h); }
};
struct Gs2Holder {
    mpkg_gs2_t h = nullptr;
    ~Gs2Holder() { mpkg_gs2_destroy(h); }
};

}  // namespace detail

/// The device the facade runs on (replaces resolve_threads, threading.hpp:34-46): device 0, or
/// the index in MPKG_DEVICE.
inline mpkg_ctx_t device_context() {
    static detail::CtxHolder ctx([] {
        const char* e = std::getenv("MPKG_DEVICE");
        return e ? std::atoi(e) : 0;
    }());
    return ctx.h;
}

/// csr.hpp:44-48
struct Triplet {
    index_t row = 0;
    index_t col = 0;
    double val = 0.0;
};

/// csr.hpp:57-65
struct CsrMatrix {
    index_t n_rows = 0;
    index_t n_cols = 0;
    std::vector<index_t> row_ptr;
    std::vector<index_t> col_idx;
    std::vector<double> values;

    index_t nnz() const { return row_ptr.empty() ? 0 : row_ptr[n_rows]; }
    void invalidate() const { dev_.reset(); }

    /// Device copy (uploaded on first use; re-uploaded if the arrays were reallocated).
    mpkg_csr_t device() const {
        if (!dev_ || dev_->rp != row_ptr.data() || dev_->ci != col_idx.data() ||
            dev_->v != values.data() || dev_->nnz != col_idx.size()) {
            auto d = std::make_shared<detail::CsrHolder>();
            detail::check(mpkg_csr_create(device_context(), n_rows, n_cols, row_ptr.data(),
                                          col_idx.data(), values.data(), &d->h));
            d->rp = row_ptr.data(), d->ci = col_idx.data(), d->v = values.data();
            d->nnz = col_idx.size();
            dev_ = d;
        }
        return dev_->h;
    }

   private:
    mutable std::shared_ptr<detail::CsrHolder> dev_;
};

/// levels.hpp:43-57
struct LevelStructure {
    index_t n_rows = 0;
    std::vector<index_t> levels;
    std::vector<index_t> perm;
    std::vector<index_t> inv_perm;
    std::vector<index_t> level_ptr;

    index_t n_levels() const {
        return level_ptr.empty() ? 0 : static_cast<index_t>(level_ptr.size() - 1);
    }
    index_t level_of_permuted(index_t new_row) const { return levels[inv_perm[new_row]]; }
    void invalidate() const { dev_.reset(); }

    mpkg_levels_t device() const {
        if (!dev_) {
            auto d = std::make_shared<detail::LevelsHolder>();
            detail::check(mpkg_levels_create(device_context(), n_rows, n_levels(),
                                             levels.empty() ? nullptr : levels.data(),
                                             perm.empty() ? nullptr : perm.data(),
                                             inv_perm.empty() ? nullptr : inv_perm.data(),
                                             level_ptr.data(), &d->h));
            dev_ = d;
        }
        return dev_->h;
    }

   private:
    mutable std::shared_ptr<detail::LevelsHolder> dev_;
    friend LevelStructure build_levels(const CsrMatrix&);
};

/// plan.hpp:41-54 (plus the level offsets the GPU executor derives dependencies from)
struct ExecutionPlan {
    int p_m = 1;
    int sub_powers = 1;
    index_t n_rows = 0;
    std::size_t cache_bytes = 0;
    std::size_t target_bytes = 0;
    std::vector<index_t> group_rows;
    std::vector<index_t> group_level_ptr;
    std::vector<std::size_t> group_footprint;
    std::vector<index_t> level_ptr;  // optional: level offsets of the structure it was built on

    index_t n_groups() const {
        return group_rows.empty() ? 0 : static_cast<index_t>(group_rows.size() - 1);
    }
    void invalidate() const { dev_.reset(); }

    mpkg_plan_t device() const {
        if (!dev_) {
            auto d = std::make_shared<detail::PlanHolder>();
            std::vector<std::uint64_t> fp(group_footprint.begin(), group_footprint.end());
            detail::check(mpkg_plan_create(
                p_m, sub_powers, n_rows, cache_bytes, target_bytes, n_groups(),
                group_rows.empty() ? nullptr : group_rows.data(),
                group_level_ptr.empty() ? nullptr : group_level_ptr.data(),
                fp.empty() ? nullptr : fp.data(),
                level_ptr.empty() ? 0u : static_cast<index_t>(level_ptr.size() - 1),
                level_ptr.empty() ? nullptr : level_ptr.data(), &d->h));
            dev_ = d;
        }
        return dev_->h;
    }

   private:
    mutable std::shared_ptr<detail::PlanHolder> dev_;
};

/// vector_block.hpp:38-57
struct VectorBlock {
    std::size_t rows = 0;
    std::size_t slices = 0;
    std::vector<double> data;

    VectorBlock() = default;
    VectorBlock(std::size_t rows_, std::size_t slices_)
        : rows(rows_), slices(slices_), data(rows_ * slices_, 0.0) {}

    double* slice(std::size_t p) {
        if (p >= slices) throw std::out_of_range("VectorBlock::slice");
        return data.data() + p * rows;
    }
    const double* slice(std::size_t p) const {
        if (p >= slices) throw std::out_of_range("VectorBlock::slice");
        return data.data() + p * rows;
    }
    void zero() { std::fill(data.begin(), data.end(), 0.0); }
};

// ---- csr.hpp ---------------------------------------------------------------------------------
/// csr.hpp:72-110 (host construction helper: stable sort by (row, col), duplicates summed in
/// input order, starting from 0.0).
inline CsrMatrix from_coo(index_t n_rows, index_t n_cols, std::vector<Triplet> entries) {
    if (entries.size() >= (std::size_t{1} << 31))
        throw std::invalid_argument("from_coo: entry count exceeds 32-bit index range");
    for (const Triplet& t : entries)
        if (t.row >= n_rows || t.col >= n_cols)
            throw std::invalid_argument("from_coo: entry index out of range");
    std::vector<std::size_t> idx(entries.size());
    for (std::size_t i = 0; i < idx.size(); ++i) idx[i] = i;
    std::stable_sort(idx.begin(), idx.end(), [&](std::size_t a, std::size_t b) {
        return entries[a].row != entries[b].row ? entries[a].row < entries[b].row
                                                : entries[a].col < entries[b].col;
    });
    CsrMatrix A;
    A.n_rows = n_rows;
    A.n_cols = n_cols;
    A.row_ptr.assign(static_cast<std::size_t>(n_rows) + 1, 0);
    for (std::size_t i = 0; i < idx.size();) {
        const index_t r = entries[idx[i]].row, c = entries[idx[i]].col;
        double sum = 0.0;
        for (; i < idx.size() && entries[idx[i]].row == r && entries[idx[i]].col == c; ++i)
            sum += entries[idx[i]].val;
        A.col_idx.push_back(c);
        A.values.push_back(sum);
        A.row_ptr[r + 1] = static_cast<index_t>(A.col_idx.size());
    }
    for (index_t r = 0; r < n_rows; ++r) A.row_ptr[r + 1] = std::max(A.row_ptr[r + 1], A.row_ptr[r]);
    return A;
}

/// csr.hpp:126-142
inline void spmv(const CsrMatrix& A, const std::vector<double>& x, std::vector<double>& y,
                 int /*threads*/ = 0) {
    if (x.size() != A.n_cols || y.size() != A.n_rows)
        throw std::invalid_argument("spmv: vector size mismatch");
    detail::check(mpkg_spmv(device_context(), A.device(), x.data(), y.data()));
}

/// csr.hpp:207-227 transpose (host; the level engine forms the union pattern on the GPU without
/// it).  Counting pass per column, then rows of A are walked in order, so every row of the
/// result lists its columns (= rows of A) ascending.
inline CsrMatrix transpose(const CsrMatrix& A) {
    CsrMatrix T;
    T.n_rows = A.n_cols;
    T.n_cols = A.n_rows;
    T.row_ptr.assign(static_cast<std::size_t>(A.n_cols) + 1, 0);
    const index_t nz = A.nnz();
    for (index_t k = 0; k < nz; ++k) ++T.row_ptr[static_cast<std::size_t>(A.col_idx[k]) + 1];
    for (std::size_t i = 1; i < T.row_ptr.size(); ++i) T.row_ptr[i] += T.row_ptr[i - 1];
    T.col_idx.resize(nz);
    T.values.resize(nz);
    std::vector<index_t> next(T.row_ptr.begin(), T.row_ptr.end() - 1);
    for (index_t r = 0; r < A.n_rows; ++r)
        for (index_t k = A.row_ptr[r]; k < A.row_ptr[r + 1]; ++k) {
            const index_t dst = next[A.col_idx[k]]++;
            T.col_idx[dst] = r;
            T.values[dst] = A.values[k];
        }
    return T;
}

/// threading.hpp:34-46 resolve_threads: explicit request > MPK_NUM_THREADS > hardware
/// concurrency, >= 1.  Kept for reference call sites that report the team size; the GPU path
/// has no thread team and ignores every `threads` argument.
inline int resolve_threads(int requested = 0) {
    if (requested > 0) return requested;
    if (const char* env = std::getenv("MPK_NUM_THREADS")) {
        char* end = nullptr;
        const long v = std::strtol(env, &end, 10);
        if (end != env && v > 0 && v < (1L << 30)) return static_cast<int>(v);
    }
    const unsigned hw = std::thread::hardware_concurrency();
    return hw ? static_cast<int>(hw) : 1;
}

inline CsrMatrix download(mpkg_csr_t h) {
    CsrMatrix B;
    index_t nnz = 0;
    detail::check(mpkg_csr_info(h, &B.n_rows, &B.n_cols, &nnz));
    B.row_ptr.resize(static_cast<std::size_t>(B.n_rows) + 1);
    B.col_idx.resize(nnz);
    B.values.resize(nnz);
    detail::check(mpkg_csr_download(h, B.row_ptr.data(), B.col_idx.data(), B.values.data()));
    return B;
}

/// matrix_market.hpp:48-113 read_matrix_market: the reference's format rules and messages
/// (std::runtime_error); text parsed on the host, assembled by the GPU from_coo.
inline CsrMatrix read_matrix_market(const std::string& path) {
    mpkg_csr_t h = nullptr;
    detail::check(mpkg_read_matrix_market(device_context(), path.c_str(), &h));
    detail::CsrHolder guard;
    guard.h = h;
    return download(h);
}

/// csr.hpp:159-188 (GPU permutation, bit-exact)
inline CsrMatrix permute(const CsrMatrix& A, const std::vector<index_t>& perm) {
    if (A.n_rows != A.n_cols) throw std::invalid_argument("permute: matrix must be square");
    if (perm.size() != A.n_rows) throw std::invalid_argument("permute: permutation size mismatch");
    mpkg_csr_t out = nullptr;
    detail::check(mpkg_permute(device_context(), A.device(), perm.data(), &out));
    CsrMatrix B = download(out);
    mpkg_csr_destroy(out);
    return B;
}

/// csr.hpp:191-204
inline std::vector<double> permute_vector(const std::vector<double>& in,
                                          const std::vector<index_t>& perm) {
    std::vector<double> out(in.size());
    detail::check(mpkg_permute_vector(device_context(), static_cast<std::uint32_t>(in.size()),
                                      in.data(), perm.data(), out.data()));
    return out;
}
inline std::vector<double> unpermute_vector(const std::vector<double>& in,
                                            const std::vector<index_t>& perm) {
    std::vector<double> out(in.size());
    detail::check(mpkg_unpermute_vector(device_context(), static_cast<std::uint32_t>(in.size()),
                                        in.data(), perm.data(), out.data()));
    return out;
}

// ---- levels.hpp ------------------------------------------------------------------------------
/// levels.hpp:65-147 (GPU BFS, bit-exact)
inline LevelStructure build_levels(const CsrMatrix& A) {
    if (A.n_rows != A.n_cols) throw std::invalid_argument("build_levels: matrix must be square");
    auto d = std::make_shared<detail::LevelsHolder>();
    detail::check(mpkg_build_levels(device_context(), A.device(), &d->h));
    LevelStructure ls;
    index_t n = 0, nl = 0;
    detail::check(mpkg_levels_info(d->h, &n, &nl));
    ls.n_rows = n;
    ls.levels.resize(n);
    ls.perm.resize(n);
    ls.inv_perm.resize(n);
    ls.level_ptr.resize(static_cast<std::size_t>(nl) + 1);
    detail::check(mpkg_levels_get(d->h, ls.levels.data(), ls.perm.data(), ls.inv_perm.data(),
                                  ls.level_ptr.data()));
    ls.dev_ = d;
    return ls;
}

/// levels.hpp:151-164
inline bool validate_levels(const CsrMatrix& A_perm, const LevelStructure& ls) {
    if (A_perm.n_rows != ls.n_rows || A_perm.n_rows != A_perm.n_cols) return false;
    int ok = 0;
    detail::check(mpkg_validate_levels(device_context(), A_perm.device(), ls.device(), &ok));
    return ok != 0;
}

// ---- plan.hpp --------------------------------------------------------------------------------
/// plan.hpp:59-64
inline std::size_t row_range_footprint(const CsrMatrix& A_perm, index_t row_s, index_t row_e,
                                       int p_m) {
    const std::size_t nnz = A_perm.row_ptr[row_e] - A_perm.row_ptr[row_s];
    const std::size_t rows = row_e - row_s;
    return 12 * nnz + 4 * rows + 8 * static_cast<std::size_t>(p_m + 1) * rows;
}

/// plan.hpp:70-85
inline std::vector<index_t> greedy_group(const std::vector<std::size_t>& level_fp,
                                         std::size_t target) {
    std::vector<std::uint64_t> fp(level_fp.begin(), level_fp.end());
    std::vector<index_t> bounds(level_fp.size() + 1);
    index_t nb = 0;
    detail::check(mpkg_greedy_group(fp.empty() ? nullptr : fp.data(),
                                    static_cast<index_t>(fp.size()), target, bounds.data(), &nb));
    bounds.resize(nb);
    return bounds;
}

/// plan.hpp:88-115
inline ExecutionPlan group_levels(const LevelStructure& ls, const CsrMatrix& A_perm,
                                  std::size_t cache_bytes, int p_m) {
    mpkg_plan_t h = nullptr;
    detail::check(mpkg_group_levels(device_context(), ls.device(), A_perm.device(), cache_bytes,
                                    p_m, &h));
    ExecutionPlan plan;
    index_t n = 0, ng = 0;
    std::uint64_t cb = 0, tb = 0;
    detail::check(mpkg_plan_info(h, &plan.p_m, &plan.sub_powers, &n, &cb, &tb, &ng));
    plan.n_rows = n;
    plan.cache_bytes = cb;
    plan.target_bytes = tb;
    plan.group_rows.resize(static_cast<std::size_t>(ng) + 1);
    plan.group_level_ptr.resize(static_cast<std::size_t>(ng) + 1);
    std::vector<std::uint64_t> fp(ng);
    detail::check(mpkg_plan_get(h, plan.group_rows.data(), plan.group_level_ptr.data(),
                                fp.empty() ? nullptr : fp.data()));
    mpkg_plan_destroy(h);
    plan.group_footprint.assign(fp.begin(), fp.end());
    plan.level_ptr = ls.level_ptr;
    return plan;
}

// ---- execute.hpp -----------------------------------------------------------------------------
/// execute.hpp:52-55
struct ScheduleCell {
    index_t group;
    int stage;
};

/// execute.hpp:59-72
inline std::vector<ScheduleCell> wavefront_schedule(index_t n_groups, int stages) {
    std::uint64_t cnt = 0;
    const std::size_t cap = stages > 0 ? static_cast<std::size_t>(n_groups) * stages : 0;
    std::vector<index_t> g(cap + 1);
    std::vector<int> q(cap + 1);
    detail::check(mpkg_wavefront_schedule(n_groups, stages, g.data(), q.data(), &cnt));
    std::vector<ScheduleCell> out(cnt);
    for (std::size_t i = 0; i < cnt; ++i) out[i] = {g[i], q[i]};
    return out;
}

/// execute.hpp:79-113 — generic host callback hook (host-side; see the header comment).
template <typename Kernel>
void execute(const ExecutionPlan& plan, Kernel&& kernel, int /*threads*/ = 0, int p_m = 0) {
    if (p_m <= 0) p_m = plan.p_m;
    if (p_m > plan.p_m) throw std::invalid_argument("execute: p_m exceeds the plan's power budget");
    const int sub = plan.sub_powers;
    for (const ScheduleCell& cell : wavefront_schedule(plan.n_groups(), p_m * sub)) {
        const index_t rs = plan.group_rows[cell.group], re = plan.group_rows[cell.group + 1];
        if (re > rs) kernel(rs, re, (cell.stage - 1) / sub + 1, (cell.stage - 1) % sub);
    }
}

// ---- mpk.hpp ---------------------------------------------------------------------------------
/// mpk.hpp:59-75
inline void baseline_mpk(const CsrMatrix& A, const std::vector<double>& x, int p_m,
                         VectorBlock& block, int /*threads*/ = 0) {
    if (x.size() != A.n_rows) throw std::invalid_argument("baseline_mpk: input size mismatch");
    detail::check(mpkg_baseline_mpk(device_context(), A.device(), x.data(), p_m,
                                    block.data.data(), block.rows, block.slices));
}

/// mpk.hpp:81-106 (GPU executor: one launch per power, or the fused tile-DAG kernel for
/// matrices with long rows)
inline void mpk(const ExecutionPlan& plan, const CsrMatrix& A_perm, const std::vector<double>& x,
                int p_m, VectorBlock& block, int /*threads*/ = 0) {
    if (x.size() != A_perm.n_rows) throw std::invalid_argument("mpk: input size mismatch");
    detail::check(mpkg_mpk(device_context(), plan.device(), A_perm.device(), x.data(), p_m,
                           block.data.data(), block.rows, block.slices));
}

/// mpk.hpp:111-127
inline void check_shift_chain(const std::vector<std::complex<double>>& shifts, const char* who) {
    std::vector<double> re(shifts.size()), im(shifts.size());
    for (std::size_t i = 0; i < shifts.size(); ++i) re[i] = shifts[i].real(), im[i] = shifts[i].imag();
    const int rc = mpkg_check_shift_chain(re.data(), im.data(), static_cast<int>(shifts.size()));
    if (rc == MPKG_EINVAL) throw std::invalid_argument(std::string(who) + ": " + mpkg_last_error());
    detail::check(rc);
}

namespace detail {
inline void split(const std::vector<std::complex<double>>& s, std::vector<double>& re,
                  std::vector<double>& im) {
    re.resize(s.size());
    im.resize(s.size());
    for (std::size_t i = 0; i < s.size(); ++i) re[i] = s[i].real(), im[i] = s[i].imag();
}
}  // namespace detail

/// mpk.hpp:160-180
inline void baseline_mpk_shifted(const CsrMatrix& A, const std::vector<double>& x,
                                 const std::vector<std::complex<double>>& shifts,
                                 VectorBlock& block, int /*threads*/ = 0) {
    if (x.size() != A.n_rows) throw std::invalid_argument("baseline_mpk_shifted: input size mismatch");
    std::vector<double> re, im;
    detail::split(shifts, re, im);
    detail::check(mpkg_baseline_mpk_shifted(device_context(), A.device(), x.data(), re.data(),
                                            im.data(), static_cast<int>(shifts.size()),
                                            block.data.data(), block.rows, block.slices));
}

/// mpk.hpp:184-207
inline void mpk_shifted(const ExecutionPlan& plan, const CsrMatrix& A_perm,
                        const std::vector<double>& x,
                        const std::vector<std::complex<double>>& shifts, VectorBlock& block,
                        int /*threads*/ = 0) {
    if (x.size() != A_perm.n_rows) throw std::invalid_argument("mpk_shifted: input size mismatch");
    std::vector<double> re, im;
    detail::split(shifts, re, im);
    detail::check(mpkg_mpk_shifted(device_context(), plan.device(), A_perm.device(), x.data(),
                                   re.data(), im.data(), static_cast<int>(shifts.size()),
                                   block.data.data(), block.rows, block.slices));
}

/// Coefficient-form polynomial z = sum_k c_k A^k x (not in the reference).
inline std::vector<double> mpk_poly(const ExecutionPlan& plan, const CsrMatrix& A_perm,
                                    const std::vector<double>& x, const std::vector<double>& c) {
    std::vector<double> z(A_perm.n_rows);
    detail::check(mpkg_mpk_poly(device_context(), plan.device(), A_perm.device(), x.data(),
                                c.data(), static_cast<int>(c.size()) - 1, z.data(), nullptr, 0, 0));
    return z;
}

// ---- jacobi.hpp / csr.hpp:231-243 -----------------------------------------
/// csr.hpp:231
inline constexpr index_t kNoDiag = 0xffffffffu;

/// csr.hpp:233-243 (host)
inline std::vector<index_t> diagonal_positions(const CsrMatrix& A) {
    std::vector<index_t> pos(A.n_rows, kNoDiag);
    for (index_t r = 0; r < A.n_rows && r < A.n_cols; ++r) {
        const auto b = A.col_idx.begin() + A.row_ptr[r], e = A.col_idx.begin() + A.row_ptr[r + 1];
        const auto it = std::lower_bound(b, e, r);
        if (it != e && *it == r) pos[r] = static_cast<index_t>(it - A.col_idx.begin());
    }
    return pos;
}

/// jacobi.hpp:41-44
struct DiagInfo {
    std::vector<index_t> pos;
    std::vector<double> inv;
};

/// jacobi.hpp:66-69; the diagonal data also lives on the device (built by jacobi_setup).
struct JacobiPrecon {
    DiagInfo diag;
    int sweeps = 1;
    mpkg_jacobi_t device() const {
        if (!dev_) throw std::invalid_argument("JacobiPrecon: not built by jacobi_setup");
        return dev_->h;
    }
    std::shared_ptr<detail::JacobiHolder> dev_;
};

/// jacobi.hpp:71-75 (+ build_diag_info 48-64): std::invalid_argument / std::runtime_error.
inline JacobiPrecon jacobi_setup(const CsrMatrix& a, int sweeps = 1) {
    JacobiPrecon p;
    p.sweeps = sweeps;
    auto d = std::make_shared<detail::JacobiHolder>();
    detail::check(mpkg_jacobi_setup(device_context(), a.device(), sweeps, &d->h));
    p.diag.pos.resize(a.n_rows);
    p.diag.inv.resize(a.n_rows);
    detail::check(mpkg_jacobi_get(d->h, p.diag.pos.data(), p.diag.inv.data()));
    p.dev_ = d;
    return p;
}

/// jacobi.hpp:155-174
inline void jacobi_apply(const JacobiPrecon& p, const CsrMatrix& a, const std::vector<double>& v,
                         std::vector<double>& z, int /*threads*/ = 0) {
    if (v.size() != a.n_rows) throw std::invalid_argument("jacobi_apply: size mismatch");
    z.resize(a.n_rows);
    detail::check(mpkg_jacobi_apply(device_context(), p.device(), a.device(), v.data(), z.data()));
}

/// jacobi.hpp:177-192
inline void jacobi_op(const JacobiPrecon& p, const CsrMatrix& a, const std::vector<double>& v,
                      std::vector<double>& y, int /*threads*/ = 0) {
    if (v.size() != a.n_rows) throw std::invalid_argument("jacobi_op: size mismatch");
    y.resize(a.n_rows);
    detail::check(mpkg_jacobi_op(device_context(), p.device(), a.device(), v.data(), y.data()));
}

/// jacobi.hpp:196-209 (plan.sub_powers must be JacobiOpChain::stages(sweeps))
inline void jacobi_op_blocked(const JacobiPrecon& p, const CsrMatrix& a_perm,
                              const ExecutionPlan& plan, const std::vector<double>& v,
                              std::vector<double>& y, int /*threads*/ = 0) {
    if (v.size() != a_perm.n_rows) throw std::invalid_argument("jacobi_op_blocked: size mismatch");
    y.resize(a_perm.n_rows);
    detail::check(mpkg_jacobi_op_blocked(device_context(), p.device(), plan.device(), a_perm.device(),
                                         v.data(), y.data()));
}

/// jacobi.hpp:129 JacobiOpChain::stages
inline int jacobi_stages(int sweeps) { return sweeps == 1 ? 1 : sweeps + 1; }

/// sstep.hpp:356-385 sstep_generate_block, Jacobi case: w.slice(0) holds the start vector on
/// entry; slices 1..shifts.size() receive the Jacobi-preconditioned Newton basis.  `plan` may
/// be null (sequential form) or carry sub_powers == jacobi_stages(sweeps).
inline void sstep_jacobi_block(const JacobiPrecon& p, const CsrMatrix& a,
                               const std::vector<std::complex<double>>& shifts, VectorBlock& w,
                               const ExecutionPlan* plan = nullptr) {
    std::vector<double> re, im;
    detail::split(shifts, re, im);
    detail::check(mpkg_sstep_jacobi(device_context(), p.device(), plan ? plan->device() : nullptr,
                                    a.device(), re.data(), im.data(), static_cast<int>(shifts.size()),
                                    w.data.data(), w.rows, w.slices));
}

// ---- gs2.hpp ---------------------------------------------------------------
/// gs2.hpp:44
enum class SweepDirection { forward, backward };

/// gs2.hpp:47-53; the diagonal data also lives on the device (built by gs2_setup).
struct Gs2Precon {
    DiagInfo diag;
    int gamma = 1;
    int sweeps = 1;
    SweepDirection direction = SweepDirection::forward;
    mpkg_gs2_t device() const {
        if (!dev_) throw std::invalid_argument("Gs2Precon: not built by gs2_setup");
        return dev_->h;
    }
    std::shared_ptr<detail::Gs2Holder> dev_;
};

/// gs2.hpp:55-62
inline Gs2Precon gs2_setup(const CsrMatrix& a, int gamma, int sweeps = 1,
                           SweepDirection direction = SweepDirection::forward) {
    Gs2Precon p;
    p.gamma = gamma, p.sweeps = sweeps, p.direction = direction;
    auto d = std::make_shared<detail::Gs2Holder>();
    detail::check(mpkg_gs2_setup(device_context(), a.device(), gamma, sweeps,
                                 direction == SweepDirection::forward ? 0 : 1, &d->h));
    p.diag.pos.resize(a.n_rows);
    p.diag.inv.resize(a.n_rows);
    detail::check(mpkg_gs2_get(d->h, p.diag.pos.data(), p.diag.inv.data()));
    p.dev_ = d;
    return p;
}

namespace detail {
inline void gs2_sizes(const CsrMatrix& a, const std::vector<double>& v, const std::vector<double>* z) {
    if (a.n_rows != a.n_cols) throw std::invalid_argument("gs2: matrix must be square");
    if (v.size() != a.n_rows || (z && z->size() != a.n_rows))
        throw std::invalid_argument("gs2: size mismatch");
}
}  // namespace detail

/// gs2.hpp:200-204
inline void gs2_smooth(const Gs2Precon& p, const CsrMatrix& a, const std::vector<double>& v,
                       std::vector<double>& z, int /*threads*/ = 0) {
    detail::gs2_sizes(a, v, &z);
    detail::check(mpkg_gs2_smooth(device_context(), p.device(), nullptr, a.device(), v.data(), z.data()));
}
/// gs2.hpp:207-212
inline void gs2_apply(const Gs2Precon& p, const CsrMatrix& a, const std::vector<double>& v,
                      std::vector<double>& z, int /*threads*/ = 0) {
    detail::gs2_sizes(a, v, nullptr);
    z.assign(a.n_rows, 0.0);
    detail::check(mpkg_gs2_apply(device_context(), p.device(), nullptr, a.device(), v.data(), z.data()));
}
/// gs2.hpp:215-220
inline void gs2_smooth_residual(const Gs2Precon& p, const CsrMatrix& a, const std::vector<double>& v,
                                std::vector<double>& z, std::vector<double>& r, int /*threads*/ = 0) {
    detail::gs2_sizes(a, v, &z);
    r.resize(a.n_rows);
    detail::check(mpkg_gs2_smooth_residual(device_context(), p.device(), nullptr, a.device(), v.data(),
                                           z.data(), r.data()));
}
/// gs2.hpp:223-228
inline void gs2_op(const Gs2Precon& p, const CsrMatrix& a, const std::vector<double>& v,
                   std::vector<double>& y, int /*threads*/ = 0) {
    detail::gs2_sizes(a, v, nullptr);
    y.resize(a.n_rows);
    detail::check(mpkg_gs2_op(device_context(), p.device(), nullptr, a.device(), v.data(), y.data()));
}
/// gs2.hpp:233-275 cache-blocked twins (plan: sub_powers == gamma + 2, budget >= sweeps)
inline void gs2_smooth_blocked(const Gs2Precon& p, const CsrMatrix& a_perm, const ExecutionPlan& plan,
                               const std::vector<double>& v, std::vector<double>& z, int /*threads*/ = 0) {
    detail::gs2_sizes(a_perm, v, &z);
    detail::check(mpkg_gs2_smooth(device_context(), p.device(), plan.device(), a_perm.device(), v.data(),
                                  z.data()));
}
inline void gs2_apply_blocked(const Gs2Precon& p, const CsrMatrix& a_perm, const ExecutionPlan& plan,
                              const std::vector<double>& v, std::vector<double>& z, int /*threads*/ = 0) {
    detail::gs2_sizes(a_perm, v, nullptr);
    z.assign(a_perm.n_rows, 0.0);
    detail::check(mpkg_gs2_apply(device_context(), p.device(), plan.device(), a_perm.device(), v.data(),
                                 z.data()));
}
inline void gs2_smooth_residual_blocked(const Gs2Precon& p, const CsrMatrix& a_perm,
                                        const ExecutionPlan& plan, const std::vector<double>& v,
                                        std::vector<double>& z, std::vector<double>& r,
                                        int /*threads*/ = 0) {
    detail::gs2_sizes(a_perm, v, &z);
    r.resize(a_perm.n_rows);
    detail::check(mpkg_gs2_smooth_residual(device_context(), p.device(), plan.device(), a_perm.device(),
                                           v.data(), z.data(), r.data()));
}
inline void gs2_op_blocked(const Gs2Precon& p, const CsrMatrix& a_perm, const ExecutionPlan& plan,
                           const std::vector<double>& v, std::vector<double>& y, int /*threads*/ = 0) {
    detail::gs2_sizes(a_perm, v, nullptr);
    y.resize(a_perm.n_rows);
    detail::check(mpkg_gs2_op(device_context(), p.device(), plan.device(), a_perm.device(), v.data(),
                              y.data()));
}

/// sstep.hpp:356-398 sstep_generate_block, GS2 case (see sstep_jacobi_block).
inline void sstep_gs2_block(const Gs2Precon& p, const CsrMatrix& a,
                            const std::vector<std::complex<double>>& shifts, VectorBlock& w,
                            const ExecutionPlan* plan = nullptr) {
    std::vector<double> re, im;
    detail::split(shifts, re, im);
    detail::check(mpkg_sstep_gs2(device_context(), p.device(), plan ? plan->device() : nullptr,
                                 a.device(), re.data(), im.data(), static_cast<int>(shifts.size()),
                                 w.data.data(), w.rows, w.slices));
}

// ---- poly.hpp ---------------------------------------------------------------
/// poly.hpp:55-61
struct PolyInner {
    enum class Kind { none, jacobi, gs2 };
    Kind kind = Kind::none;
    JacobiPrecon jacobi;
    Gs2Precon gs2;
};

/// poly.hpp:64-70: the roots (Leja-ordered, conjugate pairs adjacent) are the caller's -- the
/// reference computes them with an Eigen-based Arnoldi / harmonic-Ritz setup (poly_setup_gmres)
/// that this library does not provide.
struct PolyPrecon {
    std::vector<std::complex<double>> theta;
    int degree = 0;
    bool truncated = false;
    PolyInner inner;
};

namespace detail {
inline void poly_call(const PolyPrecon& p, const CsrMatrix& a, const ExecutionPlan* plan,
                      const std::vector<double>& v, std::vector<double>& z) {
    if (v.size() != a.n_rows) throw std::invalid_argument("poly_apply: size mismatch");
    if (p.degree < 1 || p.theta.size() != static_cast<std::size_t>(p.degree))
        throw std::invalid_argument("poly_apply: preconditioner not set up");
    std::vector<double> re, im;
    split(p.theta, re, im);
    z.assign(a.n_rows, 0.0);
    check(mpkg_poly_apply(device_context(), a.device(),
                          p.inner.kind == PolyInner::Kind::jacobi ? p.inner.jacobi.device() : nullptr,
                          p.inner.kind == PolyInner::Kind::gs2 ? p.inner.gs2.device() : nullptr,
                          re.data(), im.data(), p.degree, plan ? plan->device() : nullptr, v.data(),
                          z.data()));
}
}  // namespace detail

/// poly.hpp:364-373 z = p(A M^{-1}) v, sequential form
inline void poly_apply(const PolyPrecon& p, const CsrMatrix& a, const std::vector<double>& v,
                       std::vector<double>& z, int /*threads*/ = 0) {
    detail::poly_call(p, a, nullptr, v, z);
}
/// poly.hpp:375-380 cache-blocked twin (plan.sub_powers == poly_sub_powers(p))
inline void poly_apply_blocked(const PolyPrecon& p, const CsrMatrix& a_perm, const ExecutionPlan& plan,
                               const std::vector<double>& v, std::vector<double>& z, int /*threads*/ = 0) {
    detail::poly_call(p, a_perm, &plan, v, z);
}
/// poly.hpp:383-385
inline int poly_sub_powers(const PolyPrecon& p) {
    switch (p.inner.kind) {
        case PolyInner::Kind::jacobi: return jacobi_stages(p.inner.jacobi.sweeps);
        case PolyInner::Kind::gs2: return p.inner.gs2.gamma + 2;
        default: return 1;
    }
}

/// mpk.hpp:211-215
struct TuneResult {
    int p_opt = 1;
    std::vector<std::pair<int, double>> table;
};

/// mpk.hpp:219-233
template <typename TrialFn>
TuneResult tune_p(int p_lo, int p_hi, TrialFn&& trial) {
    if (p_lo < 1 || p_hi < p_lo) throw std::invalid_argument("tune_p: bad range");
    TuneResult res;
    std::vector<double> t;
    for (int p = p_lo; p <= p_hi; ++p) {
        t.push_back(trial(p));
        res.table.emplace_back(p, t.back());
    }
    detail::check(mpkg_tune_select(t.data(), p_lo, p_hi, &res.p_opt));
    return res;
}

/// mpk.hpp:238-258 (GPU timing with CUDA events)
// ---- block orthogonalisation (ortho.hpp) -------------------------------
// Same signatures as the reference (column-major blocks, leading dimension rows).  `threads` is
// accepted for drop-in compatibility; the device decides its own parallelism.  block_dots is
// bit-identical to the reference in MPKG_MODE_BITWISE (the default); block_update always.

// ortho.hpp:46-63
inline void block_dots(const double* q, const double* v, std::size_t rows, std::size_t qcols,
                       std::size_t vcols, double* c, int threads = 0) {
    (void)threads;
    detail::check(mpkg_block_dots(device_context(), q, v, rows, static_cast<std::uint32_t>(qcols),
                          static_cast<std::uint32_t>(vcols), c));
}

// ortho.hpp:67-92
inline void block_update(const double* q, const double* c, std::size_t rows, std::size_t qcols,
                         std::size_t vcols, double* v, int threads = 0) {
    (void)threads;
    detail::check(mpkg_block_update(device_context(), q, c, rows, static_cast<std::uint32_t>(qcols),
                            static_cast<std::uint32_t>(vcols), v));
}

// ortho.hpp:97-117
inline std::vector<double> icgs_block_orthogonalize(const double* q, std::size_t rows,
                                                    std::size_t qcols, double* v,
                                                    std::size_t vcols, int sweeps,
                                                    int threads = 0) {
    (void)threads;
    std::vector<double> coeff(qcols * vcols, 0.0);
    detail::check(mpkg_icgs_block_orthogonalize(device_context(), q, rows, static_cast<std::uint32_t>(qcols),
                                        v, static_cast<std::uint32_t>(vcols), sweeps,
                                        coeff.empty() ? nullptr : coeff.data()));
    return coeff;
}

// ortho.hpp:136-229.  panel_rows is accepted for compatibility: the device sizes its panels to
// shared memory; (Q, R) with a non-negative R diagonal is unique, so the result agrees with any
// panel tree to roundoff.
inline void tsqr(double* v, std::size_t rows, std::size_t cols, double* r,
                 std::size_t panel_rows = 4096, int threads = 0) {
    (void)panel_rows, (void)threads;
    detail::check(mpkg_tsqr(device_context(), v, rows, static_cast<std::uint32_t>(cols), r));
}

// sstep.hpp:539-545 in one call (extension): icgs_block_orthogonalize(q, rows, qcols, v, vcols,
// sweeps) then tsqr(v, rows, vcols, r); returns the ICGS coefficients.  Bit-identical to the two
// calls; for s-step blocks the last update is fused into the TSQR factor and never stored.
inline std::vector<double> ortho_block(const double* q, std::size_t rows, std::size_t qcols, double* v,
                                       std::size_t vcols, int sweeps, double* r, int threads = 0) {
    (void)threads;
    std::vector<double> coeff(qcols * vcols, 0.0);
    detail::check(mpkg_ortho_block(device_context(), q, rows, static_cast<std::uint32_t>(qcols), v,
                                   static_cast<std::uint32_t>(vcols), sweeps, coeff.data(), r));
    return coeff;
}

// ortho.hpp:231-240
inline bool tsqr_rank_deficient(const double* r, std::size_t cols, double threshold) {
    for (std::size_t j = 0; j < cols; ++j)
        if (std::abs(r[j * cols + j]) < threshold) return true;
    return false;
}

inline TuneResult tune_p(const LevelStructure& ls, const CsrMatrix& A_perm,
                         std::size_t cache_bytes, int p_lo, int p_hi, int /*threads*/ = 0,
                         int reps = 3) {
    if (p_lo < 1 || p_hi < p_lo) throw std::invalid_argument("tune_p: bad range");
    std::vector<double> t(static_cast<std::size_t>(p_hi - p_lo + 1));
    TuneResult res;
    detail::check(mpkg_tune_p(device_context(), ls.device(), A_perm.device(), cache_bytes, p_lo,
                              p_hi, reps, &res.p_opt, t.data()));
    for (int p = p_lo; p <= p_hi; ++p) res.table.emplace_back(p, t[p - p_lo]);
    return res;
}

// ---- generators.hpp (harness inputs, produced by the library's host generators) -------------
namespace detail {
inline CsrMatrix gen(int kind, index_t a, index_t b, index_t c, std::uint64_t seed) {
    mpkg_host_csr_t h = nullptr;
    check(mpkg_gen(kind, a, b, c, seed, &h));
    index_t n = 0, m = 0;
    std::uint64_t nnz = 0;
    check(mpkg_host_csr_info(h, &n, &m, &nnz));
    index_t *rp = nullptr, *ci = nullptr;
    double* v = nullptr;
    check(mpkg_host_csr_arrays(h, &rp, &ci, &v));
    CsrMatrix A;
    A.n_rows = n;
    A.n_cols = m;
    A.row_ptr.assign(rp, rp + n + 1);
    A.col_idx.assign(ci, ci + nnz);
    A.values.assign(v, v + nnz);
    mpkg_host_csr_destroy(h);
    return A;
}
}  // namespace detail

inline CsrMatrix poisson1d(index_t n) { return detail::gen(1, n, 0, 0, 0); }
inline CsrMatrix poisson2d(index_t nx, index_t ny) { return detail::gen(2, nx, ny, 0, 0); }
inline CsrMatrix poisson3d(index_t nx, index_t ny, index_t nz) { return detail::gen(3, nx, ny, nz, 0); }
inline CsrMatrix random_csr(index_t n, index_t k, std::uint64_t seed) { return detail::gen(4, n, k, 0, seed); }
inline CsrMatrix random_spd(index_t n, index_t k, std::uint64_t seed) { return detail::gen(5, n, k, 0, seed); }

}  // namespace mpkg
