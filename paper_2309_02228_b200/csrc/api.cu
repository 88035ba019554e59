// The mpkg C ABI (include/mpkg.h): argument validation with the reference's error semantics,
// host<->device staging, and dispatch to the sm_100a kernels.  No CPU fallback exists: every
// compute entry point runs on the GPU or fails with MPKG_ECUDA.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <vector>

#include "device.h"

namespace mpkg_detail {
int g_sm_count = 0;
}

using namespace mpkg_detail;

namespace mpkg_detail {

namespace {
thread_local std::string g_last_error;
}

void set_error(const char* fmt, ...) {
    char buf[1024];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    g_last_error = buf;
}

std::pair<cudaEvent_t, cudaEvent_t> timing_begin(mpkg_ctx_s* ctx) {
    if (!ctx->kernel_timing) return {nullptr, nullptr};
    std::pair<cudaEvent_t, cudaEvent_t> ev;
    if (ctx->event_pool.empty()) {
        // grow in batches: event creation costs microseconds of host time, which launch-bound
        // calls (C1) would otherwise pay inside the timed region
        for (int i = 0; i < 64; ++i) {
            MPKG_CUDA(cudaEventCreate(&ev.first));
            MPKG_CUDA(cudaEventCreate(&ev.second));
            ctx->event_pool.push_back(ev);
        }
    }
    ev = ctx->event_pool.back();
    ctx->event_pool.pop_back();
    MPKG_CUDA(cudaEventRecord(ev.first, ctx->stream));
    return ev;
}

void timing_end(mpkg_ctx_s* ctx, std::pair<cudaEvent_t, cudaEvent_t> ev) {
    if (!ev.first) return;
    MPKG_CUDA(cudaEventRecord(ev.second, ctx->stream));
    ctx->timed.push_back(ev);
}

namespace {

void use_device(mpkg_ctx_s* ctx) { MPKG_CUDA(cudaSetDevice(ctx->device)); }

// csr.hpp:53-56 invariants, checked on the host copy before upload.
void validate_csr_host(uint32_t n_rows, uint32_t n_cols, const uint32_t* rp, const uint32_t* ci) {
    require(rp != nullptr, "csr: null row_ptr");
    require(rp[0] == 0, "csr: row_ptr[0] must be 0");
    require(rp[n_rows] < (1u << 31), "csr: nnz exceeds the 32-bit index range");
    for (uint32_t r = 0; r < n_rows; ++r) {
        require(rp[r] <= rp[r + 1], "csr: row_ptr must be monotone");
        for (uint32_t k = rp[r]; k < rp[r + 1]; ++k) {
            require(ci[k] < n_cols, "csr: column index out of range");
            if (k > rp[r]) require(ci[k - 1] < ci[k], "csr: columns must be strictly ascending");
        }
    }
}

void check_workspace(const mpkg_csr_s* A, int p_m, uint64_t rows, uint64_t slices,
                     const char* who) {
    // mpk.hpp:44-53 check_power_workspace
    require(A->n_rows == A->n_cols, std::string(who) + ": matrix must be square");
    require(p_m >= 1, std::string(who) + ": p_m must be >= 1");
    require(rows == A->n_rows && slices >= (uint64_t)p_m + 1,
            std::string(who) + ": workspace too small");
}

void shift_chain(const double* re, const double* im, int ns, const char* who) {
    // mpk.hpp:111-127 check_shift_chain
    for (int i = 0; i < ns; ++i) {
        const double b = im[i];
        if (b == 0.0) continue;
        if (b < 0.0)
            fail(MPKG_EINVAL, std::string(who) + ": conjugate pair member without its partner");
        if (i + 1 == ns)
            fail(MPKG_EINVAL, std::string(who) + ": conjugate pair straddles the block end");
        if (!(re[i + 1] == re[i] && im[i + 1] == -b))
            fail(MPKG_EINVAL, std::string(who) + ": conjugate pairs must be stored adjacently");
        ++i;
    }
}

void shift_coeffs(const double* re, const double* im, int ns, std::vector<double>& a,
                  std::vector<double>& b2) {
    a.resize(ns);
    b2.resize(ns);
    for (int i = 0; i < ns; ++i) {
        a[i] = re[i];
        b2[i] = im[i] < 0.0 ? im[i] * im[i] : 0.0;  // mpk.hpp:171 / 201
    }
}

// Host-pointer wrapper: stage x, run `body(d_x, d_block)`, copy the block back.
template <class F>
void with_host_block(mpkg_ctx_s* ctx, uint32_t n, const double* x, int p_m, double* block,
                     F&& body) {
    const uint64_t elems = (uint64_t)n * (p_m + 1);
    ctx->scratch_block.ensure(std::max<uint64_t>(elems, 1));
    ctx->scratch_x.ensure(std::max<uint32_t>(n, 1));
    if (n) MPKG_CUDA(cudaMemcpyAsync(ctx->scratch_x.p, x, sizeof(double) * n, cudaMemcpyHostToDevice, ctx->stream));
    body(ctx->scratch_x.p, ctx->scratch_block.p);
    if (elems)
        MPKG_CUDA(cudaMemcpyAsync(block, ctx->scratch_block.p, sizeof(double) * elems,
                                  cudaMemcpyDeviceToHost, ctx->stream));
    MPKG_CUDA(cudaStreamSynchronize(ctx->stream));
}

// Host-pointer mpk: stage x; the executor streams every slice back to the caller's block as it
// completes (run_fused, FusedArgs::host_block); the final sync covers the copies.
// Slice 0 is x itself: the host copies it while the device works (mpk.hpp:62 / 87 semantics).
template <class F>
void host_streamed(mpkg_ctx_s* ctx, uint32_t n, const double* x, int p_m, double* block, F&& body) {
    ctx->scratch_block.ensure(std::max<uint64_t>((uint64_t)n * (p_m + 1), 1));
    ctx->scratch_x.ensure(std::max<uint32_t>(n, 1));
    if (n) MPKG_CUDA(cudaMemcpyAsync(ctx->scratch_x.p, x, sizeof(double) * n, cudaMemcpyHostToDevice, ctx->stream));
    body(ctx->scratch_x.p, ctx->scratch_block.p);
    if (n && block != x) std::memmove(block, x, sizeof(double) * n);
    MPKG_CUDA(cudaStreamSynchronize(ctx->stream));
}

void baseline_dev(mpkg_ctx_s* ctx, mpkg_csr_s* A, const double* d_x, int p_m, double* d_block,
                  uint64_t rows, uint64_t slices, const double* re, const double* im) {
    const char* who = re ? "baseline_mpk_shifted" : "baseline_mpk";
    check_workspace(A, p_m, rows, slices, who);
    if (re) shift_chain(re, im, p_m, who);
    use_device(ctx);
    const uint32_t n = A->n_rows;
    if (n == 0) return;
    MPKG_CUDA(cudaMemcpyAsync(d_block, d_x, sizeof(double) * n, cudaMemcpyDeviceToDevice, ctx->stream));
    Sell& S = csr_sell(A);
    std::vector<double> a, b2;
    if (re) shift_coeffs(re, im, p_m, a, b2);
    for (int p = 1; p <= p_m; ++p) {
        const double* src = d_block + (uint64_t)(p - 1) * n;
        double* dst = d_block + (uint64_t)p * n;
        if (re)
            launch_spmv_sell(ctx, S, true, src, dst, p >= 2 ? d_block + (uint64_t)(p - 2) * n : src,
                             a[p - 1], b2[p - 1]);
        else
            launch_spmv_sell(ctx, S, false, src, dst, nullptr, 0.0, 0.0);
    }
}

void mpk_dev(mpkg_ctx_s* ctx, mpkg_plan_s* P, mpkg_csr_s* A, const double* d_x, int p_m,
             double* d_block, uint64_t rows, uint64_t slices, const double* re, const double* im,
             const double* coef, double* d_z, const char* who, double* host_block = nullptr) {
    require(P != nullptr && A != nullptr, std::string(who) + ": null argument");
    check_workspace(A, p_m, rows, slices, who);
    require(P->n_rows == A->n_rows, std::string(who) + ": plan does not match matrix");
    // execute.hpp:81-83
    require(p_m <= P->p_m, "execute: p_m exceeds the plan's power budget");
    if (re) shift_chain(re, im, p_m, who);
    use_device(ctx);
    const uint32_t n = A->n_rows;
    if (n == 0) return;
    std::vector<double> a, b2;
    if (re) shift_coeffs(re, im, p_m, a, b2);
    // The executor runs at most kFusedSegment powers per call (its launch parameters carry the
    // per-power shifts); longer chains run segment by segment, each starting from the last slice of
    // the previous one -- the same arithmetic, so the same bits.  A segment never starts on the
    // second member of a conjugate pair (its epilogue reads slice q-2).  mpk_poly keeps d <= 32.
    constexpr int kFusedSegment = 32;
    require(!coef || p_m <= kFusedSegment, std::string(who) + ": polynomial degree above 32");
    int done = 0;
    while (done < p_m) {
        int len = std::min(kFusedSegment, p_m - done);
        if (re && done + len < p_m && b2[done + len] != 0.0) --len;
        FusedArgs fa;  // run_fused writes slice 0 = x (mpk.hpp:62) on the first segment
        fa.x = done == 0 ? d_x : d_block + (uint64_t)done * rows;
        fa.kind = re ? 1 : (coef ? 2 : 0);
        fa.p = len;
        fa.block = d_block + (uint64_t)done * rows;
        fa.rows = rows;
        if (re) {
            fa.shift_a = a.data() + done;
            fa.shift_b2 = b2.data() + done;
        }
        fa.coef = coef;
        fa.z = d_z;
        fa.host_block = host_block ? host_block + (uint64_t)done * rows : nullptr;
        run_fused(ctx, P, A, fa);
        done += len;
    }
}

}  // namespace
}  // namespace mpkg_detail

extern "C" {

const char* mpkg_last_error(void) { return mpkg_detail::g_last_error.c_str(); }
int mpkg_abi_version(void) { return MPKG_ABI_VERSION; }

// ---- context ----------------------------------------------------------------------------------
int mpkg_ctx_create(int device, mpkg_ctx_t* out) {
    return guarded([&] {
        require(out != nullptr, "ctx_create: null output");
        int count = 0;
        MPKG_CUDA(cudaGetDeviceCount(&count));
        if (count <= 0) fail(MPKG_ECUDA, "no CUDA device visible (no CPU fallback exists)");
        require(device >= 0 && device < count, "ctx_create: device index out of range");
        MPKG_CUDA(cudaSetDevice(device));
        auto* c = new mpkg_ctx_s();
        c->device = device;
        cudaDeviceProp prop{};
        MPKG_CUDA(cudaGetDeviceProperties(&prop, device));
        if (prop.major < 10) {
            delete c;
            fail(MPKG_ECUDA, "mpkg is built for sm_100a (B200); device is sm_" +
                                 std::to_string(prop.major) + std::to_string(prop.minor));
        }
        c->sm_count = prop.multiProcessorCount;
        g_sm_count = c->sm_count;
        c->l2_bytes = prop.l2CacheSize;
        c->persist_max = prop.persistingL2CacheMaxSize;
        MPKG_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
        *out = c;
    });
}

int mpkg_ctx_destroy(mpkg_ctx_t ctx) {
    if (!ctx) return MPKG_OK;
    cudaSetDevice(ctx->device);
    cudaStreamSynchronize(ctx->stream);
    ctx->scratch_x.release();
    ctx->scratch_block.release();
    ctx->chain_ws.release();
    for (auto& e : ctx->timed) cudaEventDestroy(e.first), cudaEventDestroy(e.second);
    for (auto& e : ctx->event_pool) cudaEventDestroy(e.first), cudaEventDestroy(e.second);
    for (auto e : ctx->d2h_events) cudaEventDestroy(e);
    if (ctx->d2h) cudaStreamDestroy(ctx->d2h);
    if (ctx->aux) cudaStreamDestroy(ctx->aux);
    if (ctx->fork_ev) cudaEventDestroy(ctx->fork_ev);
    if (ctx->join_ev) cudaEventDestroy(ctx->join_ev);
    cudaStreamDestroy(ctx->stream);
    delete ctx;
    return MPKG_OK;
}

int mpkg_ctx_stream(mpkg_ctx_t ctx, void** s) {
    return guarded([&] {
        require(ctx && s, "ctx_stream: null argument");
        *s = (void*)ctx->stream;
    });
}

int mpkg_ctx_synchronize(mpkg_ctx_t ctx) {
    return guarded([&] {
        require(ctx != nullptr, "ctx_synchronize: null context");
        MPKG_CUDA(cudaStreamSynchronize(ctx->stream));
    });
}

int mpkg_ctx_set_mode(mpkg_ctx_t ctx, int mode) {
    return guarded([&] {
        require(ctx != nullptr, "ctx_set_mode: null context");
        require(mode == MPKG_MODE_BITWISE || mode == MPKG_MODE_FAST,
                "ctx_set_mode: mode must be MPKG_MODE_BITWISE or MPKG_MODE_FAST");
        ctx->mode = mode;
    });
}

int mpkg_ctx_device_info(mpkg_ctx_t ctx, int* sm, size_t* l2, size_t* persist) {
    return guarded([&] {
        require(ctx != nullptr, "ctx_device_info: null context");
        if (sm) *sm = ctx->sm_count;
        if (l2) *l2 = ctx->l2_bytes;
        if (persist) *persist = ctx->persist_max;
    });
}

int mpkg_ctx_set_param(mpkg_ctx_t ctx, const char* key, int64_t value) {
    return guarded([&] {
        require(ctx && key, "ctx_set_param: null argument");
        const std::string k(key);
        if (k == "slack")
            ctx->slack = value;
        else if (k == "order")
            ctx->order = value;
        else if (k == "pass")
            ctx->pass_powers = value;
        else if (k == "l2_budget")
            ctx->l2_budget = value;
        else if (k == "ctas_per_sm")
            ctx->ctas_per_sm = value;
        else if (k == "group")
            ctx->group = value;
        else if (k == "stages")
            ctx->stages = value;
        else if (k == "kernel") {
            require(value >= 0 && value <= 5 && value != 3,
                    "ctx_set_param: kernel must be 0 (lean), 1 (staged), 2 (warp-tile) or 4 (async gather)");
            ctx->kernel = value;
        }
        else if (k == "sweep_variant") {
            require(value >= 0 && value <= 5, "ctx_set_param: sweep_variant must be 0..5");
            ctx->sweep_variant = value;
        }
        else if (k == "ortho_fused") {
            require(value >= 0 && value <= 2, "ctx_set_param: ortho_fused must be 0..2");
            ctx->ortho_fused = value;
        }
        else if (k == "coop_min") {
            require(value >= 0 && value <= 1024, "ctx_set_param: coop_min must be 0..1024");
            ctx->coop_min = value;
        }
        else if (k == "coop_variant") {
            require(value >= 0 && value <= 3, "ctx_set_param: coop_variant must be 0..3");
            ctx->coop_variant = value;
        }
        else if (k == "graphs")
            ctx->graphs = value != 0;
        else if (k == "resident")
            ctx->resident = value != 0;
        else if (k == "trace")
            ctx->trace = value != 0;
        else if (k == "wave_dict")
            ctx->wave_dict = value != 0;
        else if (k == "wave_affine") {
            require(value >= 0 && value <= 2, "ctx_set_param: wave_affine must be 0 (off), 1 (affine) or 2 (affine + banded)");
            ctx->wave_affine = value;
        }
        else if (k == "pdl")
            ctx->pdl = value != 0;
        else if (k == "schedule") {
            require(value >= 0 && value <= 3, "ctx_set_param: schedule must be 0 (auto), 1 (fused), 2 (sweeps) or 3 (wave)");
            ctx->schedule = value;
        }
        else if (k == "producers") {
            require(value >= 0 && value <= 8, "ctx_set_param: producers must be in [0, 8]");
            ctx->producers = value;
        }
        else if (k == "cgroups") {
            require(value >= 0 && value <= 8, "ctx_set_param: cgroups must be in [0, 8]");
            ctx->cgroups = value;
        }
        else if (k == "kernel_timing")
            ctx->kernel_timing = value != 0;
        else if (k == "tile_rows") {
            require(value == 32 || value == 64 || value == 128 || value == 256,
                    "ctx_set_param: tile_rows must be 32 (async kernel), 64, 128 or 256");
            ctx->tile_rows = value;
        } else if (k == "threads") {
            require(value == 0 || value == 256 || value == 512,
                    "ctx_set_param: threads must be 0 (one per tile row), 256 or 512");
            ctx->threads = value;
        }
        else
            fail(MPKG_EINVAL, "ctx_set_param: unknown key " + k);
    });
}

int mpkg_ctx_kernel_times(mpkg_ctx_t ctx, double* total_ms, uint64_t* count, double* max_ms) {
    return guarded([&] {
        require(ctx != nullptr, "ctx_kernel_times: null context");
        double tot = 0.0, mx = 0.0;
        uint64_t cnt = 0;
        for (auto& e : ctx->timed) {
            MPKG_CUDA(cudaEventSynchronize(e.second));
            float ms = 0.f;
            MPKG_CUDA(cudaEventElapsedTime(&ms, e.first, e.second));
            tot += ms;
            mx = std::max(mx, (double)ms);
            ++cnt;
            ctx->event_pool.push_back(e);
        }
        ctx->timed.clear();
        if (total_ms) *total_ms = tot;
        if (count) *count = cnt;
        if (max_ms) *max_ms = mx;
    });
}

int mpkg_ctx_launch_count(mpkg_ctx_t ctx, uint64_t* launches) {
    return guarded([&] {
        require(ctx && launches, "ctx_launch_count: null argument");
        *launches = ctx->launches;
    });
}

// ---- CSR --------------------------------------------------------------------------------------
int mpkg_csr_create(mpkg_ctx_t ctx, uint32_t n_rows, uint32_t n_cols, const uint32_t* rp,
                    const uint32_t* ci, const double* v, mpkg_csr_t* out) {
    return guarded([&] {
        require(ctx && out, "csr_create: null argument");
        validate_csr_host(n_rows, n_cols, rp, ci);
        use_device(ctx);
        auto* A = new mpkg_csr_s();
        A->ctx = ctx;
        A->device = ctx->device;
        A->n_rows = n_rows;
        A->n_cols = n_cols;
        A->nnz = rp[n_rows];
        try {
            A->row_ptr.alloc((uint64_t)n_rows + 1);
            A->col_idx.alloc((uint64_t)A->nnz + 1);
            A->values.alloc((uint64_t)A->nnz + 1);
            MPKG_CUDA(cudaMemcpyAsync(A->row_ptr.p, rp, sizeof(uint32_t) * (n_rows + 1ull),
                                      cudaMemcpyHostToDevice, ctx->stream));
            if (A->nnz) {
                MPKG_CUDA(cudaMemcpyAsync(A->col_idx.p, ci, sizeof(uint32_t) * A->nnz,
                                          cudaMemcpyHostToDevice, ctx->stream));
                MPKG_CUDA(cudaMemcpyAsync(A->values.p, v, sizeof(double) * A->nnz,
                                          cudaMemcpyHostToDevice, ctx->stream));
            }
            MPKG_CUDA(cudaStreamSynchronize(ctx->stream));
        } catch (...) {
            delete A;
            throw;
        }
        *out = A;
    });
}

int mpkg_csr_create_from_host(mpkg_ctx_t ctx, mpkg_host_csr_t h, mpkg_csr_t* out) {
    if (!h) {
        set_error("csr_create_from_host: null host matrix");
        return MPKG_EINVAL;
    }
    return mpkg_csr_create(ctx, h->n_rows, h->n_cols, h->row_ptr.p, h->col_idx.p, h->values.p, out);
}

int mpkg_csr_info(mpkg_csr_t A, uint32_t* n_rows, uint32_t* n_cols, uint32_t* nnz) {
    return guarded([&] {
        require(A != nullptr, "csr_info: null matrix");
        if (n_rows) *n_rows = A->n_rows;
        if (n_cols) *n_cols = A->n_cols;
        if (nnz) *nnz = A->nnz;
    });
}

int mpkg_csr_download(mpkg_csr_t A, uint32_t* rp, uint32_t* ci, double* v) {
    return guarded([&] {
        require(A != nullptr, "csr_download: null matrix");
        use_device(A->ctx);
        cudaStream_t st = A->ctx->stream;
        if (rp) MPKG_CUDA(cudaMemcpyAsync(rp, A->row_ptr.p, sizeof(uint32_t) * (A->n_rows + 1ull), cudaMemcpyDeviceToHost, st));
        if (ci && A->nnz) MPKG_CUDA(cudaMemcpyAsync(ci, A->col_idx.p, sizeof(uint32_t) * A->nnz, cudaMemcpyDeviceToHost, st));
        if (v && A->nnz) MPKG_CUDA(cudaMemcpyAsync(v, A->values.p, sizeof(double) * A->nnz, cudaMemcpyDeviceToHost, st));
        MPKG_CUDA(cudaStreamSynchronize(st));
    });
}

int mpkg_csr_destroy(mpkg_csr_t A) {
    if (!A) return MPKG_OK;
    // The owning context may already be gone (destruction order is the caller's); cudaFree in
    // the DevBuf destructors synchronises the device, so no stream is touched here.
    cudaSetDevice(A->device);
    delete A;
    return MPKG_OK;
}

int mpkg_spmv_dev(mpkg_ctx_t ctx, mpkg_csr_t A, const double* d_x, double* d_y) {
    return guarded([&] {
        require(ctx && A, "spmv: null argument");
        use_device(ctx);
        launch_spmv_sell(ctx, csr_sell(A), false, d_x, d_y, nullptr, 0.0, 0.0);
    });
}

int mpkg_spmv(mpkg_ctx_t ctx, mpkg_csr_t A, const double* x, double* y) {
    return guarded([&] {
        require(ctx && A, "spmv: null argument");
        use_device(ctx);
        DevBuf<double> dx(std::max<uint32_t>(A->n_cols, 1)), dy(std::max<uint32_t>(A->n_rows, 1));
        if (A->n_cols) MPKG_CUDA(cudaMemcpyAsync(dx.p, x, sizeof(double) * A->n_cols, cudaMemcpyHostToDevice, ctx->stream));
        launch_spmv_sell(ctx, csr_sell(A), false, dx.p, dy.p, nullptr, 0.0, 0.0);
        if (A->n_rows) MPKG_CUDA(cudaMemcpyAsync(y, dy.p, sizeof(double) * A->n_rows, cudaMemcpyDeviceToHost, ctx->stream));
        MPKG_CUDA(cudaStreamSynchronize(ctx->stream));
    });
}

// ---- levels -----------------------------------------------------------------------------------
int mpkg_build_levels(mpkg_ctx_t ctx, mpkg_csr_t A, mpkg_levels_t* out) {
    return guarded([&] {
        require(ctx && A && out, "build_levels: null argument");
        require(A->n_rows == A->n_cols, "build_levels: matrix must be square");  // levels.hpp:66-67
        use_device(ctx);
        auto* L = new mpkg_levels_s();
        L->ctx = ctx;
        L->device = ctx->device;
        try {
            gpu_build_levels(ctx, A, L);
        } catch (...) {
            delete L;
            throw;
        }
        *out = L;
    });
}

int mpkg_levels_create(mpkg_ctx_t ctx, uint32_t n_rows, uint32_t n_levels, const uint32_t* levels,
                       const uint32_t* perm, const uint32_t* inv_perm, const uint32_t* level_ptr,
                       mpkg_levels_t* out) {
    return guarded([&] {
        require(ctx && out && level_ptr, "levels_create: null argument");
        require(level_ptr[n_levels] == n_rows, "levels_create: level_ptr does not cover the rows");
        use_device(ctx);
        auto* L = new mpkg_levels_s();
        L->ctx = ctx;
        L->device = ctx->device;
        L->n_rows = n_rows;
        L->n_levels = n_levels;
        L->level_ptr.assign(level_ptr, level_ptr + n_levels + 1);
        L->levels.alloc(n_rows);
        L->perm.alloc(n_rows);
        L->inv_perm.alloc(n_rows);
        L->d_level_ptr.alloc(n_levels + 1);
        cudaStream_t st = ctx->stream;
        if (n_rows) {
            if (levels) MPKG_CUDA(cudaMemcpyAsync(L->levels.p, levels, 4ull * n_rows, cudaMemcpyHostToDevice, st));
            if (perm) MPKG_CUDA(cudaMemcpyAsync(L->perm.p, perm, 4ull * n_rows, cudaMemcpyHostToDevice, st));
            if (inv_perm) MPKG_CUDA(cudaMemcpyAsync(L->inv_perm.p, inv_perm, 4ull * n_rows, cudaMemcpyHostToDevice, st));
        }
        MPKG_CUDA(cudaMemcpyAsync(L->d_level_ptr.p, level_ptr, 4ull * (n_levels + 1), cudaMemcpyHostToDevice, st));
        MPKG_CUDA(cudaStreamSynchronize(st));
        *out = L;
    });
}

int mpkg_levels_info(mpkg_levels_t L, uint32_t* n_rows, uint32_t* n_levels) {
    return guarded([&] {
        require(L != nullptr, "levels_info: null handle");
        if (n_rows) *n_rows = L->n_rows;
        if (n_levels) *n_levels = L->n_levels;
    });
}

int mpkg_levels_get(mpkg_levels_t L, uint32_t* levels, uint32_t* perm, uint32_t* inv_perm,
                    uint32_t* level_ptr) {
    return guarded([&] {
        require(L != nullptr, "levels_get: null handle");
        use_device(L->ctx);
        cudaStream_t st = L->ctx->stream;
        const uint64_t b = 4ull * L->n_rows;
        if (b) {
            if (levels) MPKG_CUDA(cudaMemcpyAsync(levels, L->levels.p, b, cudaMemcpyDeviceToHost, st));
            if (perm) MPKG_CUDA(cudaMemcpyAsync(perm, L->perm.p, b, cudaMemcpyDeviceToHost, st));
            if (inv_perm) MPKG_CUDA(cudaMemcpyAsync(inv_perm, L->inv_perm.p, b, cudaMemcpyDeviceToHost, st));
        }
        MPKG_CUDA(cudaStreamSynchronize(st));
        if (level_ptr) std::memcpy(level_ptr, L->level_ptr.data(), 4ull * L->level_ptr.size());
    });
}

int mpkg_levels_destroy(mpkg_levels_t L) {
    if (!L) return MPKG_OK;
    cudaSetDevice(L->device);
    delete L;
    return MPKG_OK;
}

int mpkg_validate_levels(mpkg_ctx_t ctx, mpkg_csr_t A, mpkg_levels_t L, int* ok) {
    return guarded([&] {
        require(ctx && A && L && ok, "validate_levels: null argument");
        use_device(ctx);
        *ok = gpu_validate_levels(ctx, A, L) ? 1 : 0;
    });
}

// ---- permutation ------------------------------------------------------------------------------
int mpkg_permute(mpkg_ctx_t ctx, mpkg_csr_t A, const uint32_t* perm, mpkg_csr_t* out) {
    return guarded([&] {
        require(ctx && A && out, "permute: null argument");
        require(A->n_rows == A->n_cols, "permute: matrix must be square");
        require(perm != nullptr || A->n_rows == 0, "permute: null permutation");
        use_device(ctx);
        DevBuf<uint32_t> d(std::max<uint32_t>(A->n_rows, 1));
        if (A->n_rows)
            MPKG_CUDA(cudaMemcpyAsync(d.p, perm, 4ull * A->n_rows, cudaMemcpyHostToDevice, ctx->stream));
        gpu_check_permutation(ctx, d.p, A->n_rows);
        auto* B = new mpkg_csr_s();
        try {
            gpu_permute(ctx, A, d.p, B);
        } catch (...) {
            delete B;
            throw;
        }
        *out = B;
    });
}

int mpkg_csr_from_coo_dev(mpkg_ctx_t ctx, uint32_t n_rows, uint32_t n_cols, uint64_t nnz,
                          const uint32_t* d_r, const uint32_t* d_c, const double* d_v, mpkg_csr_t* out) {
    return guarded([&] {
        require(ctx && out, "from_coo: null argument");
        require(nnz == 0 || (d_r && d_c && d_v), "from_coo: null entry arrays");
        use_device(ctx);
        auto B = std::make_unique<mpkg_csr_s>();
        gpu_from_coo(ctx, n_rows, n_cols, nnz, d_r, d_c, d_v, B.get());
        *out = B.release();
    });
}

int mpkg_csr_from_coo(mpkg_ctx_t ctx, uint32_t n_rows, uint32_t n_cols, uint64_t nnz, const uint32_t* r,
                      const uint32_t* c, const double* v, mpkg_csr_t* out) {
    return guarded([&] {
        require(ctx && out, "from_coo: null argument");
        require(nnz == 0 || (r && c && v), "from_coo: null entry arrays");
        require(nnz < (1ull << 31), "from_coo: entry count exceeds 32-bit index range");
        use_device(ctx);
        DevBuf<uint32_t> dr(std::max<uint64_t>(nnz, 1)), dc(std::max<uint64_t>(nnz, 1));
        DevBuf<double> dv(std::max<uint64_t>(nnz, 1));
        if (nnz) {
            MPKG_CUDA(cudaMemcpyAsync(dr.p, r, 4 * nnz, cudaMemcpyHostToDevice, ctx->stream));
            MPKG_CUDA(cudaMemcpyAsync(dc.p, c, 4 * nnz, cudaMemcpyHostToDevice, ctx->stream));
            MPKG_CUDA(cudaMemcpyAsync(dv.p, v, 8 * nnz, cudaMemcpyHostToDevice, ctx->stream));
        }
        auto B = std::make_unique<mpkg_csr_s>();
        gpu_from_coo(ctx, n_rows, n_cols, nnz, dr.p, dc.p, dv.p, B.get());
        *out = B.release();
    });
}

int mpkg_read_matrix_market(mpkg_ctx_t ctx, const char* path, mpkg_csr_t* out) {
    return guarded([&] {
        require(ctx && path && out, "read_matrix_market: null argument");
        use_device(ctx);
        auto B = std::make_unique<mpkg_csr_s>();
        read_matrix_market(ctx, path, B.get());
        *out = B.release();
    });
}

int mpkg_csr_block(mpkg_ctx_t ctx, mpkg_csr_t A, uint32_t r0, uint32_t r1, uint32_t c0, uint32_t c1,
                   mpkg_csr_t* out) {
    return guarded([&] {
        require(ctx && A && out, "csr_block: null argument");
        require(r0 <= r1 && r1 <= A->n_rows, "csr_block: row range outside the matrix");
        require(c0 <= c1 && c1 <= A->n_cols, "csr_block: column range outside the matrix");
        use_device(ctx);
        auto* B = new mpkg_csr_s();
        try {
            gpu_csr_block(ctx, A, r0, r1, c0, c1, B);
        } catch (...) {
            delete B;
            throw;
        }
        *out = B;
    });
}

int mpkg_permute_levels(mpkg_ctx_t ctx, mpkg_csr_t A, mpkg_levels_t L, mpkg_csr_t* out) {
    return guarded([&] {
        require(ctx && A && L && out, "permute: null argument");
        require(A->n_rows == A->n_cols, "permute: matrix must be square");
        require(L->n_rows == A->n_rows, "permute: permutation size mismatch");
        use_device(ctx);
        auto* B = new mpkg_csr_s();
        try {
            gpu_permute(ctx, A, L->perm.p, B);
        } catch (...) {
            delete B;
            throw;
        }
        *out = B;
    });
}

static int permute_vec_common(mpkg_ctx_t ctx, uint32_t n, const double* in, const uint32_t* perm,
                              double* out, bool inverse) {
    return guarded([&] {
        require(ctx != nullptr, "permute_vector: null context");
        if (n == 0) return;
        require(in && perm && out, "permute_vector: null argument");
        use_device(ctx);
        DevBuf<double> di(n), dout(n);
        DevBuf<uint32_t> dp(n);
        MPKG_CUDA(cudaMemcpyAsync(di.p, in, 8ull * n, cudaMemcpyHostToDevice, ctx->stream));
        MPKG_CUDA(cudaMemcpyAsync(dp.p, perm, 4ull * n, cudaMemcpyHostToDevice, ctx->stream));
        gpu_permute_vector(ctx, n, di.p, dp.p, dout.p, inverse);
        MPKG_CUDA(cudaMemcpyAsync(out, dout.p, 8ull * n, cudaMemcpyDeviceToHost, ctx->stream));
        MPKG_CUDA(cudaStreamSynchronize(ctx->stream));
    });
}

int mpkg_permute_vector(mpkg_ctx_t ctx, uint32_t n, const double* in, const uint32_t* perm, double* out) {
    return permute_vec_common(ctx, n, in, perm, out, false);
}
int mpkg_unpermute_vector(mpkg_ctx_t ctx, uint32_t n, const double* in, const uint32_t* perm, double* out) {
    return permute_vec_common(ctx, n, in, perm, out, true);
}

// ---- plan -------------------------------------------------------------------------------------
int mpkg_row_range_footprint(mpkg_csr_t A, uint32_t row_s, uint32_t row_e, int p_m, uint64_t* bytes) {
    return guarded([&] {
        require(A && bytes, "row_range_footprint: null argument");
        require(row_s <= row_e && row_e <= A->n_rows, "row_range_footprint: bad row range");
        use_device(A->ctx);
        uint32_t rs = 0, re = 0;
        MPKG_CUDA(cudaMemcpy(&rs, A->row_ptr.p + row_s, 4, cudaMemcpyDeviceToHost));
        MPKG_CUDA(cudaMemcpy(&re, A->row_ptr.p + row_e, 4, cudaMemcpyDeviceToHost));
        // plan.hpp:59-64
        *bytes = 12ull * (re - rs) + 4ull * (row_e - row_s) + 8ull * (uint64_t)(p_m + 1) * (row_e - row_s);
    });
}

int mpkg_greedy_group(const uint64_t* fp, uint32_t nl, uint64_t target, uint32_t* bounds, uint32_t* nb) {
    return guarded([&] {
        require(bounds && nb && (fp || nl == 0), "greedy_group: null argument");
        // plan.hpp:70-85
        uint32_t k = 0;
        bounds[k++] = 0;
        uint64_t acc = 0;
        for (uint32_t l = 0; l < nl; ++l) {
            if (l > bounds[k - 1] && acc + fp[l] > target) {
                bounds[k++] = l;
                acc = 0;
            }
            acc += fp[l];
        }
        if (nl > 0) bounds[k++] = nl;
        *nb = k;
    });
}

int mpkg_group_levels(mpkg_ctx_t ctx, mpkg_levels_t L, mpkg_csr_t A, uint64_t cache_bytes, int p_m,
                      mpkg_plan_t* out) {
    return guarded([&] {
        require(ctx && L && A && out, "group_levels: null argument");
        // plan.hpp:90-92
        require(p_m >= 1, "group_levels: p_m must be >= 1");
        require(A->n_rows == L->n_rows, "group_levels: level structure does not match matrix");
        use_device(ctx);
        const uint32_t nl = L->n_levels;
        // row_ptr of A_perm at every level boundary, gathered on the device
        std::vector<uint32_t> nnz_at(nl + 1, 0);
        gpu_gather_row_ptr(ctx, A, L->d_level_ptr.p, nl + 1, nnz_at.data());
        auto* P = new mpkg_plan_s();
        P->p_m = p_m;
        P->n_rows = L->n_rows;
        P->cache_bytes = cache_bytes;
        P->target_bytes = cache_bytes / (uint64_t)(p_m + 1);
        P->level_ptr = L->level_ptr;
        std::vector<uint64_t> lfp(nl);
        for (uint32_t l = 0; l < nl; ++l) {
            const uint64_t rows = L->level_ptr[l + 1] - L->level_ptr[l];
            lfp[l] = 12ull * (nnz_at[l + 1] - nnz_at[l]) + 4ull * rows + 8ull * (uint64_t)(p_m + 1) * rows;
        }
        std::vector<uint32_t> bounds(nl + 1);
        uint32_t nb = 0;
        mpkg_greedy_group(lfp.data(), nl, P->target_bytes, bounds.data(), &nb);
        bounds.resize(nb);
        P->group_level_ptr = bounds;
        for (uint32_t b : bounds) P->group_rows.push_back(L->level_ptr[b]);
        for (size_t g = 0; g + 1 < bounds.size(); ++g) {
            uint64_t s = 0;
            for (uint32_t l = bounds[g]; l < bounds[g + 1]; ++l) s += lfp[l];
            P->group_footprint.push_back(s);
        }
        *out = P;
    });
}

int mpkg_plan_create(int p_m, int sub_powers, uint32_t n_rows, uint64_t cache_bytes,
                     uint64_t target_bytes, uint32_t n_groups, const uint32_t* group_rows,
                     const uint32_t* group_level_ptr, const uint64_t* group_footprint,
                     uint32_t n_levels, const uint32_t* level_ptr, mpkg_plan_t* out) {
    return guarded([&] {
        require(out != nullptr, "plan_create: null output");
        require(p_m >= 1, "plan_create: p_m must be >= 1");
        require(sub_powers >= 1, "plan_create: sub_powers must be >= 1");
        require(group_rows != nullptr || n_groups == 0, "plan_create: null group_rows");
        auto* P = new mpkg_plan_s();
        P->p_m = p_m;
        P->sub_powers = sub_powers;
        P->n_rows = n_rows;
        P->cache_bytes = cache_bytes;
        P->target_bytes = target_bytes;
        if (group_rows) P->group_rows.assign(group_rows, group_rows + n_groups + 1);
        if (group_level_ptr) P->group_level_ptr.assign(group_level_ptr, group_level_ptr + n_groups + 1);
        if (group_footprint) P->group_footprint.assign(group_footprint, group_footprint + n_groups);
        if (level_ptr) P->level_ptr.assign(level_ptr, level_ptr + n_levels + 1);
        *out = P;
    });
}

int mpkg_plan_info(mpkg_plan_t P, int* p_m, int* sub, uint32_t* n_rows, uint64_t* cache,
                   uint64_t* target, uint32_t* n_groups) {
    return guarded([&] {
        require(P != nullptr, "plan_info: null plan");
        if (p_m) *p_m = P->p_m;
        if (sub) *sub = P->sub_powers;
        if (n_rows) *n_rows = P->n_rows;
        if (cache) *cache = P->cache_bytes;
        if (target) *target = P->target_bytes;
        if (n_groups) *n_groups = P->group_rows.empty() ? 0 : (uint32_t)(P->group_rows.size() - 1);
    });
}

int mpkg_plan_get(mpkg_plan_t P, uint32_t* gr, uint32_t* glp, uint64_t* gfp) {
    return guarded([&] {
        require(P != nullptr, "plan_get: null plan");
        if (gr) std::copy(P->group_rows.begin(), P->group_rows.end(), gr);
        if (glp) std::copy(P->group_level_ptr.begin(), P->group_level_ptr.end(), glp);
        if (gfp) std::copy(P->group_footprint.begin(), P->group_footprint.end(), gfp);
    });
}

int mpkg_plan_destroy(mpkg_plan_t P) {
    delete P;
    return MPKG_OK;
}

int mpkg_plan_exec_info(mpkg_plan_t P, uint32_t* n_tiles, uint64_t* n_tickets, uint64_t* n_deps,
                        uint32_t* pass_powers) {
    return guarded([&] {
        require(P != nullptr, "plan_exec_info: null plan");
        exec_info(P, n_tiles, n_tickets, n_deps, pass_powers);
    });
}

int mpkg_plan_exec_mode(mpkg_plan_t P, int* order, int* sweeps, int* kernel, uint64_t* long_rows) {
    return guarded([&] {
        require(P != nullptr, "plan_exec_mode: null plan");
        exec_mode(P, order, sweeps, kernel, long_rows);
    });
}

int mpkg_plan_exec_wave(mpkg_plan_t P, int* format, uint64_t* n_chunks, uint64_t* n_affine,
                        uint64_t* n_banded, uint64_t* record_bytes) {
    return guarded([&] {
        require(P != nullptr, "plan_exec_wave: null plan");
        exec_wave(P, format, n_chunks, n_affine, n_banded, record_bytes);
    });
}

int mpkg_plan_exec_trace(mpkg_plan_t P, uint64_t* out, uint64_t capacity, uint64_t* n_stamps,
                         uint32_t* tile_rows) {
    return guarded([&] {
        require(P != nullptr, "plan_exec_trace: null plan");
        exec_trace(P, out, capacity, n_stamps, tile_rows);
    });
}

int mpkg_wavefront_schedule(uint32_t ng, int stages, uint32_t* group, int* stage, uint64_t* n_cells) {
    return guarded([&] {
        require(n_cells != nullptr, "wavefront_schedule: null argument");
        // execute.hpp:59-72
        uint64_t cnt = 0;
        if (ng != 0 && stages > 0) {
            for (int64_t d = 0; d <= (int64_t)ng + stages - 2; ++d)
                for (int q = 1; q <= stages; ++q) {
                    const int64_t g = d - (q - 1);
                    if (g >= 0 && g < (int64_t)ng) {
                        if (group) group[cnt] = (uint32_t)g;
                        if (stage) stage[cnt] = q;
                        ++cnt;
                    }
                }
        }
        *n_cells = cnt;
    });
}

// ---- power kernels ----------------------------------------------------------------------------
int mpkg_baseline_mpk_dev(mpkg_ctx_t ctx, mpkg_csr_t A, const double* d_x, int p_m, double* d_block,
                          uint64_t rows, uint64_t slices) {
    return guarded([&] {
        require(ctx && A, "baseline_mpk: null argument");
        baseline_dev(ctx, A, d_x, p_m, d_block, rows, slices, nullptr, nullptr);
    });
}

int mpkg_baseline_mpk(mpkg_ctx_t ctx, mpkg_csr_t A, const double* x, int p_m, double* block,
                      uint64_t rows, uint64_t slices) {
    return guarded([&] {
        require(ctx && A, "baseline_mpk: null argument");
        check_workspace(A, p_m, rows, slices, "baseline_mpk");
        use_device(ctx);
        with_host_block(ctx, A->n_rows, x, p_m, block, [&](const double* dx, double* dblk) {
            baseline_dev(ctx, A, dx, p_m, dblk, A->n_rows, (uint64_t)p_m + 1, nullptr, nullptr);
        });
    });
}

int mpkg_mpk_dev(mpkg_ctx_t ctx, mpkg_plan_t P, mpkg_csr_t A, const double* d_x, int p_m,
                 double* d_block, uint64_t rows, uint64_t slices) {
    return guarded([&] {
        require(ctx != nullptr, "mpk: null context");
        mpk_dev(ctx, P, A, d_x, p_m, d_block, rows, slices, nullptr, nullptr, nullptr, nullptr, "mpk");
    });
}

int mpkg_mpk(mpkg_ctx_t ctx, mpkg_plan_t P, mpkg_csr_t A, const double* x, int p_m, double* block,
             uint64_t rows, uint64_t slices) {
    return guarded([&] {
        require(ctx && P && A, "mpk: null argument");
        check_workspace(A, p_m, rows, slices, "mpk");
        require(P->n_rows == A->n_rows, "mpk: plan does not match matrix");
        require(p_m <= P->p_m, "execute: p_m exceeds the plan's power budget");
        use_device(ctx);
        host_streamed(ctx, A->n_rows, x, p_m, block, [&](const double* dx, double* dblk) {
            mpk_dev(ctx, P, A, dx, p_m, dblk, A->n_rows, (uint64_t)p_m + 1, nullptr, nullptr,
                    nullptr, nullptr, "mpk", block);
        });
    });
}

int mpkg_check_shift_chain(const double* re, const double* im, int ns) {
    return guarded([&] {
        require((re && im) || ns == 0, "check_shift_chain: null argument");
        shift_chain(re, im, ns, "check_shift_chain");
    });
}

int mpkg_baseline_mpk_shifted_dev(mpkg_ctx_t ctx, mpkg_csr_t A, const double* d_x, const double* re,
                                  const double* im, int ns, double* d_block, uint64_t rows,
                                  uint64_t slices) {
    return guarded([&] {
        require(ctx && A && re && im, "baseline_mpk_shifted: null argument");
        baseline_dev(ctx, A, d_x, ns, d_block, rows, slices, re, im);
    });
}

int mpkg_baseline_mpk_shifted(mpkg_ctx_t ctx, mpkg_csr_t A, const double* x, const double* re,
                              const double* im, int ns, double* block, uint64_t rows, uint64_t slices) {
    return guarded([&] {
        require(ctx && A && re && im, "baseline_mpk_shifted: null argument");
        check_workspace(A, ns, rows, slices, "baseline_mpk_shifted");
        shift_chain(re, im, ns, "baseline_mpk_shifted");
        use_device(ctx);
        with_host_block(ctx, A->n_rows, x, ns, block, [&](const double* dx, double* dblk) {
            baseline_dev(ctx, A, dx, ns, dblk, A->n_rows, (uint64_t)ns + 1, re, im);
        });
    });
}

int mpkg_mpk_shifted_dev(mpkg_ctx_t ctx, mpkg_plan_t P, mpkg_csr_t A, const double* d_x, const double* re,
                         const double* im, int ns, double* d_block, uint64_t rows, uint64_t slices) {
    return guarded([&] {
        require(ctx && re && im, "mpk_shifted: null argument");
        mpk_dev(ctx, P, A, d_x, ns, d_block, rows, slices, re, im, nullptr, nullptr, "mpk_shifted");
    });
}

int mpkg_mpk_shifted(mpkg_ctx_t ctx, mpkg_plan_t P, mpkg_csr_t A, const double* x, const double* re,
                     const double* im, int ns, double* block, uint64_t rows, uint64_t slices) {
    return guarded([&] {
        require(ctx && P && A && re && im, "mpk_shifted: null argument");
        check_workspace(A, ns, rows, slices, "mpk_shifted");
        require(P->n_rows == A->n_rows, "mpk_shifted: plan does not match matrix");
        shift_chain(re, im, ns, "mpk_shifted");
        require(ns <= P->p_m, "execute: p_m exceeds the plan's power budget");
        use_device(ctx);
        host_streamed(ctx, A->n_rows, x, ns, block, [&](const double* dx, double* dblk) {
            mpk_dev(ctx, P, A, dx, ns, dblk, A->n_rows, (uint64_t)ns + 1, re, im, nullptr, nullptr,
                    "mpk_shifted", block);
        });
    });
}

int mpkg_mpk_poly_dev(mpkg_ctx_t ctx, mpkg_plan_t P, mpkg_csr_t A, const double* d_x, const double* c,
                      int d, double* d_z, double* d_block, uint64_t rows, uint64_t slices) {
    return guarded([&] {
        require(ctx && P && A && c && d_z, "mpk_poly: null argument");
        DevBuf<double> own;
        if (!d_block) {
            own.alloc((uint64_t)A->n_rows * (d + 1) + 1);
            d_block = own.p;
            rows = A->n_rows;
            slices = (uint64_t)d + 1;
        }
        mpk_dev(ctx, P, A, d_x, d, d_block, rows, slices, nullptr, nullptr, c, d_z, "mpk_poly");
        if (own.p) MPKG_CUDA(cudaStreamSynchronize(ctx->stream));
    });
}

int mpkg_mpk_poly(mpkg_ctx_t ctx, mpkg_plan_t P, mpkg_csr_t A, const double* x, const double* c, int d,
                  double* z, double* block, uint64_t rows, uint64_t slices) {
    return guarded([&] {
        require(ctx && P && A && c && z, "mpk_poly: null argument");
        if (block) check_workspace(A, d, rows, slices, "mpk_poly");
        use_device(ctx);
        const uint32_t n = A->n_rows;
        DevBuf<double> dz(std::max<uint32_t>(n, 1));
        ctx->scratch_x.ensure(std::max<uint32_t>(n, 1));
        ctx->scratch_block.ensure((uint64_t)n * (d + 1) + 1);
        if (n) MPKG_CUDA(cudaMemcpyAsync(ctx->scratch_x.p, x, 8ull * n, cudaMemcpyHostToDevice, ctx->stream));
        // the block (if wanted) streams back slice by slice like mpkg_mpk; z after the last power
        mpk_dev(ctx, P, A, ctx->scratch_x.p, d, ctx->scratch_block.p, n, (uint64_t)d + 1, nullptr,
                nullptr, c, dz.p, "mpk_poly", block);
        if (n) MPKG_CUDA(cudaMemcpyAsync(z, dz.p, 8ull * n, cudaMemcpyDeviceToHost, ctx->stream));
        if (block && n && block != x) std::memmove(block, x, 8ull * n);
        MPKG_CUDA(cudaStreamSynchronize(ctx->stream));
    });
}

int mpkg_tune_select(const double* table, int p_lo, int p_hi, int* p_opt) {
    return guarded([&] {
        require(table && p_opt, "tune_select: null argument");
        require(p_lo >= 1 && p_hi >= p_lo, "tune_p: bad range");  // mpk.hpp:221
        double best = -1.0;
        int bp = p_lo;
        for (int p = p_lo; p <= p_hi; ++p)
            if (table[p - p_lo] > best) {
                best = table[p - p_lo];
                bp = p;
            }
        *p_opt = bp;
    });
}

int mpkg_tune_p(mpkg_ctx_t ctx, mpkg_levels_t L, mpkg_csr_t A, uint64_t cache_bytes, int p_lo,
                int p_hi, int reps, int* p_opt, double* table) {
    return guarded([&] {
        require(ctx && L && A && p_opt && table, "tune_p: null argument");
        require(p_lo >= 1 && p_hi >= p_lo, "tune_p: bad range");
        if (reps < 3) reps = 3;  // mpk.hpp:241
        use_device(ctx);
        const uint32_t n = A->n_rows;
        DevBuf<double> x(std::max<uint32_t>(n, 1)), blk((uint64_t)n * (p_hi + 1) + 1);
        std::vector<double> ones(n, 1.0);  // mpk.hpp:242
        if (n) MPKG_CUDA(cudaMemcpy(x.p, ones.data(), 8ull * n, cudaMemcpyHostToDevice));
        cudaEvent_t e0, e1;
        MPKG_CUDA(cudaEventCreate(&e0));
        MPKG_CUDA(cudaEventCreate(&e1));
        for (int p = p_lo; p <= p_hi; ++p) {
            mpkg_plan_t P = nullptr;
            int rc = mpkg_group_levels(ctx, L, A, cache_bytes, p, &P);
            if (rc) fail(rc, mpkg_last_error());
            std::unique_ptr<mpkg_plan_s> guard(P);
            mpk_dev(ctx, P, A, x.p, p, blk.p, n, (uint64_t)p + 1, nullptr, nullptr, nullptr, nullptr, "tune_p");
            std::vector<double> t(reps);
            for (int r = 0; r < reps; ++r) {
                MPKG_CUDA(cudaEventRecord(e0, ctx->stream));
                mpk_dev(ctx, P, A, x.p, p, blk.p, n, (uint64_t)p + 1, nullptr, nullptr, nullptr, nullptr, "tune_p");
                MPKG_CUDA(cudaEventRecord(e1, ctx->stream));
                MPKG_CUDA(cudaEventSynchronize(e1));
                float ms = 0.f;
                MPKG_CUDA(cudaEventElapsedTime(&ms, e0, e1));
                t[r] = ms * 1e-3;
            }
            std::nth_element(t.begin(), t.begin() + reps / 2, t.end());
            table[p - p_lo] = 2.0 * A->nnz * p / t[reps / 2] * 1e-9;
        }
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        mpkg_tune_select(table, p_lo, p_hi, p_opt);
    });
}

// ---- Jacobi-preconditioned chains (precon.cu) -------------------------------------------------
int mpkg_jacobi_setup(mpkg_ctx_t ctx, mpkg_csr_t A, int sweeps, mpkg_jacobi_t* out) {
    return guarded([&] {
        require(ctx && A && out, "jacobi_setup: null argument");
        require(sweeps >= 1, "jacobi_setup: sweeps must be >= 1");           // jacobi.hpp:73
        require(A->n_rows == A->n_cols, "jacobi_setup: matrix must be square");  // jacobi.hpp:49
        use_device(ctx);
        auto J = std::make_unique<mpkg_jacobi_s>();
        J->ctx = ctx;
        J->device = ctx->device;
        J->sweeps = sweeps;
        gpu_jacobi_setup(ctx, A, J.get());
        *out = J.release();
    });
}

int mpkg_jacobi_info(mpkg_jacobi_t J, uint32_t* n, int* sweeps) {
    return guarded([&] {
        require(J != nullptr, "jacobi_info: null handle");
        if (n) *n = J->n;
        if (sweeps) *sweeps = J->sweeps;
    });
}

int mpkg_jacobi_get(mpkg_jacobi_t J, uint32_t* pos, double* inv) {
    return guarded([&] {
        require(J != nullptr, "jacobi_get: null handle");
        MPKG_CUDA(cudaSetDevice(J->device));
        if (pos && J->n) MPKG_CUDA(cudaMemcpy(pos, J->pos.p, 4ull * J->n, cudaMemcpyDeviceToHost));
        if (inv && J->n) MPKG_CUDA(cudaMemcpy(inv, J->inv.p, 8ull * J->n, cudaMemcpyDeviceToHost));
    });
}

int mpkg_jacobi_destroy(mpkg_jacobi_t J) {
    if (J) {
        cudaSetDevice(J->device);
        delete J;
    }
    return MPKG_OK;
}

}  // extern "C"

namespace {
void jacobi_args(mpkg_ctx_t ctx, mpkg_jacobi_t J, mpkg_csr_t A, const char* who) {
    require(ctx && J && A, std::string(who) + ": null argument");
    require(A->n_rows == A->n_cols, std::string(who) + ": matrix must be square");
    require(A->n_rows == J->n, std::string(who) + ": size mismatch");  // jacobi.hpp:160 / 182
    use_device(ctx);
}

void jacobi_plan(mpkg_plan_t P, mpkg_jacobi_t J, const char* who) {
    require(P != nullptr, std::string(who) + ": null plan");
    require(P->n_rows == J->n, std::string(who) + ": plan does not match matrix");
    const int stages = J->sweeps == 1 ? 1 : J->sweeps + 1;  // jacobi.hpp:129 JacobiOpChain::stages
    require(P->sub_powers == stages, std::string(who) + ": plan sub_powers mismatch");
}

template <class F>
void host_vec(mpkg_ctx_s* ctx, uint32_t n, const double* in, double* out, F&& body) {
    ctx->scratch_x.ensure(std::max<uint32_t>(n, 1));
    ctx->scratch_block.ensure(std::max<uint32_t>(n, 1));
    if (n) MPKG_CUDA(cudaMemcpyAsync(ctx->scratch_x.p, in, 8ull * n, cudaMemcpyHostToDevice, ctx->stream));
    body(ctx->scratch_x.p, ctx->scratch_block.p);
    if (n) MPKG_CUDA(cudaMemcpyAsync(out, ctx->scratch_block.p, 8ull * n, cudaMemcpyDeviceToHost, ctx->stream));
    MPKG_CUDA(cudaStreamSynchronize(ctx->stream));
}

void sstep_jacobi_dev(mpkg_ctx_t ctx, mpkg_jacobi_t J, mpkg_plan_t P, mpkg_csr_t A,
                      const double* re, const double* im, int s, double* d_block, uint64_t rows,
                      uint64_t slices) {
    jacobi_args(ctx, J, A, "sstep_gmres");
    require(s >= 1, "sstep_gmres: s must be >= 1");
    require(re && im, "sstep_gmres: null shifts");
    require(rows == A->n_rows && slices >= (uint64_t)s + 1, "sstep_gmres: workspace too small");
    shift_chain(re, im, s, "sstep_gmres");
    if (P) {
        jacobi_plan(P, J, "sstep_gmres");
        require(s <= P->p_m, "execute: p_m exceeds the plan's power budget");  // execute.hpp:81-83
    }
    std::vector<double> a, b2;
    shift_coeffs(re, im, s, a, b2);
    gpu_sstep_jacobi(ctx, J, A, d_block, rows, s, a.data(), b2.data());
}
}  // namespace

extern "C" {

int mpkg_jacobi_apply(mpkg_ctx_t ctx, mpkg_jacobi_t J, mpkg_csr_t A, const double* v, double* z) {
    return guarded([&] {
        jacobi_args(ctx, J, A, "jacobi_apply");
        require(v && z, "jacobi_apply: null vector");
        host_vec(ctx, J->n, v, z, [&](const double* dv, double* dz) { gpu_jacobi_apply(ctx, J, A, dv, dz); });
    });
}
int mpkg_jacobi_apply_dev(mpkg_ctx_t ctx, mpkg_jacobi_t J, mpkg_csr_t A, const double* d_v, double* d_z) {
    return guarded([&] {
        jacobi_args(ctx, J, A, "jacobi_apply");
        gpu_jacobi_apply(ctx, J, A, d_v, d_z);
    });
}
int mpkg_jacobi_op(mpkg_ctx_t ctx, mpkg_jacobi_t J, mpkg_csr_t A, const double* v, double* y) {
    return guarded([&] {
        jacobi_args(ctx, J, A, "jacobi_op");
        require(v && y, "jacobi_op: null vector");
        host_vec(ctx, J->n, v, y, [&](const double* dv, double* dy) { gpu_jacobi_op(ctx, J, A, dv, dy); });
    });
}
int mpkg_jacobi_op_dev(mpkg_ctx_t ctx, mpkg_jacobi_t J, mpkg_csr_t A, const double* d_v, double* d_y) {
    return guarded([&] {
        jacobi_args(ctx, J, A, "jacobi_op");
        gpu_jacobi_op(ctx, J, A, d_v, d_y);
    });
}
int mpkg_jacobi_op_blocked(mpkg_ctx_t ctx, mpkg_jacobi_t J, mpkg_plan_t P, mpkg_csr_t A,
                           const double* v, double* y) {
    return guarded([&] {
        jacobi_args(ctx, J, A, "jacobi_op_blocked");
        jacobi_plan(P, J, "jacobi_op_blocked");
        require(v && y, "jacobi_op_blocked: null vector");
        host_vec(ctx, J->n, v, y, [&](const double* dv, double* dy) { gpu_jacobi_op(ctx, J, A, dv, dy); });
    });
}
int mpkg_jacobi_op_blocked_dev(mpkg_ctx_t ctx, mpkg_jacobi_t J, mpkg_plan_t P, mpkg_csr_t A,
                               const double* d_v, double* d_y) {
    return guarded([&] {
        jacobi_args(ctx, J, A, "jacobi_op_blocked");
        jacobi_plan(P, J, "jacobi_op_blocked");
        gpu_jacobi_op(ctx, J, A, d_v, d_y);
    });
}
int mpkg_sstep_jacobi(mpkg_ctx_t ctx, mpkg_jacobi_t J, mpkg_plan_t P, mpkg_csr_t A,
                      const double* re, const double* im, int s, double* block, uint64_t rows,
                      uint64_t slices) {
    return guarded([&] {
        require(block != nullptr, "sstep_gmres: null block");
        require(ctx && A, "sstep_gmres: null argument");
        const uint64_t elems = rows * slices;
        ctx->scratch_block.ensure(std::max<uint64_t>(elems, 1));
        if (elems)
            MPKG_CUDA(cudaMemcpyAsync(ctx->scratch_block.p, block, 8ull * elems, cudaMemcpyHostToDevice, ctx->stream));
        sstep_jacobi_dev(ctx, J, P, A, re, im, s, ctx->scratch_block.p, rows, slices);
        if (elems)
            MPKG_CUDA(cudaMemcpyAsync(block, ctx->scratch_block.p, 8ull * elems, cudaMemcpyDeviceToHost, ctx->stream));
        MPKG_CUDA(cudaStreamSynchronize(ctx->stream));
    });
}
int mpkg_sstep_jacobi_dev(mpkg_ctx_t ctx, mpkg_jacobi_t J, mpkg_plan_t P, mpkg_csr_t A,
                          const double* re, const double* im, int s, double* d_block, uint64_t rows,
                          uint64_t slices) {
    return guarded([&] { sstep_jacobi_dev(ctx, J, P, A, re, im, s, d_block, rows, slices); });
}

// ---- GS2 chains (precon.cu) -------------------------------------------------------------------
int mpkg_gs2_setup(mpkg_ctx_t ctx, mpkg_csr_t A, int gamma, int sweeps, int direction, mpkg_gs2_t* out) {
    return guarded([&] {
        require(ctx && A && out, "gs2_setup: null argument");
        require(gamma >= 0, "gs2_setup: gamma must be >= 0");   // gs2.hpp:57
        require(sweeps >= 1, "gs2_setup: sweeps must be >= 1");  // gs2.hpp:58
        require(direction == 0 || direction == 1, "gs2_setup: direction must be 0 (forward) or 1 (backward)");
        require(A->n_rows == A->n_cols, "gs2_setup: matrix must be square");
        use_device(ctx);
        auto G = std::make_unique<mpkg_gs2_s>();
        G->diag.ctx = ctx;
        G->diag.device = ctx->device;
        G->gamma = gamma;
        G->sweeps = sweeps;
        G->forward = direction == 0;
        try {
            gpu_jacobi_setup(ctx, A, &G->diag);
        } catch (const Status& e) {  // build_diag_info names its caller (jacobi.hpp:48)
            std::string m = e.what();
            const std::string from = "jacobi_setup", to = "gs2_setup";
            if (m.compare(0, from.size(), from) == 0) m = to + m.substr(from.size());
            fail(e.code, m);
        }
        *out = G.release();
    });
}

int mpkg_gs2_info(mpkg_gs2_t G, uint32_t* n, int* gamma, int* sweeps, int* direction) {
    return guarded([&] {
        require(G != nullptr, "gs2_info: null handle");
        if (n) *n = G->diag.n;
        if (gamma) *gamma = G->gamma;
        if (sweeps) *sweeps = G->sweeps;
        if (direction) *direction = G->forward ? 0 : 1;
    });
}

int mpkg_gs2_get(mpkg_gs2_t G, uint32_t* pos, double* inv) {
    return guarded([&] {
        require(G != nullptr, "gs2_get: null handle");
        MPKG_CUDA(cudaSetDevice(G->diag.device));
        const uint32_t n = G->diag.n;
        if (pos && n) MPKG_CUDA(cudaMemcpy(pos, G->diag.pos.p, 4ull * n, cudaMemcpyDeviceToHost));
        if (inv && n) MPKG_CUDA(cudaMemcpy(inv, G->diag.inv.p, 8ull * n, cudaMemcpyDeviceToHost));
    });
}

int mpkg_gs2_destroy(mpkg_gs2_t G) {
    if (G) {
        cudaSetDevice(G->diag.device);
        delete G;
    }
    return MPKG_OK;
}

}  // extern "C"

namespace {
void gs2_checks(mpkg_ctx_t ctx, mpkg_gs2_t G, mpkg_plan_t P, mpkg_csr_t A, int budget) {
    require(ctx && G && A, "gs2: null argument");
    require(A->n_rows == A->n_cols, "gs2: matrix must be square");        // gs2.hpp:165
    require(A->n_rows == G->diag.n, "gs2: size mismatch");                 // gs2.hpp:166-167
    if (P) {
        require(P->n_rows == G->diag.n, "gs2: plan does not match matrix");  // gs2.hpp:174
        require(P->sub_powers == G->gamma + 2, "gs2: plan sub_powers mismatch");
        require(budget <= P->p_m, "execute: p_m exceeds the plan's power budget");
    }
    use_device(ctx);
}

void gs2_run(mpkg_ctx_t ctx, mpkg_gs2_t G, mpkg_plan_t P, mpkg_csr_t A, int mode, const double* d_v,
             double* d_z, double* d_out) {
    gs2_checks(ctx, G, P, A, G->sweeps);
    require(mode >= 0 && mode <= 3, "gs2: mode must be 0..3");
    if (G->diag.n == 0) return;
    if (mode == 1 || mode == 3)  // gs2_apply / gs2_op: zero initial guess
        MPKG_CUDA(cudaMemsetAsync(d_z, 0, 8ull * G->diag.n, ctx->stream));
    gpu_gs2_chain(ctx, G, A, d_v, d_z, mode == 2 ? 2 : (mode == 3 ? 1 : 0), d_out);
}

void gs2_host(mpkg_ctx_t ctx, mpkg_gs2_t G, mpkg_plan_t P, mpkg_csr_t A, int mode, const double* v,
              double* z, double* out) {
    gs2_checks(ctx, G, P, A, G->sweeps);
    require(v != nullptr, "gs2: null vector");
    const uint32_t n = G->diag.n;
    DevBuf<double> buf(3ull * std::max<uint32_t>(n, 1));
    double *dv = buf.p, *dz = buf.p + n, *dout = buf.p + 2ull * n;
    if (n) {
        MPKG_CUDA(cudaMemcpyAsync(dv, v, 8ull * n, cudaMemcpyHostToDevice, ctx->stream));
        if (mode == 0 || mode == 2)
            MPKG_CUDA(cudaMemcpyAsync(dz, z, 8ull * n, cudaMemcpyHostToDevice, ctx->stream));
    }
    gs2_run(ctx, G, P, A, mode, dv, dz, dout);
    if (n) {
        if (z) MPKG_CUDA(cudaMemcpyAsync(z, dz, 8ull * n, cudaMemcpyDeviceToHost, ctx->stream));
        if (out) MPKG_CUDA(cudaMemcpyAsync(out, dout, 8ull * n, cudaMemcpyDeviceToHost, ctx->stream));
    }
    MPKG_CUDA(cudaStreamSynchronize(ctx->stream));
}

void sstep_gs2_dev(mpkg_ctx_t ctx, mpkg_gs2_t G, mpkg_plan_t P, mpkg_csr_t A, const double* re,
                   const double* im, int s, double* d_block, uint64_t rows, uint64_t slices) {
    require(s >= 1, "sstep_gmres: s must be >= 1");
    require(re && im, "sstep_gmres: null shifts");
    gs2_checks(ctx, G, nullptr, A, 0);
    if (P) {  // sstep.hpp:386-391 + sstep_plan_powers (sstep.hpp:235-247)
        require(P->n_rows == G->diag.n, "sstep_gmres: plan does not match matrix");
        require(P->sub_powers == G->gamma + 2, "sstep_gmres: plan sub_powers mismatch");
        require(s * G->sweeps <= P->p_m, "execute: p_m exceeds the plan's power budget");
    }
    require(rows == A->n_rows && slices >= (uint64_t)s + 1, "sstep_gmres: workspace too small");
    shift_chain(re, im, s, "sstep_gmres");
    std::vector<double> a, b2;
    shift_coeffs(re, im, s, a, b2);
    gpu_sstep_gs2(ctx, G, A, d_block, rows, s, a.data(), b2.data());
}
}  // namespace

extern "C" {

int mpkg_gs2_smooth(mpkg_ctx_t ctx, mpkg_gs2_t G, mpkg_plan_t P, mpkg_csr_t A, const double* v, double* z) {
    return guarded([&] {
        require(z != nullptr, "gs2_smooth: null iterate");
        gs2_host(ctx, G, P, A, 0, v, z, nullptr);
    });
}
int mpkg_gs2_apply(mpkg_ctx_t ctx, mpkg_gs2_t G, mpkg_plan_t P, mpkg_csr_t A, const double* v, double* z) {
    return guarded([&] {
        require(z != nullptr, "gs2_apply: null output");
        gs2_host(ctx, G, P, A, 1, v, z, nullptr);
    });
}
int mpkg_gs2_smooth_residual(mpkg_ctx_t ctx, mpkg_gs2_t G, mpkg_plan_t P, mpkg_csr_t A,
                             const double* v, double* z, double* r) {
    return guarded([&] {
        require(z && r, "gs2_smooth_residual: null output");
        gs2_host(ctx, G, P, A, 2, v, z, r);
    });
}
int mpkg_gs2_op(mpkg_ctx_t ctx, mpkg_gs2_t G, mpkg_plan_t P, mpkg_csr_t A, const double* v, double* y) {
    return guarded([&] {
        require(y != nullptr, "gs2_op: null output");
        gs2_host(ctx, G, P, A, 3, v, nullptr, y);
    });
}
int mpkg_gs2_run_dev(mpkg_ctx_t ctx, mpkg_gs2_t G, mpkg_plan_t P, mpkg_csr_t A, int mode,
                     const double* d_v, double* d_z, double* d_out) {
    return guarded([&] { gs2_run(ctx, G, P, A, mode, d_v, d_z, d_out); });
}
int mpkg_sstep_gs2(mpkg_ctx_t ctx, mpkg_gs2_t G, mpkg_plan_t P, mpkg_csr_t A, const double* re,
                   const double* im, int s, double* block, uint64_t rows, uint64_t slices) {
    return guarded([&] {
        require(ctx && block, "sstep_gmres: null argument");
        const uint64_t elems = rows * slices;
        ctx->scratch_block.ensure(std::max<uint64_t>(elems, 1));
        if (elems)
            MPKG_CUDA(cudaMemcpyAsync(ctx->scratch_block.p, block, 8ull * elems, cudaMemcpyHostToDevice, ctx->stream));
        sstep_gs2_dev(ctx, G, P, A, re, im, s, ctx->scratch_block.p, rows, slices);
        if (elems)
            MPKG_CUDA(cudaMemcpyAsync(block, ctx->scratch_block.p, 8ull * elems, cudaMemcpyDeviceToHost, ctx->stream));
        MPKG_CUDA(cudaStreamSynchronize(ctx->stream));
    });
}
int mpkg_sstep_gs2_dev(mpkg_ctx_t ctx, mpkg_gs2_t G, mpkg_plan_t P, mpkg_csr_t A, const double* re,
                       const double* im, int s, double* d_block, uint64_t rows, uint64_t slices) {
    return guarded([&] { sstep_gs2_dev(ctx, G, P, A, re, im, s, d_block, rows, slices); });
}

}  // extern "C"

namespace {
void poly_run(mpkg_ctx_t ctx, mpkg_csr_t A, mpkg_jacobi_t J, mpkg_gs2_t G, const double* re,
              const double* im, int degree, mpkg_plan_t P, const double* d_v, double* d_z) {
    require(ctx && A, "poly_apply: null argument");
    require(!(J && G), "poly_apply: one inner preconditioner at most");
    require(A->n_rows == A->n_cols, "poly_apply: matrix must be square");
    require(degree >= 1 && re && im, "poly_apply: preconditioner not set up");     // poly.hpp:235-236
    require(!G || G->sweeps == 1, "poly_apply: gs2 inner must use a single sweep");  // poly.hpp:237-238
    require(!J || J->n == A->n_rows, "poly_apply: size mismatch");
    require(!G || G->diag.n == A->n_rows, "poly_apply: size mismatch");
    std::vector<uint8_t> role(degree);  // poly.hpp:77-93 poly_roles
    for (int i = 0; i < degree;) {
        if (im[i] == 0.0) {
            role[i++] = 0;
            continue;
        }
        require(i + 1 < degree && re[i + 1] == re[i] && im[i + 1] == -im[i], "poly: conjugate pair not adjacent");
        role[i] = 1, role[i + 1] = 2;
        i += 2;
    }
    if (P) {  // poly.hpp:255-260
        require(P->n_rows == A->n_rows, "poly_apply: plan does not match matrix");
        const int sub = J ? (J->sweeps == 1 ? 1 : J->sweeps + 1) : (G ? G->gamma + 2 : 1);
        require(P->sub_powers == sub, "poly_apply: plan sub_powers mismatch");
    }
    use_device(ctx);
    gpu_poly_apply(ctx, A, J, G, re, im, role.data(), degree, d_v, d_z);
}
}  // namespace

extern "C" {

int mpkg_poly_apply_dev(mpkg_ctx_t ctx, mpkg_csr_t A, mpkg_jacobi_t J, mpkg_gs2_t G, const double* re,
                        const double* im, int degree, mpkg_plan_t P, const double* d_v, double* d_z) {
    return guarded([&] { poly_run(ctx, A, J, G, re, im, degree, P, d_v, d_z); });
}

int mpkg_poly_apply(mpkg_ctx_t ctx, mpkg_csr_t A, mpkg_jacobi_t J, mpkg_gs2_t G, const double* re,
                    const double* im, int degree, mpkg_plan_t P, const double* v, double* z) {
    return guarded([&] {
        require(ctx && A && v && z, "poly_apply: null argument");
        const uint32_t n = A->n_rows;
        use_device(ctx);
        DevBuf<double> buf(2ull * std::max<uint32_t>(n, 1));
        if (n) MPKG_CUDA(cudaMemcpyAsync(buf.p, v, 8ull * n, cudaMemcpyHostToDevice, ctx->stream));
        poly_run(ctx, A, J, G, re, im, degree, P, buf.p, buf.p + n);
        if (n) MPKG_CUDA(cudaMemcpyAsync(z, buf.p + n, 8ull * n, cudaMemcpyDeviceToHost, ctx->stream));
        MPKG_CUDA(cudaStreamSynchronize(ctx->stream));
    });
}

}  // extern "C"

// ---- block orthogonalisation (ortho.hpp) --------------------------------------------------
namespace {
using namespace mpkg_detail;

void ortho_dims(uint64_t rows, uint32_t a, uint32_t b) {
    require(rows < (1ull << 40) && (uint64_t)a * b < (1ull << 31), "ortho: block too large");
}

void icgs_check(mpkg_ctx_t ctx, const double* q, const double* v, uint64_t rows, uint32_t qcols, uint32_t vcols,
                int sweeps, const double* coeff) {
    require(ctx != nullptr, "icgs_block_orthogonalize: null context");
    ortho_dims(rows, qcols, vcols);
    if (qcols == 0 || vcols == 0) return;  // ortho.hpp:102-104: before the sweeps check
    require(sweeps >= 1, "icgs_block_orthogonalize: sweeps must be >= 1");  // ortho.hpp:105-107
    require(q && v && coeff, "icgs_block_orthogonalize: null argument");
}

void tsqr_check(mpkg_ctx_t ctx, const double* v, uint64_t rows, uint32_t cols, const double* r) {
    require(ctx != nullptr, "tsqr: null context");
    if (cols == 0) return;  // ortho.hpp:148-150
    require(rows >= cols, "tsqr: block must have at least as many rows as columns");  // ortho.hpp:151-153
    require(cols <= kTsqrMaxCols, "tsqr: at most 64 columns per block on the GPU");
    ortho_dims(rows, cols, cols);
    require(v && r, "tsqr: null argument");
}

// Host block of rows x cols doubles on the device for the duration of a host-pointer call.
struct HostBlock {
    DevBuf<double> d;
    HostBlock(mpkg_ctx_t ctx, const double* h, uint64_t count) : d(std::max<uint64_t>(count, 1)) {
        if (h && count) MPKG_CUDA(cudaMemcpyAsync(d.p, h, 8ull * count, cudaMemcpyHostToDevice, ctx->stream));
    }
    void back(mpkg_ctx_t ctx, double* h, uint64_t count) {
        if (count) MPKG_CUDA(cudaMemcpyAsync(h, d.p, 8ull * count, cudaMemcpyDeviceToHost, ctx->stream));
    }
};

}  // namespace

extern "C" {

int mpkg_block_dots_dev(mpkg_ctx_t ctx, const double* d_q, const double* d_v, uint64_t rows, uint32_t qcols,
                        uint32_t vcols, double* d_c) {
    return guarded([&] {
        require(ctx != nullptr, "block_dots: null context");
        ortho_dims(rows, qcols, vcols);
        if (!qcols || !vcols) return;
        require(d_q && d_v && d_c, "block_dots: null argument");
        use_device(ctx);
        gpu_block_dots(ctx, d_q, d_v, rows, qcols, vcols, d_c);
    });
}

int mpkg_block_dots(mpkg_ctx_t ctx, const double* q, const double* v, uint64_t rows, uint32_t qcols,
                    uint32_t vcols, double* c) {
    return guarded([&] {
        require(ctx != nullptr, "block_dots: null context");
        ortho_dims(rows, qcols, vcols);
        if (!qcols || !vcols) return;
        require(q && v && c, "block_dots: null argument");
        use_device(ctx);
        HostBlock dq(ctx, q, rows * qcols), dv(ctx, v, rows * vcols), dc(ctx, nullptr, (uint64_t)qcols * vcols);
        gpu_block_dots(ctx, dq.d.p, dv.d.p, rows, qcols, vcols, dc.d.p);
        dc.back(ctx, c, (uint64_t)qcols * vcols);
        MPKG_CUDA(cudaStreamSynchronize(ctx->stream));
    });
}

int mpkg_block_update_dev(mpkg_ctx_t ctx, const double* d_q, const double* d_c, uint64_t rows, uint32_t qcols,
                          uint32_t vcols, double* d_v) {
    return guarded([&] {
        require(ctx != nullptr, "block_update: null context");
        ortho_dims(rows, qcols, vcols);
        if (!qcols || !vcols) return;
        require(d_q && d_c && d_v, "block_update: null argument");
        use_device(ctx);
        gpu_block_update(ctx, d_q, d_c, rows, qcols, vcols, d_v);
    });
}

int mpkg_block_update(mpkg_ctx_t ctx, const double* q, const double* c, uint64_t rows, uint32_t qcols,
                      uint32_t vcols, double* v) {
    return guarded([&] {
        require(ctx != nullptr, "block_update: null context");
        ortho_dims(rows, qcols, vcols);
        if (!qcols || !vcols) return;
        require(q && c && v, "block_update: null argument");
        use_device(ctx);
        HostBlock dq(ctx, q, rows * qcols), dc(ctx, c, (uint64_t)qcols * vcols), dv(ctx, v, rows * vcols);
        gpu_block_update(ctx, dq.d.p, dc.d.p, rows, qcols, vcols, dv.d.p);
        dv.back(ctx, v, rows * vcols);
        MPKG_CUDA(cudaStreamSynchronize(ctx->stream));
    });
}

int mpkg_icgs_block_orthogonalize_dev(mpkg_ctx_t ctx, const double* d_q, uint64_t rows, uint32_t qcols,
                                      double* d_v, uint32_t vcols, int sweeps, double* d_coeff) {
    return guarded([&] {
        icgs_check(ctx, d_q, d_v, rows, qcols, vcols, sweeps, d_coeff);
        if (!qcols || !vcols) return;
        use_device(ctx);
        gpu_icgs(ctx, d_q, rows, qcols, d_v, vcols, sweeps, d_coeff);
    });
}

int mpkg_icgs_block_orthogonalize(mpkg_ctx_t ctx, const double* q, uint64_t rows, uint32_t qcols, double* v,
                                  uint32_t vcols, int sweeps, double* coeff) {
    return guarded([&] {
        icgs_check(ctx, q, v, rows, qcols, vcols, sweeps, coeff);
        if (!qcols || !vcols) return;
        use_device(ctx);
        HostBlock dq(ctx, q, rows * qcols), dv(ctx, v, rows * vcols), dc(ctx, nullptr, (uint64_t)qcols * vcols);
        gpu_icgs(ctx, dq.d.p, rows, qcols, dv.d.p, vcols, sweeps, dc.d.p);
        dv.back(ctx, v, rows * vcols);
        dc.back(ctx, coeff, (uint64_t)qcols * vcols);
        MPKG_CUDA(cudaStreamSynchronize(ctx->stream));
    });
}

int mpkg_tsqr_dev(mpkg_ctx_t ctx, double* d_v, uint64_t rows, uint32_t cols, double* d_r) {
    return guarded([&] {
        tsqr_check(ctx, d_v, rows, cols, d_r);
        if (!cols) return;
        use_device(ctx);
        gpu_tsqr(ctx, d_v, rows, cols, d_r);
    });
}

int mpkg_tsqr(mpkg_ctx_t ctx, double* v, uint64_t rows, uint32_t cols, double* r) {
    return guarded([&] {
        tsqr_check(ctx, v, rows, cols, r);
        if (!cols) return;
        use_device(ctx);
        HostBlock dv(ctx, v, rows * cols), dr(ctx, nullptr, (uint64_t)cols * cols);
        gpu_tsqr(ctx, dv.d.p, rows, cols, dr.d.p);
        dv.back(ctx, v, rows * cols);
        dr.back(ctx, r, (uint64_t)cols * cols);
        MPKG_CUDA(cudaStreamSynchronize(ctx->stream));
    });
}

int mpkg_ortho_block_dev(mpkg_ctx_t ctx, const double* d_q, uint64_t rows, uint32_t qcols, double* d_v,
                         uint32_t vcols, int sweeps, double* d_coeff, double* d_r) {
    return guarded([&] {
        icgs_check(ctx, d_q, d_v, rows, qcols, vcols, sweeps, d_coeff);
        tsqr_check(ctx, d_v, rows, vcols, d_r);
        if (!vcols) return;
        use_device(ctx);
        gpu_ortho_block(ctx, d_q, rows, qcols, d_v, vcols, sweeps, d_coeff, d_r);
    });
}

int mpkg_ortho_block(mpkg_ctx_t ctx, const double* q, uint64_t rows, uint32_t qcols, double* v, uint32_t vcols,
                     int sweeps, double* coeff, double* r) {
    return guarded([&] {
        icgs_check(ctx, q, v, rows, qcols, vcols, sweeps, coeff);
        tsqr_check(ctx, v, rows, vcols, r);
        if (!vcols) return;
        use_device(ctx);
        HostBlock dq(ctx, qcols ? q : nullptr, rows * qcols), dv(ctx, v, rows * vcols),
            dc(ctx, nullptr, (uint64_t)qcols * vcols), dr(ctx, nullptr, (uint64_t)vcols * vcols);
        gpu_ortho_block(ctx, dq.d.p, rows, qcols, dv.d.p, vcols, sweeps, dc.d.p, dr.d.p);
        dv.back(ctx, v, rows * vcols);
        if (qcols) dc.back(ctx, coeff, (uint64_t)qcols * vcols);
        dr.back(ctx, r, (uint64_t)vcols * vcols);
        MPKG_CUDA(cudaStreamSynchronize(ctx->stream));
    });
}

}  // extern "C"
