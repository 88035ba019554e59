// Internal device-side types of the mpkg library (not part of the ABI).
#pragma once
#include <utility>

#include <cuda_runtime.h>

#include <cstdint>
#include <memory>
#include <string>
#include <vector>

#include "common.h"
#include "host_csr.h"

namespace mpkg_detail {

#define MPKG_CUDA(call)                                                                        \
    do {                                                                                       \
        cudaError_t e_ = (call);                                                               \
        if (e_ != cudaSuccess) {                                                               \
            (void)cudaGetLastError();                                                          \
            ::mpkg_detail::fail(e_ == cudaErrorMemoryAllocation ? MPKG_ENOMEM : MPKG_ECUDA,    \
                                std::string(#call) + ": " + cudaGetErrorString(e_));           \
        }                                                                                      \
    } while (0)

#define MPKG_LAUNCH_CHECK() MPKG_CUDA(cudaGetLastError())

// Owning device allocation.
template <class T>
struct DevBuf {
    T* p = nullptr;
    uint64_t n = 0;
    DevBuf() = default;
    explicit DevBuf(uint64_t count) { alloc(count); }
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    DevBuf(DevBuf&& o) noexcept : p(o.p), n(o.n) { o.p = nullptr, o.n = 0; }
    DevBuf& operator=(DevBuf&& o) noexcept {
        if (this != &o) {
            release();
            p = o.p, n = o.n;
            o.p = nullptr, o.n = 0;
        }
        return *this;
    }
    ~DevBuf() { release(); }
    void alloc(uint64_t count) {
        release();
        if (count) MPKG_CUDA(cudaMalloc(reinterpret_cast<void**>(&p), sizeof(T) * count));
        n = count;
    }
    // Grow-only reuse for scratch buffers.
    void ensure(uint64_t count) {
        if (count > n) alloc(count);
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        n = 0;
    }
    uint64_t bytes() const { return sizeof(T) * n; }
};

struct Ctx;

// Sliced-ELLPACK (SELL-32) copy of a CSR in a given slot order: the storage the row kernels
// read.  Rows keep their stored entry order (bitwise parity), slot s holds row slot_row[s]
// (identity when slot_row is empty).  Layout per 32-row chunk c starting at entry off[c], the
// same for columns and values (rowdot.cuh sell_pos):
//   (lane, k) -> off + (k/2)*64 + lane*2 + k%2, the odd tail entry at off + Lp*32 + lane
struct Sell {
    uint32_t n_rows = 0;
    uint32_t n_slots = 0;  // multiple of 32
    uint32_t n_chunks = 0;
    uint64_t n_entries = 0;  // padded
    uint32_t long_cap = 0xffffffffu;  // rows longer than this are not stored (fused long path)
    DevBuf<uint64_t> chunk_off;
    DevBuf<uint32_t> row_len;   // per slot
    DevBuf<uint32_t> slot_row;  // per slot, optional (padding slots hold 0xffffffff)
    DevBuf<uint32_t> cols;
    DevBuf<double> vals;
};

struct Executor;  // fused-kernel schedule (mpk_exec.cu)

}  // namespace mpkg_detail

struct mpkg_ctx_s {
    int device = 0;
    cudaStream_t stream = nullptr;
    int sm_count = 0;
    size_t l2_bytes = 0;
    size_t persist_max = 0;
    int mode = MPKG_MODE_BITWISE;
    // executor knobs (mpkg_ctx_set_param)
    int64_t tile_rows = 128;  // rows per fused-kernel tile (32, 64, 128 or 256)
    int64_t slack = -1;  // -1: resident CTA count
    int64_t order = -1;       // -1 auto, 0 A_perm order, 1 Cuthill-McKee, 2 longest rows first
    int64_t pass_powers = 0;  // >0: force powers per fused pass
    int64_t l2_budget = 0;    // >0: live-window budget in bytes (default 0.6 L2)
    int64_t ctas_per_sm = 0;  // >0: cap on resident fused-kernel CTAs per SM
    int64_t group = 8;        // phase-1 gathers in flight per thread (8 or 16)
    int64_t stages = 0;       // >0: staged tickets per CTA (default from smem)
    int64_t threads = 0;      // fused-kernel consumer threads (0: one per tile row)
    int64_t kernel = 0;       // 0: lean (no staging), 1: TMA-staged + producer warp, 2: warp-tile, 4: async gather
    bool graphs = true;       // sweep schedule: replay the p launches as one CUDA graph
    bool pdl = true;          // sweep schedule: programmatic dependent launch between powers
    bool resident = false;    // sweep schedule, L2-resident matrix: one cooperative launch (off:
                              // slower than the per-power graph on C1)
    int64_t sweep_variant = 0;  // sweep-kernel row loop (mpk_exec.cu launch_sweep)
    int64_t ortho_fused = 2;    // fast ICGS: 0 unfused, 1 update+dots re-reading Q from L1/L2, 2 Q staged in smem
    int64_t coop_min = 0;       // fast mode: rows longer than this run warp-cooperatively (0 = 128)
    int64_t coop_variant = 0;   // k_coop_rows: bit 0 = 16 gathers in flight, bit 1 = L2-only gathers
    int64_t wave_dict = 1;    // wave: value-dictionary chunk records when the matrix allows (0: plain)
    int64_t wave_affine = 2;  // wave, dict format: 1 affine records for diagonal-piece chunks, 2 also banded
                              // records where the diagonals break (0: neither)
    int64_t schedule = 0;     // 0 auto, 1 fused kernel, 2 one launch per power, 3 wave (mpk_exec.cu)
    bool trace = false;       // record per-(tile, power) globaltimer stamps (mpkg_plan_exec_trace)
    int64_t producers = 0;    // async kernel: producer warps per CTA (0: 4)
    int64_t cgroups = 0;      // async kernel: consumer groups per CTA (0: 128 / tile_rows)
    uint64_t launches = 0;
    // live timing of the fused / power kernels (mpkg_ctx_set_param "kernel_timing")
    bool kernel_timing = false;
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> timed;  // recorded, not yet read
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> event_pool;
    // device-to-host copy stream + per-slice events for host-pointer calls (run_fused)
    cudaStream_t d2h = nullptr;
    cudaStream_t aux = nullptr;             // side stream of fast-mode sweeps (k_coop_rows)
    cudaEvent_t fork_ev = nullptr, join_ev = nullptr;
    std::vector<cudaEvent_t> d2h_events;
    // scratch
    mpkg_detail::DevBuf<double> scratch_x;
    mpkg_detail::DevBuf<double> scratch_block;
    mpkg_detail::DevBuf<double> chain_ws;  // preconditioned chains' workspace (precon.cu)
    mpkg_detail::DevBuf<double> ortho_c;   // ICGS per-sweep coefficients (ortho.cu)
    mpkg_detail::DevBuf<double> tsqr_ws;   // TSQR tree workspace (ortho.cu)
};

struct mpkg_csr_s {
    mpkg_ctx_s* ctx = nullptr;
    int device = 0;
    uint32_t n_rows = 0;
    uint32_t n_cols = 0;
    uint32_t nnz = 0;
    mpkg_detail::DevBuf<uint32_t> row_ptr;
    mpkg_detail::DevBuf<uint32_t> col_idx;
    mpkg_detail::DevBuf<double> values;
    std::unique_ptr<mpkg_detail::Sell> sell;  // lazily built identity-order SELL copy
};

struct mpkg_levels_s {
    mpkg_ctx_s* ctx = nullptr;
    int device = 0;
    uint32_t n_rows = 0;
    uint32_t n_levels = 0;
    mpkg_detail::DevBuf<uint32_t> levels;
    mpkg_detail::DevBuf<uint32_t> perm;
    mpkg_detail::DevBuf<uint32_t> inv_perm;
    std::vector<uint32_t> level_ptr;  // host copy (n_levels+1)
    mpkg_detail::DevBuf<uint32_t> d_level_ptr;
};

// Jacobi preconditioner (jacobi.hpp:41-76 DiagInfo + JacobiPrecon) on the device.
struct mpkg_jacobi_s {
    mpkg_ctx_s* ctx = nullptr;
    int device = 0;
    uint32_t n = 0;
    int sweeps = 1;
    mpkg_detail::DevBuf<uint32_t> pos;    // index of A(r,r) in col_idx (csr.hpp:233-243)
    mpkg_detail::DevBuf<uint32_t> kdiag;  // the same inside its row (skip index of the sweep)
    mpkg_detail::DevBuf<double> inv;      // 1 / A(r,r)
};

// GS2 preconditioner (gs2.hpp:47-61): DiagInfo + gamma / sweeps / direction.
struct mpkg_gs2_s {
    mpkg_jacobi_s diag;  // pos / kdiag / inv (n), sweeps unused
    int gamma = 1;
    int sweeps = 1;
    bool forward = true;
};

struct mpkg_plan_s {
    int p_m = 1;
    int sub_powers = 1;
    uint32_t n_rows = 0;
    uint64_t cache_bytes = 0;
    uint64_t target_bytes = 0;
    std::vector<uint32_t> group_rows;
    std::vector<uint32_t> group_level_ptr;
    std::vector<uint64_t> group_footprint;
    std::vector<uint32_t> level_ptr;  // the level structure the plan was built on
    std::shared_ptr<mpkg_detail::Executor> exec;
    const mpkg_csr_s* exec_csr = nullptr;  // matrix the executor was built for
};

namespace mpkg_detail {

// Event pair around one kernel launch when ctx->kernel_timing is on (api.cu).
std::pair<cudaEvent_t, cudaEvent_t> timing_begin(mpkg_ctx_s* ctx);
void timing_end(mpkg_ctx_s* ctx, std::pair<cudaEvent_t, cudaEvent_t> ev);

// Kernel launch that may start before the previous kernel on the stream finishes (programmatic
// dependent launch): the kernel's griddepcontrol.wait holds its reads until the predecessor has
// completed and flushed.  Hides the launch gap between back-to-back powers.
template <typename... Ex, typename... Act>
inline void launch_maybe_pdl(bool pdl, void (*k)(Ex...), unsigned grid, unsigned block, cudaStream_t st,
                             Act&&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(block);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
    MPKG_CUDA(cudaLaunchKernelEx(&cfg, k, std::forward<Act>(args)...));
}

// In a kernel launched with launch_maybe_pdl: wait for the predecessor, then let the successor
// launch (one kernel ahead).  Both are no-ops without the launch attribute.
#define MPKG_PDL_ENTRY()                                              \
    do {                                                              \
        asm volatile("griddepcontrol.wait;" ::: "memory");            \
        asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); \
    } while (0)

// SM count of the device the last context was created on (queried in mpkg_ctx_create, never
// assumed): the default grid cap of grid-stride kernels is 32 CTAs per SM.
extern int g_sm_count;
inline unsigned grid_for(uint64_t work, unsigned block, unsigned cap = 0) {
    if (cap == 0) cap = 32u * (unsigned)(g_sm_count > 0 ? g_sm_count : 1);
    uint64_t g = (work + block - 1) / block;
    if (g < 1) g = 1;
    if (g > cap) g = cap;
    return static_cast<unsigned>(g);
}

// sell.cu
Sell& csr_sell(mpkg_csr_s* A);
// d_slot_row: slot -> row (nullptr = identity); d_col_map: column relabel (nullptr = none).
// Rows longer than long_cap are left out of the SELL arrays (row_len keeps their true length).
void build_sell(mpkg_ctx_s* ctx, const mpkg_csr_s* A, const uint32_t* d_slot_row,
                const uint32_t* d_col_map, Sell& out, uint32_t long_cap);

// reorder.cu: GPU-private Cuthill-McKee order inside BFS levels.
void gpu_level_cm_order(mpkg_ctx_s* ctx, const mpkg_csr_s* A, const std::vector<uint32_t>& level_ptr,
                        uint32_t n_slots, DevBuf<uint32_t>& slot_row, DevBuf<uint32_t>& pos,
                        int mode);
uint32_t gpu_max_row_len(mpkg_ctx_s* ctx, const mpkg_csr_s* A);
double gpu_mean_first_col_jump(mpkg_ctx_s* ctx, const mpkg_csr_s* A);
void launch_spmv_sell(mpkg_ctx_s* ctx, const Sell& S, bool shifted, const double* src,
                      double* dst, const double* src2, double shift_a, double shift_b2);
// the same launch without the kernel-timing events (callers that time a whole step)
void launch_spmv_sell_raw(mpkg_ctx_s* ctx, const Sell& S, bool shifted, const double* src,
                          double* dst, const double* src2, double a, double b2, bool pdl = false);

// levels.cu
void gpu_build_levels(mpkg_ctx_s* ctx, const mpkg_csr_s* A, mpkg_levels_s* L);
bool gpu_validate_levels(mpkg_ctx_s* ctx, const mpkg_csr_s* A_perm, const mpkg_levels_s* L);

// permute.cu
void gpu_check_permutation(mpkg_ctx_s* ctx, const uint32_t* d_perm, uint32_t n);
void gpu_permute(mpkg_ctx_s* ctx, const mpkg_csr_s* A, const uint32_t* d_perm, mpkg_csr_s* B);
void gpu_permute_vector(mpkg_ctx_s* ctx, uint32_t n, const double* d_in, const uint32_t* d_perm,
                        double* d_out, bool inverse);
void gpu_csr_block(mpkg_ctx_s* ctx, const mpkg_csr_s* A, uint32_t r0, uint32_t r1, uint32_t c0,
                   uint32_t c1, mpkg_csr_s* B);
void gpu_gather_row_ptr(mpkg_ctx_s* ctx, const mpkg_csr_s* A, const uint32_t* d_idx, uint32_t m,
                        uint32_t* h_out);

// ingest.cu
void gpu_from_coo(mpkg_ctx_s* ctx, uint32_t n_rows, uint32_t n_cols, uint64_t m, const uint32_t* d_r,
                  const uint32_t* d_c, const double* d_v, mpkg_csr_s* B);
void read_matrix_market(mpkg_ctx_s* ctx, const char* path, mpkg_csr_s* B);

// precon.cu
void gpu_jacobi_setup(mpkg_ctx_s* ctx, const mpkg_csr_s* A, mpkg_jacobi_s* J);
void gpu_jacobi_apply(mpkg_ctx_s* ctx, const mpkg_jacobi_s* J, mpkg_csr_s* A, const double* d_v,
                      double* d_z);
void gpu_jacobi_op(mpkg_ctx_s* ctx, const mpkg_jacobi_s* J, mpkg_csr_s* A, const double* d_v,
                   double* d_y);
void gpu_sstep_jacobi(mpkg_ctx_s* ctx, const mpkg_jacobi_s* J, mpkg_csr_s* A, double* d_block,
                      uint64_t rows, int ns, const double* a, const double* b2);
// terminal: 0 none, 1 apply_a (out = A z), 2 residual (out = v - A z); d_z in/out.
void gpu_gs2_chain(mpkg_ctx_s* ctx, const mpkg_gs2_s* G, mpkg_csr_s* A, const double* d_v,
                   double* d_z, int terminal, double* d_out);
void gpu_sstep_gs2(mpkg_ctx_s* ctx, const mpkg_gs2_s* G, mpkg_csr_s* A, double* d_block,
                   uint64_t rows, int ns, const double* a, const double* b2);
// poly.hpp:146-281 product-form polynomial; J / G select the inner preconditioner (both null:
// none); role[i] 0 real, 1 / 2 first / second member of a conjugate pair.
void gpu_poly_apply(mpkg_ctx_s* ctx, mpkg_csr_s* A, const mpkg_jacobi_s* J, const mpkg_gs2_s* G,
                    const double* re, const double* im, const uint8_t* role, int degree,
                    const double* d_v, double* d_z);

// mpk_exec.cu
struct FusedArgs {
    int kind = 0;  // 0 plain, 1 shifted, 2 poly
    int p = 0;
    const double* x = nullptr;
    double* block = nullptr;  // slice-major, stride = rows
    uint64_t rows = 0;
    const double* shift_a = nullptr;   // host arrays, p entries
    const double* shift_b2 = nullptr;  // host arrays, p entries
    const double* coef = nullptr;      // host, p+1 entries
    double* z = nullptr;
    // host-pointer calls: the caller's host block.  run_fused copies slices 1..p there (on a
    // second stream, each slice as soon as its power is done in the sweep schedule) and the
    // context stream waits for the copies; slice 0 (a copy of x) is the caller's job.
    double* host_block = nullptr;
};
void run_fused(mpkg_ctx_s* ctx, mpkg_plan_s* P, mpkg_csr_s* A, const FusedArgs& a);
void exec_info(const mpkg_plan_s* P, uint32_t* n_tiles, uint64_t* n_tickets, uint64_t* n_deps,
               uint32_t* pass_powers);
void exec_mode(const mpkg_plan_s* P, int* order, int* sweeps, int* kernel, uint64_t* long_rows);
void exec_wave(const mpkg_plan_s* P, int* format, uint64_t* n_chunks, uint64_t* n_affine, uint64_t* n_banded,
               uint64_t* record_bytes);
void exec_trace(const mpkg_plan_s* P, uint64_t* out, uint64_t cap, uint64_t* n, uint32_t* tile_rows);

// ortho.cu: block orthogonalisation (reference ortho.hpp)
void gpu_block_dots(mpkg_ctx_s* ctx, const double* q, const double* v, uint64_t rows, uint32_t qcols,
                    uint32_t vcols, double* c);
void gpu_block_update(mpkg_ctx_s* ctx, const double* q, const double* c, uint64_t rows, uint32_t qcols,
                      uint32_t vcols, double* v);
void gpu_icgs(mpkg_ctx_s* ctx, const double* q, uint64_t rows, uint32_t qcols, double* v, uint32_t vcols,
              int sweeps, double* coeff, const double** last_c = nullptr);
void gpu_tsqr(mpkg_ctx_s* ctx, double* v, uint64_t rows, uint32_t c, double* r, const double* upd_q = nullptr,
              const double* upd_coef = nullptr, uint32_t upd_qcols = 0);
void gpu_ortho_block(mpkg_ctx_s* ctx, const double* q, uint64_t rows, uint32_t qcols, double* v, uint32_t vcols,
                     int sweeps, double* coeff, double* r);
constexpr uint32_t kTsqrMaxCols = 64;

}  // namespace mpkg_detail
