// The MPK executor: y_k = A y_{k-1} (plain, shifted, polynomial epilogues) for k = 1..p over the
// level-permuted matrix, bit-identical to the reference (rowdot.cuh's row formula).
//
// Reference behaviour replaced: execute.hpp:79-113 runs every (group, power) cell of the diagonal
// wavefront (execute.hpp:59-72) with an OpenMP team and a barrier after every cell; mpk.hpp:81-106 /
// 184-207 are its kernels.  On the GPU there are three schedules ("schedule" knob, 0 = auto):
//   * wave (3) -- the default for matrices larger than the L2 whose rows are at most 8 entries
//     (C5): cross-power L2 reuse.  One persistent launch per PASS of p' powers; tickets (a tile of
//     two 32-row SELL chunks, one power) run in a host-computed skewed order so the p' power fronts
//     trail each other by about a BFS level and a tile's matrix slice, read from HBM by the first
//     front, is re-read from L2 by the others.  p' is the plan's cache budget applied to this GPU's
//     L2 (plan.hpp:88-115).  Synchronisation is by value (signalling-NaN sentinel fill, no flags).
//     The matrix is kept as chunk records -- general (value dictionary or plain), affine, banded;
//     see "The wave engine" below -- and each warp stages its next ticket's records with one TMA
//     bulk copy (k_mpk_wave);
//   * sweeps (2) -- one launch per power (k_mpk_sweep, replayed as one CUDA graph), with hub rows on
//     a side stream (k_long_rows_bitwise / k_coop_rows): the default otherwise (27-point stencils,
//     R-MAT), where the wave's stage would not hold a chunk;
//   * fused tile-DAG (1) -- all p powers in one launch, per-tile completion flags, TMA-staged tiles
//     (k_mpk_lean and variants): kept, tested, measured slower.
// Rows execute in a GPU-private order sigma that stays inside each BFS level (reorder.cu:
// Cuthill-McKee within levels, longest rows first, or the identity); every result is also stored
// at its A_perm position in the caller's block.  Results are bit-identical to the
// one-launch-per-power baseline (and so to the reference): every row is computed by the same
// formula, from the same inputs, in any order.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <array>
#include <map>
#include <numeric>
#include <parallel/algorithm>
#include <vector>

#include "device.h"
#include "rowdot.cuh"

namespace mpkg_detail {

constexpr int kMaxThreads = 512;         // threads per CTA: 256 or 512 (knob "threads")
constexpr int kMaxStages = 8;            // staged tickets per CTA
constexpr int kMaxFusedP = 32;           // powers per fused launch
constexpr int kBuckets = 4;              // neighbouring-level buckets per tile
constexpr uint32_t kLastUse = 1u << 30;  // ticket flag: last use of the tile in its pass
constexpr uint32_t kBig = 1u << 31;      // ticket flag: tile too large for the smem buffer
constexpr uint32_t kMaxBufBytes = 96 * 1024;
constexpr uint32_t kLongCap = 1024;    // rows longer than this take the CTA-cooperative path
constexpr uint32_t kSB = 64;           // tiles per completion-counter superblock
constexpr uint32_t kLongChunk = 1024;  // products per chunk of a long row (x2 smem ring)
constexpr uint32_t kMedCap = 128;      // fast-mode sweeps: rows longer than this go to k_coop_rows (C3: 128 > 96 > 64 > 256)
constexpr uint32_t kCoopSeg = 2048;    // entries per k_coop_rows work item (longer rows are split)
constexpr uint32_t kLeanRingBytes = 2 * kLongChunk * sizeof(double);
#ifndef MPKG_GROUP
#define MPKG_GROUP 16
#endif
constexpr int kGroup = MPKG_GROUP;       // entries per row issued together (rowdot.cuh)

struct Executor {
    int order = 0;  // 0: A_perm order, 1: Cuthill-McKee inside levels
    uint32_t n_rows = 0, n_slots = 0, n_tiles = 0;
    int grid = 0;
    int64_t slack = 0;
    uint32_t buf_bytes = 0;  // one smem staging buffer (cols + vals of the largest tile)
    uint32_t stages = 2;     // staging buffers (claimed tickets) per CTA
    uint32_t tile_rows = 128;
    uint32_t threads = 256;
    Sell own;                // sigma-order SELL (order 1)
    const Sell* S = nullptr;
    DevBuf<uint32_t> slot_row, pos;  // order 1
    DevBuf<uint32_t> dep_ptr, dep_lo, dep_hi;
    DevBuf<uint64_t> tile_off;  // entry offset of every tile (n_tiles + 1)
    std::vector<uint32_t> h_ptr, h_lo, h_hi;
    std::vector<uint8_t> big;
    std::map<int, DevBuf<uint32_t>> tickets;  // by p
    std::map<int, int> pass_len;              // powers per pass, by p
    std::vector<uint64_t> tile_bytes;         // matrix + vector bytes one tile-power touches
    std::array<int64_t, 4> knobs{};           // slack, pass, l2_budget, ctas/SM in effect
    int group = 16;                           // row group width G of the kernel instance
    int64_t stage_knob = 0;                   // ctx->stages the executor was built with
    int64_t tile_knob = 0, thread_knob = 0;   // ctx->tile_rows / ctx->threads likewise
    int kernel = 0;                           // 0: k_mpk_lean, 1: k_mpk_fused, 2: k_mpk_warptile, 4: k_mpk_async
    uint64_t ne_max = 0;                      // most SELL entries in one tile
    uint32_t n_prod = 0, n_cgroups = 0;       // k_mpk_async roles
    bool sb = false;                          // poll dependencies through superblock counters
    bool last_sweep = false;                  // the last run used one launch per power
    bool last_wave = false;                   // the last run used the wave schedule
    bool fused_ready = false;                 // build_fused() has run
    // sweep schedule: instantiated CUDA graphs by launch parameters (run_fused)
    std::vector<std::pair<std::vector<unsigned char>, cudaGraphExec_t>> graphs;
    Executor() = default;
    Executor(const Executor&) = delete;
    Executor& operator=(const Executor&) = delete;
    ~Executor() {
        for (auto& g : graphs) cudaGraphExecDestroy(g.second);
    }
    int64_t prod_knob = 0, cg_knob = 0;
    uint32_t wt_lmax = 0;                     // warp-tile: chunk width handled flat
    int64_t order_knob = -1;                  // ctx->order the executor was built with
    uint32_t long_cap = 0xffffffffu;          // rows above this length: CTA-cooperative path
    uint64_t long_rows = 0;                   // how many
    bool kernel_forced_lean = false;          // variable tiles need the lean kernel
    int64_t kernel_knob = 0;                  // ctx->kernel the executor was built with
    std::vector<uint32_t> h_tile_start;       // variable tiles (empty: fixed tile_rows)
    DevBuf<uint32_t> long_slots;              // slots of the long rows
    DevBuf<uint32_t> tile_start;
    int occ_max = 1;                          // resident CTAs per SM the smem/regs allow
    DevBuf<uint32_t> done, counter;
    DevBuf<uint32_t> sb_count;                // (kMaxFusedP+1) x n_sb superblock counters
    DevBuf<double> V;   // sigma-order working vectors (order 1)
    DevBuf<double> zs;  // sigma-order polynomial accumulator (order 1)
    // fast-mode cooperative rows (build_coop): work items {slot, k0, k1, part or ~0u}, rows split
    // over several items {slot, first part, parts, 0}, and the per-item partial sums
    bool coop_ready = false;
    uint32_t coop_min = kMedCap;  // rows longer than this are cooperative (knob coop_min)
    DevBuf<uint32_t> long_sorted;  // long slots, longest row first (k_long_rows_bitwise)
    DevBuf<uint32_t> res_bar;    // k_mpk_resident grid barrier {arrivals, generation}
    int res_grid[6] = {0, 0, 0, 0, 0, 0};  // cooperative grid per (kind, sigma)
    DevBuf<uint4> coop_items, coop_multi;
    // wave schedule (schedule knob 3): per p, the pass ticket lists and pass boundaries
    struct Wave {
        DevBuf<uint32_t> tickets;
        DevBuf<uint2> desc;             // k_mpk_wave's ticket descriptors (k_wave_desc)
        std::vector<uint32_t> t_begin;  // first ticket of every pass (+ the end)
        std::vector<int> q_begin;       // first power of every pass (+ p+1)
        int pass_len = 0;
        int64_t slack = 0;
        uint64_t window = 0;            // simulated live window of the chosen pass length
    };
    std::map<int, Wave> wave;
    int wave_grid = 0;                        // resident CTAs of k_mpk_wave (256 threads)
    DevBuf<char> wrec;                        // chunk records (k_wave_pack)
    DevBuf<uint32_t> wrec_off;                // record offsets, 16-byte units (n_tiles * kWaveChunks + 1)
    DevBuf<uint8_t> wave_narrow;              // per tile: every chunk at most 8 entries wide (staged)
    int wave_fmt = 0;                         // chunk-record format: 0 plain, 1 value dictionary
    DevBuf<double> wave_dict;                 // the distinct values (wave_fmt 1)
    uint32_t n_dict = 0;
    DevBuf<double> poly_coef;                 // k_poly_combine's coefficients
    uint64_t wave_affine_chunks = 0;          // chunks stored as affine records
    uint64_t wave_banded_chunks = 0;          // chunks stored as banded records
    uint64_t wave_rec_total = 0;              // bytes of all chunk records
    uint64_t wave_pol[2] = {0, 0};            // createpolicy evict_first / evict_last values
    DevBuf<unsigned long long> trace;         // "trace" knob (FusedParams::trace)
    uint64_t trace_n = 0;
    bool wave_auto = false;                   // schedule 0 picked the wave (get_executor)
    std::vector<uint32_t> wave_reach;         // per tile: furthest tile read by tiles <= T
    uint64_t wave_dep_tiles = 0;              // dependency bucket spans (tiles), summed over tiles
    int64_t sched_knob = 0;
    DevBuf<double> coop_part;
    uint32_t n_coop = 0, n_multi = 0;
};

struct FusedParams {
    const uint32_t* cols;
    const double* vals;
    const uint64_t* chunk_off;
    const uint64_t* tile_off;
    const uint32_t* row_len;
    const uint32_t* slot_row;  // nullptr: identity
    const uint32_t* tickets;
    const uint2* wdesc;        // wave schedule: ticket descriptors
    const char* wrec;          // wave schedule: chunk records
    const uint32_t* wrec_off;
    const double* dict;        // wave: distinct values (dict-format records)
    uint32_t n_dict;
    uint64_t pol_first;        // L2 policies (createpolicy results, k_l2_policies)
    uint64_t pol_last;
    const uint32_t* dep_ptr;
    const uint32_t* dep_lo;
    const uint32_t* dep_hi;
    uint32_t* done;
    uint32_t* counter;
    uint32_t* dbg;  // wave schedule: value-wait count (MPKG_WAVE_DEBUG)
    // "trace" knob: per (power, tile) two globaltimer stamps, [2 (q n_tiles + T)] = inputs complete,
    // [.. + 1] = results about to be stored / published (tests/test_gpu_trace.py audits them)
    unsigned long long* trace;
    uint32_t n_tickets;
    uint32_t n_rows;
    uint32_t n_slots;
    uint32_t p;
    uint32_t buf_bytes;
    uint32_t stages;
    uint32_t tile_rows;
    uint32_t wt_lmax;  // warp-tile kernel: widest chunk handled flat (smem slice per warp)
    const uint32_t* tile_start;  // variable tiles (n_tiles+1 slot offsets) or nullptr
    uint32_t long_cap;           // rows longer than this are not in the SELL arrays
    const uint32_t* csr_rp;      // A_perm CSR (long rows)
    const uint32_t* csr_ci;
    const double* csr_v;
    uint32_t* sb_count;          // [(p+1) * n_sb] completions per power and superblock
    uint32_t n_sb;
    uint32_t n_tiles;
    const uint32_t* long_slots;  // fast mode: slots of the long rows (n_long)
    uint32_t n_long;
    uint32_t n_prod;        // async kernel: producer warps per CTA
    uint32_t n_cgroups;     // async kernel: consumer groups (tile_rows threads each) per CTA
    uint32_t sweep_cap;          // k_mpk_sweep skips rows longer than this
    const uint4* coop_items;     // fast mode: k_coop_rows work items (n_coop)
    const uint4* coop_multi;     // rows split over several items (n_multi)
    double* coop_part;
    uint32_t n_coop;
    uint32_t n_multi;
    uint64_t vstride;  // stride of V slices
    double* V;         // working vectors (== out when identity)
    uint64_t rows;     // stride of the caller's block
    double* out;
    double* zs;
    double* z;
    double shift_a[kMaxFusedP];
    double shift_b2[kMaxFusedP];
    double coef[kMaxFusedP + 1];
};

namespace {

__device__ __forceinline__ uint32_t ld_acquire(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ uint32_t ld_relaxed(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release(uint32_t* p, uint32_t v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar) {
    asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(smem_u32(bar)));
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
    uint32_t done = 0;
    while (!done)
        asm volatile(
            "{ .reg .pred P; mbarrier.try_wait.parity.shared.b64 P, [%1], %2; selp.u32 %0,1,0,P; }"
            : "=r"(done)
            : "r"(smem_u32(bar)), "r"(phase)
            : "memory");
}

__device__ __forceinline__ uint64_t l2_policy(bool last_use) {
    return last_use ? l2_policy_first() : l2_policy_last();
}

// Producer lane only: stage one tile's column indices (one contiguous range of the SELL column
// array) into `buf` with a 1D TMA bulk copy completing on `bar`.
__device__ __forceinline__ void tma_tile(const FusedParams& P, uint32_t T, bool last_use,
                                         char* buf, uint64_t* bar) {
    const uint64_t e0 = P.tile_off[T], e1 = P.tile_off[T + 1];
    const uint32_t cb = (uint32_t)(e1 - e0) * 4u;
    const uint64_t pol = l2_policy(last_use);
    // order earlier generic-proxy accesses of this buffer before the async-proxy writes
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(cb)
                 : "memory");
    if (cb)
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
            "[%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(buf)),
            "l"(P.cols + e0), "r"(cb), "r"(smem_u32(bar)), "l"(pol)
            : "memory");
}

// Dependency check over the runs of tile T for power `need` (= q-1).  A run [lo, hi] is walked
// as units: whole superblocks of kSB tiles (one completion counter per power and superblock,
// incremented by every tile that finishes that power) and the individual flags of the tiles at
// its ragged ends, thread-strided.  Power-law matrices (R-MAT) have runs of ~10^4-10^5 tiles;
// counters bound the poll to O(run/kSB + 2*kSB) loads.
template <bool ACQUIRE>
__device__ __forceinline__ int deps_ready(const FusedParams& P, uint32_t r0, uint32_t r1,
                                          uint32_t need, uint32_t tid, uint32_t nt) {
    for (uint32_t run = r0; run < r1; ++run) {
        const uint32_t lo = P.dep_lo[run], hi = P.dep_hi[run] + 1;  // [lo, hi)
        const uint32_t sb_lo = (lo + kSB - 1) / kSB, sb_hi = hi / kSB;
        uint32_t head, n_sb;
        if (sb_lo < sb_hi) {
            head = sb_lo * kSB - lo;
            n_sb = sb_hi - sb_lo;
        } else {
            head = hi - lo;
            n_sb = 0;
        }
        const uint32_t tail_lo = n_sb ? sb_hi * kSB : hi;
        const uint32_t units = head + n_sb + (hi - tail_lo);
        for (uint32_t u = tid; u < units; u += nt) {
            uint32_t v;
            bool ok;
            if (u < head) {
                const uint32_t* f = P.done + lo + u;
                v = ACQUIRE ? ld_acquire(f) : ld_relaxed(f);
                ok = v >= need;
            } else if (u < head + n_sb) {
                const uint32_t sb = sb_lo + (u - head);
                const uint32_t* f = P.sb_count + (uint64_t)need * P.n_sb + sb;
                v = ACQUIRE ? ld_acquire(f) : ld_relaxed(f);
                ok = v >= min(kSB, P.n_tiles - sb * kSB);
            } else {
                const uint32_t* f = P.done + tail_lo + (u - head - n_sb);
                v = ACQUIRE ? ld_acquire(f) : ld_relaxed(f);
                ok = v >= need;
            }
            if (!ACQUIRE && !ok) return 0;
        }
    }
    return 1;
}

// Dependency check over tile flags only (short runs: every 3D stencil after the level order).
template <bool ACQUIRE>
__device__ __forceinline__ int deps_ready_flags(const FusedParams& P, uint32_t r0, uint32_t r1,
                                                uint32_t need, uint32_t tid, uint32_t nt) {
    for (uint32_t run = r0; run < r1; ++run) {
        const uint32_t hi = P.dep_hi[run];
        for (uint32_t u = P.dep_lo[run] + tid; u <= hi; u += nt) {
            const uint32_t v = ACQUIRE ? ld_acquire(P.done + u) : ld_relaxed(P.done + u);
            if (!ACQUIRE && v < need) return 0;
        }
    }
    return 1;
}

// Publishes "tile T finished power q": the tile flag and its superblock's counter for q.  One
// release fence covers both strong writes (fence + relaxed store / reduction = two release
// patterns), so the publishing thread pays for a single fence.
__device__ __forceinline__ void publish(const FusedParams& P, uint32_t T, uint32_t q) {
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
    asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(P.done + T), "r"(q) : "memory");
    asm volatile("red.relaxed.gpu.global.add.u32 [%0], 1;" ::"l"(P.sb_count + (uint64_t)q * P.n_sb + T / kSB)
                 : "memory");
}

__device__ __forceinline__ unsigned long long global_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ void trace_stamp(const FusedParams& P, uint32_t T, uint32_t q, uint32_t which) {
    if (P.trace) P.trace[2ull * ((uint64_t)q * P.n_tiles + T) + which] = global_ns();
}

__device__ __forceinline__ uint32_t level_of(const uint32_t* __restrict__ lp, uint32_t nl, uint32_t s) {
    uint32_t lo = 0, hi = nl;  // largest l with lp[l] <= s
    while (hi - lo > 1) {
        const uint32_t mid = (lo + hi) >> 1;
        if (lp[mid] <= s)
            lo = mid;
        else
            hi = mid;
    }
    return lo;
}

// Per tile and per neighbouring level bucket (level of the tile's first slot - 1 .. +2), the
// min / max sigma slot of any column read by the tile's rows.
__global__ void k_dep_buckets(const uint32_t* __restrict__ rp, const uint32_t* __restrict__ ci,
                              uint32_t n, const uint32_t* __restrict__ slot_row,
                              const uint32_t* __restrict__ pos, const uint32_t* __restrict__ lp,
                              uint32_t nl, uint32_t tile_rows,
                              const uint32_t* __restrict__ tile_start, uint32_t n_tiles,
                              uint32_t* __restrict__ bmin, uint32_t* __restrict__ bmax) {
    for (uint64_t s = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; s < n;
         s += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t r = slot_row ? slot_row[s] : (uint32_t)s;
        // tile of slot s: fixed-size tiles, or the variable tiles of tile_start
        const uint32_t T = tile_start ? level_of(tile_start, n_tiles, (uint32_t)s) : (uint32_t)(s / tile_rows);
        const uint32_t lt = level_of(lp, nl, tile_start ? tile_start[T] : T * tile_rows);
        const uint32_t L = level_of(lp, nl, (uint32_t)s);
        const uint32_t lb = lp[L], le = lp[L + 1];
        for (uint32_t k = rp[r]; k < rp[r + 1]; ++k) {
            const uint32_t c = ci[k];
            const uint32_t lc = c < lb ? L - 1 : (c >= le ? L + 1 : L);
            int b = (int)lc - (int)lt + 1;
            b = b < 0 ? 0 : (b >= kBuckets ? kBuckets - 1 : b);
            const uint32_t sc = pos ? pos[c] : c;
            atomicMin(bmin + (uint64_t)T * kBuckets + b, sc);
            atomicMax(bmax + (uint64_t)T * kBuckets + b, sc);
        }
    }
}

__global__ void k_gather_x(const double* __restrict__ x, const uint32_t* __restrict__ slot_row,
                           uint32_t n_slots, uint32_t n, double* __restrict__ xs) {
    for (uint64_t s = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; s < n_slots;
         s += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t r = slot_row[s];
        xs[s] = r < n ? x[r] : 0.0;
    }
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// Consumer-only barrier (named barrier 1; the producer warp never joins it).
__device__ __forceinline__ void consumers_sync(uint32_t n) {
    asm volatile("bar.sync 1, %0;" ::"r"(n) : "memory");
}
__device__ __forceinline__ int consumers_and(int v, uint32_t n) {
    int r;
    asm volatile(
        "{ .reg .pred p; setp.ne.s32 p, %1, 0; bar.red.and.pred p, 1, %2, p; selp.s32 %0, 1, 0, p; }"
        : "=r"(r)
        : "r"(v), "r"(n)
        : "memory");
    return r;
}

constexpr uint32_t kNoTicket = 0xffffffffu;

// KIND 0 plain, 1 shifted (Newton), 2 polynomial; SIGMA: private row order; G: gathers in
// flight per thread in phase 1.
//
// Warp-specialised CTA: the LAST warp is the producer, the first blockDim.x-32 threads are
// consumers.  The producer claims tickets (global atomic, in order), stashes ticket + code in a
// ring of P.stages smem slots and stages each tile with TMA into the slot's buffer (mbarrier
// full[slot]); consumers process the slots in order and hand each buffer back through
// empty[slot].  Claims stay in increasing order per CTA and consumers process them in order, so
// the lowest unfinished ticket is always being processed: deadlock-free.
template <int KIND, bool SIGMA, int G>
__global__ void __launch_bounds__(kMaxThreads + 32) k_mpk_fused(const __grid_constant__ FusedParams P) {
    extern __shared__ __align__(128) char smem[];
    __shared__ __align__(8) uint64_t full[kMaxStages];
    __shared__ __align__(8) uint64_t empty[kMaxStages];
    __shared__ uint32_t s_tick[kMaxStages], s_code[kMaxStages];
    const uint32_t tid = threadIdx.x;
    const uint32_t nc = blockDim.x - 32;  // consumer threads
    const uint32_t S = P.stages;
    if (tid == 0) {
        for (uint32_t i = 0; i < S; ++i) {
            mbar_init(&full[i]);
            mbar_init(&empty[i]);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (tid >= nc) {
        // ---------------- producer warp (one lane) ----------------
        if (tid == nc) {
            for (uint32_t i = 0;; ++i) {
                const uint32_t slot = i % S;
                if (i >= S) mbar_wait(&empty[slot], ((i / S) - 1u) & 1u);
                const uint32_t t = atomicAdd(P.counter, 1u);
                if (t >= P.n_tickets) {
                    s_tick[slot] = kNoTicket;
                    mbar_arrive(&full[slot]);
                    break;
                }
                const uint32_t code = P.tickets[t];
                s_tick[slot] = t;
                s_code[slot] = code;
                if (!(code & kBig))
                    tma_tile(P, code & 0xffffffu, code & kLastUse, smem + slot * P.buf_bytes, &full[slot]);
                else
                    mbar_arrive(&full[slot]);
            }
        }
        return;
    }
    // ---------------- consumers ----------------
    for (uint32_t i = 0;; ++i) {
        const uint32_t buf = i % S;
        mbar_wait(&full[buf], (i / S) & 1u);
        if (s_tick[buf] == kNoTicket) return;
        const uint32_t code = s_code[buf];
        const uint32_t T = code & 0xffffffu;
        const uint32_t q = (code >> 24) & 63u;
        if (q > 1) {
            // Poll with relaxed loads (no L1 invalidation), then acquire each observed flag
            // once (flags are monotone).
            const uint32_t r0 = P.dep_ptr[T], r1 = P.dep_ptr[T + 1];
            while (!consumers_and(deps_ready<false>(P, r0, r1, q - 1, tid, nc), nc)) __nanosleep(32);
            (void)deps_ready<true>(P, r0, r1, q - 1, tid, nc);  // acquire each unit once
            consumers_sync(nc);  // publishes every consumer's acquires to all consumers
        }
        const bool big = code & kBig;
        const double* src = P.V + (uint64_t)(q - 1) * P.vstride;
        const uint64_t e0 = P.tile_off[T];
        const uint32_t* cs = reinterpret_cast<const uint32_t*>(smem + buf * P.buf_bytes);
        const uint64_t pol = l2_policy(code & kLastUse);
        // one thread per row: stored-order sequential accumulation + epilogue
        for (uint32_t row = tid; row < P.tile_rows; row += nc) {
            const uint32_t s = T * P.tile_rows + row;
            const uint32_t r = SIGMA ? (s < P.n_slots ? P.slot_row[s] : 0xffffffffu) : s;
            if (r >= P.n_rows) continue;
            const uint32_t len = P.row_len[s];
            const uint64_t c = s >> 5;
            const uint64_t off = P.chunk_off[c];
            const uint32_t L = (uint32_t)((P.chunk_off[c + 1] - off) >> 5);
            double acc;
            if (!big) {
                const uint32_t rel = (uint32_t)(off - e0);
                acc = q == 1 ? sell_row_dot_staged<true, G>(cs, P.vals, rel, off, L, s & 31, len, src, pol)
                             : sell_row_dot_staged<false, G>(cs, P.vals, rel, off, L, s & 31, len, src, pol);
            } else {
                acc = q == 1 ? sell_row_dot<true, 8>(P.cols, P.vals, off, L, s & 31, len, src, pol)
                             : sell_row_dot<false, 8>(P.cols, P.vals, off, L, s & 31, len, src, pol);
            }
            if constexpr (KIND == 1) {
                const double a = P.shift_a[q - 1], b2 = P.shift_b2[q - 1];
                const double own = src[s];
                const double own2 = b2 != 0.0 ? P.V[(uint64_t)(q - 2) * P.vstride + s] : 0.0;
                acc = shift_epilogue(acc, a, b2, own, own2);
            }
            P.V[(uint64_t)q * P.vstride + s] = acc;
            if constexpr (SIGMA) P.out[(uint64_t)q * P.rows + r] = acc;
            if constexpr (KIND == 2) {
                // z = c0*y0 + c1*y1 (+ c2*y2 ...), ascending k, mul then add.
                double zr;
                if (q == 1)
                    zr = __dadd_rn(__dmul_rn(P.coef[0], src[s]), __dmul_rn(P.coef[1], acc));
                else
                    zr = __dadd_rn(P.zs[s], __dmul_rn(P.coef[q], acc));
                P.zs[s] = zr;
                if (SIGMA && q == P.p) P.z[r] = zr;
            }
        }
        consumers_sync(nc);  // tile done: results written, buffer no longer read
        if (tid == 0) {
            publish(P, T, q);
            mbar_arrive(&empty[buf]);
        }
    }
}

// Epilogue of one finished row (slot s, A_perm row r) at power q: shift, stores, polynomial.
template <int KIND, bool SIGMA>
__device__ __forceinline__ void row_epilogue(const FusedParams& P, uint32_t s, uint32_t r, uint32_t q,
                                             const double* src, double acc) {
    if constexpr (KIND == 1) {
        const double a = P.shift_a[q - 1], b2 = P.shift_b2[q - 1];
        const double own = src[s];
        const double own2 = b2 != 0.0 ? P.V[(uint64_t)(q - 2) * P.vstride + s] : 0.0;
        acc = shift_epilogue(acc, a, b2, own, own2);
    }
    P.V[(uint64_t)q * P.vstride + s] = acc;
    if constexpr (SIGMA) P.out[(uint64_t)q * P.rows + r] = acc;
    if constexpr (KIND == 2) {
        double zr;
        if (q == 1)
            zr = __dadd_rn(__dmul_rn(P.coef[0], src[s]), __dmul_rn(P.coef[1], acc));
        else
            zr = __dadd_rn(P.zs[s], __dmul_rn(P.coef[q], acc));
        P.zs[s] = zr;
        if (SIGMA && q == P.p) P.z[r] = zr;
    }
}

// Long row of a single-row tile (see k_mpk_lean).  Bitwise mode must add the row's products
// in stored order, so a hub row is a chain of `len` dependent DADDs (R-MAT scale 21: 102,493):
// that chain is the critical path, and everything else is arranged around it.  Warps 1..3
// compute the products of chunk c+1 (coalesced CSR reads, x gathers) into one half of a
// double-buffered shared-memory ring while thread 0 adds chunk c from the other half at
// shared-memory latency, two products per LDS.128.  Returns true (sum in thread 0's `acc`)
// when slot s0 holds a long row.
template <bool SIGMA, uint32_t kLongChunk = kLongChunk>
__device__ __forceinline__ bool long_row_dot(const FusedParams& P, uint32_t s0, uint32_t q,
                                             uint64_t pol, uint32_t tid, uint32_t nt, double& acc,
                                             double* ring) {
    const uint32_t r = SIGMA ? P.slot_row[s0] : s0;
    const uint32_t len = r < P.n_rows ? P.row_len[s0] : 0u;
    if (len <= P.long_cap) return false;
    const uint32_t b = P.csr_rp[r];
    const double* srcA = P.out + (uint64_t)(q - 1) * P.rows;
    const uint32_t nchunks = (len + kLongChunk - 1) / kLongChunk;
    auto produce = [&](uint32_t c) {  // warps 1.. only; 8 independent gathers in flight per thread
        constexpr int U = 8;
        const uint32_t base = c * kLongChunk, m = min(kLongChunk, len - base);
        double* buf = ring + (c & 1u) * kLongChunk;
        const uint32_t np = nt - 32u;
        for (uint32_t i0 = tid - 32u; i0 < m; i0 += U * np) {
            uint32_t col[U];
            double val[U], xv[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const uint32_t i = i0 + u * np;
                col[u] = i < m ? P.csr_ci[b + base + i] : 0u;
                val[u] = i < m ? ld_mat_d(P.csr_v + b + base + i, pol) : 0.0;
            }
#pragma unroll
            for (int u = 0; u < U; ++u)
                xv[u] = i0 + u * np < m ? (q == 1 ? ld_vec<true>(srcA + col[u]) : ld_vec<false>(srcA + col[u])) : 0.0;
#pragma unroll
            for (int u = 0; u < U; ++u)
                if (i0 + u * np < m) buf[i0 + u * np] = __dmul_rn(val[u], xv[u]);
        }
    };
    acc = 0.0;
    if (tid >= 32) produce(0);
    __syncthreads();
    for (uint32_t c = 0; c < nchunks; ++c) {
        if (tid >= 32) {
            if (c + 1 < nchunks) produce(c + 1);
        } else if (tid == 0) {
            const uint32_t m = min(kLongChunk, len - c * kLongChunk);
            const double2* cur = reinterpret_cast<const double2*>(ring + (c & 1u) * kLongChunk);
            uint32_t i = 0;
            // the next 8 products are loaded while the current 8 are added: the chain pays DADD
            // latency only, not shared-memory latency
            double2 nx[4];
            if (m >= 8) {
#pragma unroll
                for (int j = 0; j < 4; ++j) nx[j] = cur[j];
            }
            for (; i + 8 <= m; i += 8) {
                double2 v[4];
#pragma unroll
                for (int j = 0; j < 4; ++j) v[j] = nx[j];
                if (i + 16 <= m) {
#pragma unroll
                    for (int j = 0; j < 4; ++j) nx[j] = cur[(i + 8) / 2 + j];
                }
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    acc = __dadd_rn(acc, v[j].x);
                    acc = __dadd_rn(acc, v[j].y);
                }
            }
            const double* tail = ring + (c & 1u) * kLongChunk;
            for (; i < m; ++i) acc = __dadd_rn(acc, tail[i]);
        }
        __syncthreads();
    }
    return true;
}

// Sweep schedule: one launch per power over the executor's SELL (private order), grid-stride
// rows, the grouped row loop (8 gathers in flight per thread).  Slice q-1 is complete before the
// launch, so every gather takes the read-only path.  Used when no temporal blocking fits in L2
// (the fused kernel would only add ticket and dependency overhead), see run_fused.
template <int KIND, bool SIGMA, int V>
__global__ void __launch_bounds__(256, V == 1 ? 5 : 0) k_mpk_sweep(const __grid_constant__ FusedParams P, uint32_t q) {
    MPKG_PDL_ENTRY();
    const double* src = P.V + (uint64_t)(q - 1) * P.vstride;
    double* const dst = P.V + (uint64_t)q * P.vstride;
    const uint64_t pol = l2_policy_first();
    for (uint64_t s = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; s < P.n_slots;
         s += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t r = SIGMA ? P.slot_row[s] : (uint32_t)s;
        if (r >= P.n_rows) continue;
        const uint32_t len = P.row_len[s];
        if (len > P.sweep_cap) continue;  // long rows: k_coop_rows / k_long_rows_fast (fast mode)
        const uint64_t off = P.chunk_off[s >> 5];
        const uint32_t L = (uint32_t)((P.chunk_off[(s >> 5) + 1] - off) >> 5);
        double acc;
        if constexpr (V == 2)
            acc = sell_row_dot<true, 4>(P.cols, P.vals, off, L, (uint32_t)(s & 31), len, src, pol);
        else if constexpr (V == 3)
            acc = sell_row_dot_pipe<true>(P.cols, P.vals, off, L, (uint32_t)(s & 31), len, src, pol);
        else if constexpr (V == 4)
            acc = sell_row_dot<true, 28>(P.cols, P.vals, off, L, (uint32_t)(s & 31), len, src, pol);
        else if constexpr (V == 5)
            acc = sell_row_dot<true, 16>(P.cols, P.vals, off, L, (uint32_t)(s & 31), len, src, pol);
        else
            acc = sell_row_dot<true, 8>(P.cols, P.vals, off, L, (uint32_t)(s & 31), len, src, pol);
        if constexpr (KIND == 0 && !SIGMA)
            dst[s] = acc;  // plain powers in A_perm order: the block slice is the working vector
        else
            row_epilogue<KIND, SIGMA>(P, (uint32_t)s, r, q, src, acc);
    }
}

// L2-resident matrices (matrix + p+1 working vectors within half the L2, e.g. config C1): all p
// powers in ONE cooperative launch, a grid-wide barrier between powers instead of a kernel
// boundary.  The matrix is read from HBM once and from L2 by every later power; the launch-gap
// per power disappears.  Power q >= 2 reads the slice written in this launch: plain loads after
// an acquire of the barrier generation (the fused kernels' pattern), never the nc path.
__device__ __forceinline__ void grid_barrier(uint32_t* bar, uint32_t nblocks, uint32_t& gen) {
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
        const uint32_t a = atomicAdd(bar, 1u);
        if (a == nblocks - 1) {
            asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(bar), "r"(0u) : "memory");
            st_release(bar + 1, gen + 1);
        } else {
            while (ld_acquire(bar + 1) == gen) {
            }
        }
    }
    __syncthreads();
    (void)ld_acquire(bar + 1);
    ++gen;
}

template <int KIND, bool SIGMA>
__global__ void __launch_bounds__(256) k_mpk_resident(const __grid_constant__ FusedParams P, uint32_t* bar) {
    uint32_t gen = ld_acquire(bar + 1);
    const uint64_t pol = l2_policy_last();
    for (uint32_t q = 1; q <= P.p; ++q) {
        const double* src = P.V + (uint64_t)(q - 1) * P.vstride;
        for (uint64_t s = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; s < P.n_slots;
             s += (uint64_t)gridDim.x * blockDim.x) {
            const uint32_t r = SIGMA ? P.slot_row[s] : (uint32_t)s;
            if (r >= P.n_rows) continue;
            const uint32_t len = P.row_len[s];
            const uint64_t off = P.chunk_off[s >> 5];
            const uint32_t L = (uint32_t)((P.chunk_off[(s >> 5) + 1] - off) >> 5);
            const double acc = q == 1 ? sell_row_dot<true, 8>(P.cols, P.vals, off, L, (uint32_t)(s & 31), len, src, pol)
                                      : sell_row_dot<false, 8>(P.cols, P.vals, off, L, (uint32_t)(s & 31), len, src, pol);
            row_epilogue<KIND, SIGMA>(P, (uint32_t)s, r, q, src, acc);
        }
        if (q < P.p) grid_barrier(bar, gridDim.x, gen);
    }
}

// Sweep-kernel row-loop variants ("sweep_variant" knob): 0 groups of 8 (64 regs, 4 CTAs/SM),
// 1 the same capped at 5 CTAs/SM, 2 groups of 4, 3 software-pipelined pairs.
template <int KIND, bool SIGMA>
void launch_sweep(int v, unsigned g, cudaStream_t st, const FusedParams& P, uint32_t q, bool pdl = false) {
    if (v == 0) {
        launch_maybe_pdl(pdl, k_mpk_sweep<KIND, SIGMA, 0>, g, 256, st, P, q);
        return;
    }
    switch (v) {
        case 1: k_mpk_sweep<KIND, SIGMA, 1><<<g, 256, 0, st>>>(P, q); break;
        case 2: k_mpk_sweep<KIND, SIGMA, 2><<<g, 256, 0, st>>>(P, q); break;
        case 3: k_mpk_sweep<KIND, SIGMA, 3><<<g, 256, 0, st>>>(P, q); break;
        case 4: k_mpk_sweep<KIND, SIGMA, 4><<<g, 256, 0, st>>>(P, q); break;
        case 5: k_mpk_sweep<KIND, SIGMA, 5><<<g, 256, 0, st>>>(P, q); break;
        default: k_mpk_sweep<KIND, SIGMA, 0><<<g, 256, 0, st>>>(P, q); break;
    }
}

// MPKG_MODE_FAST, sweep schedule: the long rows of power q (left out of the SELL arrays), one
// CTA per row.  Each thread adds its strided share of the products, then a fixed-shape tree
// (warp shuffles, then the per-warp partials in order) combines them: deterministic run to run,
// not the reference's summation order.  Error vs the sequential sum <= ~(log2(len)+nt) * eps
// * sum|products| (below the sequential sum's own len * eps bound); checked
// against the oracle at the north star's 1e-12 inf-norm tolerance.
template <int KIND, bool SIGMA>
__global__ void __launch_bounds__(256) k_long_rows_fast(const __grid_constant__ FusedParams P, uint32_t q) {
    __shared__ double part[8];
    const double* srcA = P.out + (uint64_t)(q - 1) * P.rows;  // A_perm-order copy of y_{q-1}
    const double* src = P.V + (uint64_t)(q - 1) * P.vstride;
    const uint64_t pol = l2_policy_first();
    for (uint32_t i = blockIdx.x; i < P.n_long; i += gridDim.x) {
        const uint32_t s = P.long_slots[i];
        const uint32_t r = SIGMA ? P.slot_row[s] : s;
        const uint32_t b = P.csr_rp[r], e = P.csr_rp[r + 1];
        double acc = 0.0;
        constexpr int U = 8;  // independent gathers in flight per thread
        for (uint32_t k0 = b + threadIdx.x; k0 < e; k0 += U * blockDim.x) {
            uint32_t col[U];
            double val[U], xv[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const uint32_t k = k0 + u * blockDim.x;
                col[u] = k < e ? P.csr_ci[k] : 0u;
                val[u] = k < e ? ld_mat_d(P.csr_v + k, pol) : 0.0;
            }
#pragma unroll
            for (int u = 0; u < U; ++u) xv[u] = k0 + u * blockDim.x < e ? __ldg(srcA + col[u]) : 0.0;
#pragma unroll
            for (int u = 0; u < U; ++u)
                if (k0 + u * blockDim.x < e) acc = __fma_rn(val[u], xv[u], acc);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = acc;
        __syncthreads();
        if (threadIdx.x == 0) {
            double t = 0.0;
            for (uint32_t w = 0; w < blockDim.x / 32; ++w) t += part[w];
            row_epilogue<KIND, SIGMA>(P, s, r, q, src, t);
        }
        __syncthreads();
    }
}

// Bitwise mode, sweep schedule: the long rows (left out of the SELL arrays), one CTA per row,
// longest first, on a side stream concurrently with the power's k_mpk_sweep.  Warps 1..7 form the
// products of a row chunk by chunk into a kBwSlots-deep shared-memory ring; thread 0 adds them in
// stored order -- the reference's sum, bit for bit.  Producers and the adder synchronise through
// per-slot sequence numbers in shared memory (producers: a named barrier, then one release), so
// the producers run up to kBwSlots chunks ahead and a slow gather round never stalls the add
// chain.  The longest row's chain of dependent adds bounds the power.
constexpr uint32_t kBwChunk = 1024;  // products per ring slot
constexpr uint32_t kBwSlots = 4;     // ring depth (4 x 8 KB)

template <int KIND, bool SIGMA>
__global__ void __launch_bounds__(256) k_long_rows_bitwise(const __grid_constant__ FusedParams P, uint32_t q) {
    extern __shared__ __align__(16) double bw_ring[];  // kBwSlots x kBwChunk products
    __shared__ volatile uint32_t full_seq[kBwSlots];   // chunk id + 1 produced into the slot
    __shared__ volatile uint32_t free_seq[kBwSlots];   // chunk id + 1 consumed from the slot
    const double* src = P.V + (uint64_t)(q - 1) * P.vstride;
    const double* srcA = P.out + (uint64_t)(q - 1) * P.rows;  // A_perm-order y_{q-1}
    const uint64_t pol = l2_policy_first();
    const uint32_t tid = threadIdx.x, np = blockDim.x - 32u;
    for (uint32_t it = blockIdx.x; it < P.n_long; it += gridDim.x) {
        if (tid < kBwSlots) full_seq[tid] = 0u, free_seq[tid] = 0u;
        __syncthreads();
        const uint32_t s = P.long_slots[it];
        const uint32_t r = SIGMA ? P.slot_row[s] : s;
        const uint32_t b = P.csr_rp[r], len = P.csr_rp[r + 1] - b;
        const uint32_t nchunks = (len + kBwChunk - 1) / kBwChunk;
        if (tid >= 32) {
            // producers: chunk c into slot c % kBwSlots once the adder has released it
            for (uint32_t c = 0; c < nchunks; ++c) {
                const uint32_t slot = c % kBwSlots;
                if (c >= kBwSlots)
                    while (free_seq[slot] < c + 1 - kBwSlots) __nanosleep(20);
                const uint32_t base = c * kBwChunk, m = min(kBwChunk, len - base);
                double* buf = bw_ring + slot * kBwChunk;
                constexpr int U = 8;
                for (uint32_t i0 = tid - 32u; i0 < m; i0 += U * np) {
                    uint32_t col[U];
                    double val[U], xv[U];
#pragma unroll
                    for (int u = 0; u < U; ++u) {
                        const uint32_t i = i0 + u * np;
                        col[u] = i < m ? P.csr_ci[b + base + i] : 0u;
                        val[u] = i < m ? ld_mat_d(P.csr_v + b + base + i, pol) : 0.0;
                    }
#pragma unroll
                    for (int u = 0; u < U; ++u) xv[u] = i0 + u * np < m ? __ldg(srcA + col[u]) : 0.0;
#pragma unroll
                    for (int u = 0; u < U; ++u)
                        if (i0 + u * np < m) buf[i0 + u * np] = __dmul_rn(val[u], xv[u]);
                }
                asm volatile("bar.sync 1, %0;" ::"r"(np) : "memory");  // every producer wrote chunk c
                if (tid == 32) {
                    __threadfence_block();
                    full_seq[slot] = c + 1;
                }
            }
        } else if (tid == 0) {
            double acc = 0.0;
            for (uint32_t c = 0; c < nchunks; ++c) {
                const uint32_t slot = c % kBwSlots;
                while (full_seq[slot] < c + 1) {
                }
                __threadfence_block();
                const uint32_t m = min(kBwChunk, len - c * kBwChunk);
                const double2* cur = reinterpret_cast<const double2*>(bw_ring + slot * kBwChunk);
                uint32_t i = 0;
                // two register groups loaded alternately, no copies: the adder issues about one
                // instruction per add besides the DADD itself (it shares its SM sub-partition with
                // producer and sweep warps, so every extra instruction lengthens the chain)
                double2 ga[4], gb[4];
                if (m >= 8) {
#pragma unroll
                    for (int j = 0; j < 4; ++j) ga[j] = cur[j];
                }
                for (; i + 16 <= m; i += 16) {
#pragma unroll
                    for (int j = 0; j < 4; ++j) gb[j] = cur[(i + 8) / 2 + j];
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        acc = __dadd_rn(acc, ga[j].x);
                        acc = __dadd_rn(acc, ga[j].y);
                    }
                    if (i + 24 <= m) {
#pragma unroll
                        for (int j = 0; j < 4; ++j) ga[j] = cur[(i + 16) / 2 + j];
                    }
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        acc = __dadd_rn(acc, gb[j].x);
                        acc = __dadd_rn(acc, gb[j].y);
                    }
                }
                if (i + 8 <= m) {  // ga holds products i .. i+7
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        acc = __dadd_rn(acc, ga[j].x);
                        acc = __dadd_rn(acc, ga[j].y);
                    }
                    i += 8;
                }
                const double* tail = bw_ring + slot * kBwChunk;
                for (; i < m; ++i) acc = __dadd_rn(acc, tail[i]);
                __threadfence_block();
                free_seq[slot] = c + 1;
            }
            row_epilogue<KIND, SIGMA>(P, s, r, q, src, acc);
        }
        __syncthreads();
    }
}

// MPKG_MODE_FAST, sweep schedule, rows longer than kMedCap (power-law matrices): one WARP per work
// item -- a whole row, or a kCoopSeg-entry segment of a longer one -- lanes striding the row's
// CSR entries with 8 gathers in flight, a per-lane FMA chain, then a fixed xor-butterfly.  A row
// split over several items leaves its partials in coop_part; k_coop_finish adds them in item
// order.  Deterministic run to run; checked at the north star's 1e-12 inf-norm tolerance.  Runs
// on a side stream concurrently with the power's k_mpk_sweep (disjoint rows, same input slice).
template <int KIND, bool SIGMA, int U, bool CG>
__global__ void __launch_bounds__(256) k_coop_rows(const __grid_constant__ FusedParams P, uint32_t q) {
    const double* srcA = P.out + (uint64_t)(q - 1) * P.rows;  // A_perm-order copy of y_{q-1}
    const double* src = P.V + (uint64_t)(q - 1) * P.vstride;
    const uint64_t pol = l2_policy_first();
    const uint32_t lane = threadIdx.x & 31u;
    const uint32_t nw = gridDim.x * (blockDim.x >> 5);
    for (uint32_t it = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; it < P.n_coop; it += nw) {
        const uint4 d = P.coop_items[it];
        double acc = 0.0;
        for (uint32_t k0 = d.y + lane; k0 < d.z; k0 += U * 32) {
            uint32_t col[U];
            double val[U], xv[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const uint32_t k = k0 + 32u * u;
                col[u] = k < d.z ? ld_mat_u32(P.csr_ci + k, pol) : 0u;
                val[u] = k < d.z ? ld_mat_d(P.csr_v + k, pol) : 0.0;
            }
#pragma unroll
            for (int u = 0; u < U; ++u)
                xv[u] = k0 + 32u * u < d.z ? (CG ? __ldcg(srcA + col[u]) : __ldg(srcA + col[u])) : 0.0;
#pragma unroll
            for (int u = 0; u < U; ++u)
                if (k0 + 32u * u < d.z) acc = __fma_rn(val[u], xv[u], acc);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (lane == 0) {
            if (d.w == 0xffffffffu)
                row_epilogue<KIND, SIGMA>(P, d.x, SIGMA ? P.slot_row[d.x] : d.x, q, src, acc);
            else
                P.coop_part[d.w] = acc;
        }
    }
}

template <int KIND, bool SIGMA>
__global__ void k_coop_finish(const __grid_constant__ FusedParams P, uint32_t q) {
    const double* src = P.V + (uint64_t)(q - 1) * P.vstride;
    for (uint32_t m = blockIdx.x * blockDim.x + threadIdx.x; m < P.n_multi; m += gridDim.x * blockDim.x) {
        const uint4 d = P.coop_multi[m];
        double t = 0.0;
        for (uint32_t i = 0; i < d.z; ++i) t += P.coop_part[d.y + i];
        row_epilogue<KIND, SIGMA>(P, d.x, SIGMA ? P.slot_row[d.x] : d.x, q, src, t);
    }
}

// Lean variant ("kernel" knob 0): no shared-memory staging and no producer warp, so registers
// stay low and many warps are resident (the row loop is latency-bound: throughput follows
// resident warps).  One thread per tile row; thread 0 claims the next ticket while the current
// one runs (double-buffered claim, deadlock-free for the same reason as above).
// Row loop: software-pipelined pairs (sell_row_dot_pipe), ~40 registers -> 12 CTAs per SM.
// No minimum-blocks bound: capping ptxas at 40 registers makes it spill, left alone it fits.
// VT: variable tiles (long rows, single-row tiles); SB: wide dependency runs polled through the
// superblock counters (otherwise tile flags only).
template <int KIND, bool SIGMA, bool VT, bool SB>
__global__ void __launch_bounds__(128) k_mpk_lean(const __grid_constant__ FusedParams P) {
    extern __shared__ __align__(16) double lring[];  // VT: 2 x kLongChunk long-row products
    __shared__ uint32_t s_ticket[2];
    const uint32_t tid = threadIdx.x;
    const uint32_t nt = blockDim.x;
    if (tid == 0) s_ticket[0] = atomicAdd(P.counter, 1u);
    __syncthreads();
    for (uint32_t buf = 0;; buf ^= 1u) {
        const uint32_t t = s_ticket[buf];
        if (t >= P.n_tickets) return;
        if (tid == 0) s_ticket[buf ^ 1u] = atomicAdd(P.counter, 1u);
        const uint32_t code = P.tickets[t];
        const uint32_t T = code & 0xffffffu;
        const uint32_t q = (code >> 24) & 63u;
        if (q > 1) {
            const uint32_t r0 = P.dep_ptr[T], r1 = P.dep_ptr[T + 1];
            if constexpr (SB) {
                while (!__syncthreads_and(deps_ready<false>(P, r0, r1, q - 1, tid, nt))) __nanosleep(32);
                (void)deps_ready<true>(P, r0, r1, q - 1, tid, nt);  // acquire each unit once
            } else {
                while (!__syncthreads_and(deps_ready_flags<false>(P, r0, r1, q - 1, tid, nt))) __nanosleep(32);
                (void)deps_ready_flags<true>(P, r0, r1, q - 1, tid, nt);
            }
            __syncthreads();
        }
        if (tid == 0) trace_stamp(P, T, q, 0);
        const double* src = P.V + (uint64_t)(q - 1) * P.vstride;
        const uint64_t pol = l2_policy(code & kLastUse);
        const uint32_t s0 = VT ? P.tile_start[T] : T * P.tile_rows;
        const uint32_t s1 = VT ? P.tile_start[T + 1] : s0 + P.tile_rows;
        double long_acc = 0.0;
        if (VT && s1 - s0 == 1 && long_row_dot<SIGMA>(P, s0, q, pol, tid, nt, long_acc, lring)) {
            // A single-row tile holding a long row (len > SELL long_cap, e.g. an R-MAT hub): the
            // CTA computes the products from the row's contiguous A_perm CSR slice in chunks,
            // gathering from the A_perm-order copy of y_{q-1} in the caller's block, and one
            // thread adds them in stored order (same formula, same order: bitwise).
            if (tid == 0) row_epilogue<KIND, SIGMA>(P, s0, SIGMA ? P.slot_row[s0] : s0, q, src, long_acc);
        } else {
            const uint32_t nrows = VT ? s1 - s0 : P.tile_rows;
            for (uint32_t row = tid; row < nrows; row += nt) {
                const uint32_t s = (VT ? s0 : T * P.tile_rows) + row;
                const uint32_t r = SIGMA ? (s < P.n_slots ? P.slot_row[s] : 0xffffffffu) : s;
                if (r >= P.n_rows) continue;
                const uint32_t len = P.row_len[s];
                const uint64_t c = s >> 5;
                const uint64_t off = P.chunk_off[c];
                const uint32_t L = (uint32_t)((P.chunk_off[c + 1] - off) >> 5);
                const double acc =
                    q == 1 ? sell_row_dot_pipe<true>(P.cols, P.vals, off, L, s & 31, len, src, pol)
                           : sell_row_dot_pipe<false>(P.cols, P.vals, off, L, s & 31, len, src, pol);
                row_epilogue<KIND, SIGMA>(P, s, r, q, src, acc);
            }
        }
        __syncthreads();
        if (tid == 0) {
            trace_stamp(P, T, q, 1);
            publish(P, T, q);
        }
    }
}

// ---- Wave schedule ("schedule" knob 3): cross-power L2 reuse ------------------------------------
//
// One persistent launch per PASS of p' consecutive powers q0..q1.  The unit of work is a ticket
// (tile = one 32-slot SELL chunk, power q), executed by ONE WARP (lane = row).  The pass's tickets
// are listed in a host-computed skewed order (wave_order: ready(T, q) = ready(reach(T), q-1) +
// slack, reach(T) = the furthest tile T's rows read), so the p' powers sweep the matrix as p'
// fronts a little more than one BFS level apart: a tile's matrix slice is read from HBM by the
// front of power q0 and from L2 by the fronts behind it, as long as the live window (p'-1 level
// lags plus the tickets in flight) fits the L2 budget.  get_wave picks p' by evaluating that
// window on the ticket order -- the plan's cache budget (plan.hpp:88-115) sized for this GPU.
//
// Synchronisation is by VALUE, not by flags.  Before a pass, slices q0..q1-1 (the ones read inside
// the pass) are filled with kWaveEmpty, a signalling-NaN bit pattern that fp64 arithmetic never
// produces (every NaN result is quiet).  Producers store results with relaxed (single-copy atomic)
// stores; a consumer gathers y_{q-1} with relaxed L2 loads and re-loads any value that still reads
// kWaveEmpty.  A row therefore starts only when exactly the values it reads exist -- the
// reference's wavefront rule (execute.hpp:59-72: cell (g, q) after (g-1..g+1, q-1)) at the finest
// possible granularity -- with no flags, no polls and no fences on the path.  Tickets are
// statically assigned (ticket t runs on warp t mod warps, each warp in increasing t) under a
// cooperative launch (all CTAs resident): every input of the lowest unfinished ticket was stored by
// a lower, finished ticket and stores become visible, so it always progresses (deadlock-free).
// Row arithmetic is rowdot.cuh's (stored order, mul then add): bitwise.  Slice 0 and the slices of
// earlier passes are complete before the launch and read through the non-coherent path.
#ifndef MPKG_WAVE_CHUNKS
#define MPKG_WAVE_CHUNKS 2
#endif
#ifndef MPKG_WAVE_CTAS
#define MPKG_WAVE_CTAS 4
#endif
constexpr int kWaveCtas = MPKG_WAVE_CTAS;  // resident CTAs per SM k_mpk_wave is compiled for (register cap)
constexpr uint32_t kWaveChunks = MPKG_WAVE_CHUNKS;  // SELL chunks per tile (processed one after the other)
constexpr uint32_t kWaveRows = 32 * kWaveChunks;   // rows per tile
static_assert(kWaveChunks % 2 == 0, "the fast-tile path takes chunks two at a time");
constexpr unsigned long long kWaveEmpty = 0x7ff4dead5eed0001ull;

// Relaxed (morally strong, single-copy atomic) loads and stores of in-pass slices.  The plain load
// is non-volatile so the compiler may schedule the gathers freely (the value itself is the
// synchronisation); the re-load in the wait loop is volatile so it is really re-issued.
__device__ __forceinline__ double ld_strong(const double* p) {
    double v;
    asm("ld.relaxed.gpu.global.f64 %0, [%1];" : "=d"(v) : "l"(p));
    return v;
}
__device__ __forceinline__ double ld_strong_again(const double* p) {
    double v;
    asm volatile("ld.relaxed.gpu.global.f64 %0, [%1];" : "=d"(v) : "l"(p));
    return v;
}
__device__ __forceinline__ void st_strong(double* p, double v) {
    asm volatile("st.relaxed.gpu.global.f64 [%0], %1;" ::"l"(p), "d"(v));
}
__device__ __forceinline__ bool wave_empty(double v) {
    return (unsigned long long)__double_as_longlong(v) == kWaveEmpty;
}
// A value of a slice written in this launch: re-read until its producer has stored it.
__device__ __forceinline__ double wave_wait(const double* p, double v) {
    while (wave_empty(v)) {
        __nanosleep(100);
        v = ld_strong_again(p);
    }
    return v;
}

// ---- The wave engine ------------------------------------------------------------------------
//
// Chunk records.  The wave keeps its own packed copy of the executor's SELL-32 arrays: chunk T (32
// rows, width L) is ONE contiguous, 16-byte aligned record, so a ticket's whole matrix slice moves
// with one 1D bulk copy.  Two formats (one per matrix):
//   plain (F = 0): len[32] u32 | slot_row[32] u32 (private order only) | cols[32 L] u32 | vals[32 L] f64
//   dict  (F = 1): len[32] u8  | slot_row[32] u32 (private order only) | cols[32 L] u32
//                  | vidx[32][L8] u8 (lane-major, L8 = L rounded up to 8)
// cols / vals in rowdot.cuh's pair interleave.  The dict format stores each value as an 8-bit
// index into the matrix's table of distinct values (CSR-VI value compression; lossless, chosen when
// the matrix has at most 255 distinct values and rows of at most 255 entries): 5 B per entry
// instead of 12 on the HBM stream, and a 1,440-byte stage instead of 3,328 (more warps per SM).
// A dict-format chunk whose 32 rows are all full (len == L <= 8) and whose entry k has column
// base_k + lane and one value v_k in every lane (a piece of a diagonal: what a level-ordered
// stencil's interior looks like) is stored as an AFFINE record instead (info.w = kWaveAffine):
//   len[32] u8 | info | slot_row[32] u32 (private order only) | base[8] u32 | v[8] f64
// 144 bytes instead of 1,200 for a 7-point chunk, no per-lane column or value loads, the same
// entries in the same stored order (lossless; detected per chunk by k_wave_affine, knob
// wave_affine).
// rec_off[T] is the record's offset in 16-byte units.
constexpr uint32_t kWaveAffine = 1u;
// A dict-format chunk of width <= 8 whose rows are not all alike, but each a sub-sequence of one of
// at most TWO row templates (entry k: column base[t][k] + lane, value v[t][k]) is stored as a BANDED
// record (info.w = kWaveBanded): the chunks where a level-ordered stencil's diagonals break (a run
// of grid points ends, boundary rows miss a neighbour).
//   len[32] u8 | info | slot_row[32] u32 (private order only) | meta[32] u16 | base[2][8] u32 | v[2][8] f64
// meta = the lane's template (bit 8) and which of its 8 entries the row has (bits 0-7), in stored
// order: 304 bytes instead of 1,200 (k_wave_affine decides, k_wave_pack fills).
constexpr uint32_t kWaveBanded = 2u;
// info.w bit 2 of a pair's first record (k_wave_pairs): both chunks affine of width 7 and the second
// continues the first one's diagonals (bases + 32, same values): one record serves both.
constexpr uint32_t kWavePair7 = 4u;
constexpr int kWaveMaxPass = 16;  // q - q0 has 4 bits
constexpr int kWaveAutoPass = 3;
constexpr uint32_t kWaveDictMax = 255;

template <int F, bool SIGMA>
struct WaveRec {
    static constexpr uint32_t len_bytes = F == 0 ? 128u : 32u;
    static constexpr uint32_t info = len_bytes;                      // u32 {tile, L, 0, 0}
    static constexpr uint32_t hdr = len_bytes + 16u + (SIGMA ? 128u : 0u);
    __host__ __device__ static constexpr uint32_t l8(uint32_t L) { return (L + 7u) & ~7u; }
    __host__ __device__ static constexpr uint32_t bytes(uint32_t L) {
        return F == 0 ? hdr + 384u * L : hdr + 128u * L + 32u * l8(L);
    }
    static constexpr uint32_t max_staged = bytes(8);
    static constexpr uint32_t affine_bytes = hdr + 96u;
    static constexpr uint32_t banded_bytes = hdr + 256u;
    __device__ static uint32_t len(const char* r, uint32_t lane) {
        if constexpr (F == 0) return reinterpret_cast<const uint32_t*>(r)[lane];
        else return reinterpret_cast<const uint8_t*>(r)[lane];
    }
    __device__ static uint32_t slot(const char* r, uint32_t lane) {
        return reinterpret_cast<const uint32_t*>(r + len_bytes + 16u)[lane];
    }
    __device__ static uint2 tile_l(const char* r) { return *reinterpret_cast<const uint2*>(r + info); }
    __device__ static uint4 info4(const char* r) { return *reinterpret_cast<const uint4*>(r + info); }
};
__host__ __device__ constexpr uint32_t wave_affine_bytes(bool sigma) {
    return sigma ? WaveRec<1, true>::affine_bytes : WaveRec<1, false>::affine_bytes;
}
__host__ __device__ constexpr uint32_t wave_banded_bytes(bool sigma) {
    return sigma ? WaveRec<1, true>::banded_bytes : WaveRec<1, false>::banded_bytes;
}
__host__ __device__ constexpr uint32_t wave_rec_bytes(int F, bool sigma, uint32_t L) {
    return F == 0 ? (sigma ? WaveRec<0, true>::bytes(L) : WaveRec<0, false>::bytes(L))
                  : (sigma ? WaveRec<1, true>::bytes(L) : WaveRec<1, false>::bytes(L));
}

template <typename T>
__device__ __forceinline__ T* opaque_ptr(T* p) {
    asm("" : "+l"(p));
    return p;
}
// Gathers of x_{q-1}: weak and L1-allocating, so the 7 gathers of a 7-point row, which share lines
// ((i,j-1,k) and (i,j,k-1) are neighbours in level l-1), hit L1.  Every location of an in-pass
// slice holds kWaveEmpty or its final value (written once per launch), so a non-empty value read
// this way is final; an empty one (a producer behind, or a stale L1 copy of a line read while it
// still held empty values) is re-read with relaxed L2 loads until its producer has stored it.
__device__ __forceinline__ double ld_gather(const double* p) {
    double v;
    asm("ld.global.ca.f64 %0, [%1];" : "=d"(v) : "l"(p));
    return v;
}
__device__ __forceinline__ bool is_nan_bits(double v) {
    return ((unsigned long long)__double_as_longlong(v) << 1) > (0x7ff0000000000000ull << 1);
}

// Entry k of `lane`'s row in a record (global or staged): its column and its value.
template <int F>
__device__ __forceinline__ uint32_t rec_entry(const char* body, uint32_t L, uint32_t k, uint32_t lane,
                                              const double* dict, double& v, bool affine = false) {
    if (F == 1 && affine) {
        v = reinterpret_cast<const double*>(body + 32)[k];
        return reinterpret_cast<const uint32_t*>(body)[k] + lane;
    }
    const uint32_t Lp = L & ~1u;
    const uint32_t e = k < Lp ? (k >> 1) * 64u + lane * 2u + (k & 1u) : Lp * 32u + lane;
    const uint32_t c = reinterpret_cast<const uint32_t*>(body)[e];
    if constexpr (F == 0) {
        v = reinterpret_cast<const double*>(body + 128u * L)[e];
    } else {
        const uint8_t ix = reinterpret_cast<const uint8_t*>(body + 128u * L)[lane * ((L + 7u) & ~7u) + k];
        v = dict[ix];
    }
    return c;
}

// Cold path: the row of `lane` from a record (global memory for wide chunks), every in-pass value
// awaited (first: the source slice is complete, read-only path).
template <int F>
__device__ __forceinline__ double wave_row_slow(const char* body, uint32_t L, uint32_t lane, uint32_t len,
                                                const double* src, bool first, const double* dict, uint32_t* dbg,
                                                bool affine) {
    if (dbg) atomicAdd(dbg, 1u);
    double acc = 0.0;
    for (uint32_t k = 0; k < len; ++k) {
        double v;
        const uint32_t c = rec_entry<F>(body, L, k, lane, dict, v, affine);
        double x;
        if (first) {
            x = __ldg(src + c);
        } else {
            x = ld_strong_again(src + c);
            while (wave_empty(x)) {
                __nanosleep(64);
                x = ld_strong_again(src + c);
            }
        }
        acc = __dadd_rn(acc, __dmul_rn(v, x));
    }
    return acc;
}

// Hot path: a staged chunk of compile-time width L, one row per lane, summed in stored order.  A
// lane's padding entries (len <= k < L, value 0.0) gather nothing and add 0.0 * 0.0 = +0, which
// leaves the sum unchanged (it starts at +0 and round-to-nearest never makes it -0): rowdot.cuh's
// sum over k < len, bit for bit.
template <int L, int F>
__device__ __forceinline__ double wave_dot(const char* body, uint32_t lane, uint32_t len, const double* src,
                                           const double* dict) {
    constexpr int Lp = L & ~1;
    double x[8];
    const uint32_t* sc = reinterpret_cast<const uint32_t*>(body);
#pragma unroll
    for (int j = 0; j < Lp; j += 2) {
        const uint2 cc = *reinterpret_cast<const uint2*>(sc + (j >> 1) * 64 + lane * 2);
        x[j] = (uint32_t)j < len ? ld_gather(src + cc.x) : 0.0;
        x[j + 1] = (uint32_t)j + 1 < len ? ld_gather(src + cc.y) : 0.0;
    }
    if (L & 1) x[Lp] = (uint32_t)Lp < len ? ld_gather(src + sc[Lp * 32 + lane]) : 0.0;
#pragma unroll
    for (int j = L; j < 8; ++j) x[j] = 0.0;
    double acc = 0.0;
    if constexpr (F == 0) {
        const double* sv = reinterpret_cast<const double*>(body + 128 * L);
#pragma unroll
        for (int j = 0; j < Lp; j += 2) {
            const double2 vv = *reinterpret_cast<const double2*>(sv + (j >> 1) * 64 + lane * 2);
            acc = __dadd_rn(acc, __dmul_rn(vv.x, x[j]));
            acc = __dadd_rn(acc, __dmul_rn(vv.y, x[j + 1]));
        }
        if (L & 1) acc = __dadd_rn(acc, __dmul_rn(sv[Lp * 32 + lane], x[Lp]));
    } else {
        const uint2 vi = *reinterpret_cast<const uint2*>(body + 128 * L + lane * 8);
#pragma unroll
        for (int j = 0; j < L; ++j) {
            const uint32_t ix = ((j < 4 ? vi.x : vi.y) >> (8 * (j & 3))) & 255u;
            acc = __dadd_rn(acc, __dmul_rn(dict[ix], x[j]));
        }
    }
    return acc;
}

// Shared-memory loads by 32-bit shared address (the fast-tile path forms no generic pointer into
// the stage); volatile so they stay behind the stage's mbarrier wait.
__device__ __forceinline__ uint4 lds_v4(uint32_t a) {
    uint4 r;
    asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "r"(a));
    return r;
}
__device__ __forceinline__ double2 lds_d2(uint32_t a) {
    double2 r;
    asm volatile("ld.shared.v2.f64 {%0,%1}, [%2];" : "=d"(r.x), "=d"(r.y) : "r"(a));
    return r;
}
__device__ __forceinline__ uint32_t lds_u32(uint32_t a) {
    uint32_t r;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(r) : "r"(a));
    return r;
}
template <int L>
__device__ __forceinline__ void affine_gather_s(uint32_t body, const double* src_lane, double (&x)[L]) {
    const uint4 b0 = lds_v4(body);
    uint4 b1 = make_uint4(0u, 0u, 0u, 0u);
    if (L > 4) b1 = lds_v4(body + 16u);
    const uint32_t b[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
    for (int j = 0; j < L; ++j) x[j] = ld_gather(src_lane + b[j]);
}
template <int L>
__device__ __forceinline__ double affine_sum_s(uint32_t body, const double (&x)[L]) {
    double acc = 0.0;
#pragma unroll
    for (int j = 0; j < L; j += 2) {
        const double2 vv = lds_d2(body + 32u + 8u * j);
        acc = __dadd_rn(acc, __dmul_rn(vv.x, x[j]));
        if (j + 1 < L) acc = __dadd_rn(acc, __dmul_rn(vv.y, x[j + 1]));
    }
    return acc;
}

// An affine chunk (see the record formats): entry k of lane's row is column base[k] + lane with
// value v[k]; every row is full, so there are no length predicates and no padding.  src_lane =
// src + lane.  The same products in the same stored order as wave_dot.  Gathers and sum are
// separate so that a tile's chunks can have all their gathers in flight together.
template <int L>
__device__ __forceinline__ void affine_gather(const char* body, const double* src_lane, double (&x)[L]) {
    const uint4 b0 = *reinterpret_cast<const uint4*>(body);
    uint4 b1 = make_uint4(0u, 0u, 0u, 0u);
    if (L > 4) b1 = *reinterpret_cast<const uint4*>(body + 16);
    const uint32_t b[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
    for (int j = 0; j < L; ++j) x[j] = ld_gather(src_lane + b[j]);
}
template <int L>
__device__ __forceinline__ double affine_sum(const char* body, const double (&x)[L]) {
    const double2* v = reinterpret_cast<const double2*>(body + 32);
    double acc = 0.0;
#pragma unroll
    for (int j = 0; j < L; j += 2) {
        const double2 vv = v[j >> 1];
        acc = __dadd_rn(acc, __dmul_rn(vv.x, x[j]));
        if (j + 1 < L) acc = __dadd_rn(acc, __dmul_rn(vv.y, x[j + 1]));
    }
    return acc;
}
// Any width 1..8 (warp-uniform guards).
__device__ __forceinline__ double wave_dot_affine_any(const char* body, uint32_t L, const double* src_lane) {
    const uint32_t* b = reinterpret_cast<const uint32_t*>(body);
    const double* v = reinterpret_cast<const double*>(body + 32);
    double x[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) x[j] = (uint32_t)j < L ? ld_gather(src_lane + b[j]) : 0.0;
    double acc = 0.0;
#pragma unroll
    for (int j = 0; j < 8; ++j)
        if ((uint32_t)j < L) acc = __dadd_rn(acc, __dmul_rn(v[j], x[j]));
    return acc;
}
// An affine row whose sum came out NaN (an empty value among its inputs, or a NaN in the data):
// every input re-read with relaxed L2 loads until it is stored, then the sum again in stored
// order.  Cold: a rolled loop, and the hot path keeps no gathered value alive for it.
__device__ __forceinline__ double wave_redo_affine(const char* body, uint32_t L, const double* src_lane, uint32_t* dbg) {
    if (dbg) atomicAdd(dbg, 1u);
    const uint32_t* b = reinterpret_cast<const uint32_t*>(body);
    const double* v = reinterpret_cast<const double*>(body + 32);
    double acc = 0.0;
#pragma unroll 1
    for (uint32_t k = 0; k < L; ++k) {
        const double* p = src_lane + b[k];
        double x = ld_strong_again(p);
        while (wave_empty(x)) {
            __nanosleep(32);
            x = ld_strong_again(p);
        }
        acc = __dadd_rn(acc, __dmul_rn(v[k], x));
    }
    return acc;
}

// A banded chunk (see the record formats).  The row's entries are the template entries its mask
// names, in template (= stored) order: the same products and sums as wave_dot.
__device__ __forceinline__ double wave_dot_banded(const char* body, uint32_t lane, const double* src) {
    const uint32_t meta = reinterpret_cast<const uint16_t*>(body)[lane];
    const char* tb = body + 64 + (meta >> 8) * 32u;
    const uint4 b0 = *reinterpret_cast<const uint4*>(tb), b1 = *reinterpret_cast<const uint4*>(tb + 16);
    const uint32_t b[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
    double x[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) x[j] = (meta >> j) & 1u ? ld_gather(src + (b[j] + lane)) : 0.0;
    const double* v = reinterpret_cast<const double*>(body + 128 + (meta >> 8) * 64u);
    double acc = 0.0;
#pragma unroll
    for (int j = 0; j < 8; ++j)
        if ((meta >> j) & 1u) acc = __dadd_rn(acc, __dmul_rn(v[j], x[j]));
    return acc;
}
// The same row with every in-pass input awaited (first: the source slice is complete); rolled.
__device__ __forceinline__ double wave_row_banded_slow(const char* body, uint32_t lane, const double* src, bool first,
                                                       uint32_t* dbg) {
    if (dbg) atomicAdd(dbg, 1u);
    const uint32_t meta = reinterpret_cast<const uint16_t*>(body)[lane];
    const uint32_t* b = reinterpret_cast<const uint32_t*>(body + 64 + (meta >> 8) * 32u);
    const double* v = reinterpret_cast<const double*>(body + 128 + (meta >> 8) * 64u);
    double acc = 0.0;
#pragma unroll 1
    for (uint32_t k = 0; k < 8; ++k) {
        if (!((meta >> k) & 1u)) continue;
        const double* p = src + (b[k] + lane);
        double x;
        if (first) {
            x = __ldg(p);
        } else {
            x = ld_strong_again(p);
            while (wave_empty(x)) {
                __nanosleep(32);
                x = ld_strong_again(p);
            }
        }
        acc = __dadd_rn(acc, __dmul_rn(v[k], x));
    }
    return acc;
}

// row_epilogue with the wave's rules: in-pass values are awaited, working-vector stores are
// single-copy atomic (KIND 2 never runs here: the polynomial runs the plain powers on the wave and
// forms z from the finished slices, k_poly_combine).
template <int KIND, bool SIGMA>
__device__ __forceinline__ void wave_epilogue(const FusedParams& P, uint32_t s, uint32_t r, uint32_t q,
                                              uint32_t q0, const double* src, double acc) {
    if constexpr (KIND == 1) {
        const double a = P.shift_a[q - 1], b2 = P.shift_b2[q - 1];
        const double own = q == q0 ? __ldg(src + s) : wave_wait(src + s, ld_strong(src + s));
        double own2 = 0.0;
        if (b2 != 0.0) {
            const double* p2 = P.V + (uint64_t)(q - 2) * P.vstride + s;
            own2 = q - 2 >= q0 ? wave_wait(p2, ld_strong(p2)) : __ldg(p2);
        }
        acc = shift_epilogue(acc, a, b2, own, own2);
    }
    st_strong(P.V + (uint64_t)q * P.vstride + s, acc);
    if constexpr (SIGMA) P.out[(uint64_t)q * P.rows + r] = acc;
}

// Tickets are claimed dynamically, in order, from kWaveStreams interleaved counters (stream i hands
// out tickets i, i + S, i + 2S, ... to the warps with warp id = i mod S; one counter alone tops out
// near 1.5 claims/ns).  Each warp holds the ticket it runs, the next one (staged) and the one
// after (descriptor loading), plus one claim in flight, all in increasing order from its stream:
// the tickets in flight are always the ~3 x warps most recently claimed (no warp drifts behind the
// front, which lets a small slack, and so a small L2 window, suffice), and the lowest unfinished
// ticket is always one a warp is running.  A ticket waits only on values of lower tickets, so it
// always progresses: deadlock-free without co-residency.
#ifndef MPKG_WAVE_STREAMS
#define MPKG_WAVE_STREAMS 16
#endif
constexpr uint32_t kWaveStreams = MPKG_WAVE_STREAMS;

// Every warp owns a two-stage shared-memory ring; lane 0 stages the NEXT ticket's chunk record
// with one 1D bulk copy (cp.async.bulk, mbarrier complete_tx, L2 evict_last, evict_first on the
// tile's last use in the pass), so the matrix stream is asynchronous and holds no registers, and a
// ticket costs one dependent hop: the gathers.  Records of chunks wider than 8 entries are not
// staged (their rows take wave_row_slow from global memory).
constexpr uint32_t kWaveWarps = 8;
constexpr uint32_t kWaveThreads = 32 * kWaveWarps;
// A stage holds two general chunk records of width 8; a tile whose records need more (tiles of more
// than two chunks that are not mostly affine) is not staged.
template <int F, bool SIGMA>
__host__ __device__ constexpr uint32_t wave_stage_bytes() {
    return (2u * WaveRec<F, SIGMA>::max_staged + 127u) & ~127u;
}
template <int F, bool SIGMA>
__host__ __device__ constexpr uint32_t wave_smem() { return kWaveWarps * 2 * wave_stage_bytes<F, SIGMA>(); }

__device__ __forceinline__ void bulk_g2s_cta(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar,
                                             uint64_t pol) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
        "[%0], [%1], %2, [%3], %4;" ::"r"(dst),
        "l"(src), "r"(bytes), "r"(bar), "l"(pol)
        : "memory");
}

// Ticket descriptor (k_wave_desc): x = rec_off[kWaveChunks T] (16-byte units, the tile's first
// chunk record; its records are contiguous), y = the bytes to stage / 16 (0: a chunk wider than 8
// entries, nothing staged but the first header) | (q - q0) << 16 | fast-tile width << 24 |
// pair tile << 28 | the tile's last power in the pass << 29 (its records are then evict_first).  The tile index and the chunk
// widths travel in the record headers.
__device__ __forceinline__ uint2 ld_desc(const uint2* p) {
    uint2 r;
    asm("ld.global.nc.L1::no_allocate.v2.u32 {%0,%1}, [%2];" : "=r"(r.x), "=r"(r.y) : "l"(p));
    return r;
}

// Lane 0: stage the records of ticket descriptor d.
template <int F, bool SIGMA>
__device__ __forceinline__ void wave_stage(const FusedParams& P, uint2 d, uint32_t q0, uint32_t q1,
                                           uint32_t stage, uint32_t bar) {
    const uint32_t b16 = d.y & 0xffffu;
    const uint32_t bytes = b16 ? b16 * 16u : WaveRec<F, SIGMA>::hdr;
    asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
    bulk_g2s_cta(stage, P.wrec + (uint64_t)d.x * 16u, bytes, bar, (d.y & (1u << 29)) ? P.pol_first : P.pol_last);
}

template <int KIND, bool SIGMA, int F, bool TRACE>
__global__ void __launch_bounds__(kWaveThreads, kWaveCtas) k_mpk_wave(const __grid_constant__ FusedParams P, uint32_t t0,
                                                            uint32_t t1, uint32_t q0, uint32_t q1, uint32_t fill_lo,
                                                            uint32_t fill_hi) {
    extern __shared__ __align__(128) char wsm[];
    __shared__ __align__(8) uint64_t bars[kWaveWarps][2];
    __shared__ double sdict[F == 1 ? kWaveDictMax + 1 : 1];
    using R = WaveRec<F, SIGMA>;
    constexpr uint32_t SB = wave_stage_bytes<F, SIGMA>();
    const uint32_t lane = threadIdx.x & 31u, wib = threadIdx.x >> 5;
    const uint32_t gw = blockIdx.x * kWaveWarps + wib;
    const uint32_t sid = gw % kWaveStreams;
    uint32_t* const ctr = P.counter + sid * 32u;  // one 128-B line per stream
    char* const ring = wsm + wib * 2u * SB;
    uint32_t ring_s = smem_u32(ring), bar0 = smem_u32(&bars[wib][0]);
    asm volatile("" : "+r"(ring_s), "+r"(bar0));  // opaque: kept in registers, not re-derived per ticket
    if constexpr (F == 1) {
        for (uint32_t i = threadIdx.x; i < P.n_dict; i += blockDim.x) sdict[i] = P.dict[i];
        __syncthreads();
    }
    const double* dict = sdict;
    if (lane == 0) {
        asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(bar0));
        asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(bar0 + 8u));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    auto claim = [&]() -> uint32_t {
        uint32_t k = 0;
        if (lane == 0) k = atomicAdd(ctr, 1u);
        return k;
    };
    uint32_t tbase = t0 + sid;
    asm volatile("" : "+r"(tbase));  // opaque, as above
    auto ticket = [&](uint32_t k) { return tbase + kWaveStreams * __shfl_sync(0xffffffffu, k, 0); };
    uint32_t t = ticket(claim());
    uint32_t tn = ticket(claim());
    uint2 d = t < t1 ? ld_desc(P.wdesc + t) : make_uint2(0u, 0u);
    uint2 dn = tn < t1 ? ld_desc(P.wdesc + tn) : make_uint2(0u, 0u);
    uint32_t kc = claim();
    if (lane == 0) {
        if (t < t1) wave_stage<F, SIGMA>(P, d, q0, q1, ring_s, bar0);
        if (tn < t1) wave_stage<F, SIGMA>(P, dn, q0, q1, ring_s + SB, bar0 + 8u);
    }
    uint32_t it = 0;  // tickets done: stage it & 1, whose completions alternate parity (it >> 1) & 1
    while (t < t1) {
        const uint32_t st = it & 1u;
        const uint32_t tnn = ticket(kc);
        uint2 dnn = make_uint2(0u, 0u);
        if (tnn < t1) {
            dnn = ld_desc(P.wdesc + tnn);
            kc = claim();
        }
        {  // wait for this ticket's stage
            const uint32_t bar = bar0 + 8u * st, par = (it >> 1) & 1u;
            uint32_t done = 0;
            while (!done)
                asm volatile(
                    "{ .reg .pred p; mbarrier.try_wait.parity.shared.b64 p, [%1], %2; selp.u32 %0,1,0,p; }"
                    : "=r"(done)
                    : "r"(bar), "r"(par)
                    : "memory");
        }
        const uint32_t stage_s = ring_s + st * SB;
        const uint32_t q = q0 + ((d.y >> 16) & 15u);
        const uint32_t T = lds_u32(stage_s + R::info);
        // opaque: every gather is then one IMAD.WIDE off this base (otherwise the compiler folds
        // (q-1) * vstride into each gather's index arithmetic)
        const double* src = opaque_ptr(P.V + (uint64_t)(q - 1) * P.vstride);
        const double* src_lane = opaque_ptr(src + lane);  // opaque: one IMAD.WIDE per affine gather
        double tr_acc[TRACE ? kWaveChunks : 1];
        uint32_t tr_off[TRACE ? kWaveChunks : 1];
        // One record for a chunk pair (kWavePair7): chunk b = chunk a 32 rows down the same diagonals.
        auto pair7 = [&](uint32_t sa, double& a0, double& a1) {
            double xa[7], xb[7];
            const uint4 b0 = lds_v4(sa), b1 = lds_v4(sa + 16u);
            const uint32_t b[7] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z};
            const double* src_lane32 = src_lane + 32;
#pragma unroll
            for (int j = 0; j < 7; ++j) xa[j] = ld_gather(src_lane + b[j]);
#pragma unroll
            for (int j = 0; j < 7; ++j) xb[j] = ld_gather(src_lane32 + b[j]);
            a0 = 0.0, a1 = 0.0;
#pragma unroll
            for (int j = 0; j < 7; j += 2) {
                const double2 vv = lds_d2(sa + 32u + 8u * j);
                a0 = __dadd_rn(a0, __dmul_rn(vv.x, xa[j]));
                a1 = __dadd_rn(a1, __dmul_rn(vv.x, xb[j]));
                if (j + 1 < 7) {
                    a0 = __dadd_rn(a0, __dmul_rn(vv.y, xa[j + 1]));
                    a1 = __dadd_rn(a1, __dmul_rn(vv.y, xb[j + 1]));
                }
            }
        };
        // Stores and next-pass fills of a pair whose rows are all real (affine chunks).
        auto pair_store = [&](const char* ra, uint32_t s, double a0, double a1) {
            if (q != q0 && (is_nan_bits(a0) || is_nan_bits(a1))) {
                if (is_nan_bits(a0)) a0 = wave_redo_affine(ra + R::hdr, 7u, src_lane, P.dbg);
                if (is_nan_bits(a1)) a1 = wave_redo_affine(ra + R::affine_bytes + R::hdr, 7u, src_lane, P.dbg);
            }
            if constexpr (KIND == 0 && !SIGMA) {
                double* const dst = P.V + (uint64_t)q * P.vstride;
                st_strong(dst + s, a0);
                st_strong(dst + s + 32u, a1);
            } else {
                wave_epilogue<KIND, SIGMA>(P, s, SIGMA ? R::slot(ra, lane) : s, q, q0, src, a0);
                wave_epilogue<KIND, SIGMA>(P, s + 32u, SIGMA ? R::slot(ra + R::affine_bytes, lane) : s + 32u, q, q0,
                                           src, a1);
            }
            if (q == q1) {
                const double e = __longlong_as_double((long long)kWaveEmpty);
                for (uint32_t f = fill_lo; f < fill_hi; ++f) {
                    P.V[(uint64_t)f * P.vstride + s] = e;
                    P.V[(uint64_t)f * P.vstride + s + 32u] = e;
                }
            }
        };
        if (F == 1 && !TRACE && ((d.y >> 24) & 15u) == 7u) {
            // Fast tile (descriptor bits 24-27): every chunk an affine record of width 7 (the
            // interior of a level-ordered 3D 7-point stencil).  Two chunks at a time: both chunks'
            // gathers are in flight before the first sum.
#pragma unroll
            for (uint32_t c = 0; c < kWaveChunks; c += 2) {
                const uint32_t sa = stage_s + c * R::affine_bytes + R::hdr, sb = sa + R::affine_bytes;
                const uint32_t s = T * kWaveRows + c * 32u + lane;
                double a0, a1;
                if (d.y & (1u << 28)) {  // pair tile
                    pair7(sa, a0, a1);
                } else {
                    double xa[7], xb[7];
                    affine_gather_s<7>(sa, src_lane, xa);
                    affine_gather_s<7>(sb, src_lane, xb);
                    a0 = affine_sum_s<7>(sa, xa);
                    a1 = affine_sum_s<7>(sb, xb);
                }
                pair_store(ring + st * SB + c * R::affine_bytes, s, a0, a1);
            }
        } else {
        const char* stage = ring + st * SB;
        const bool staged = (d.y & 0xffffu) != 0;
        const char* rec = stage;
#pragma unroll 1
        for (uint32_t c = 0; c < kWaveChunks; ++c) {
            if constexpr (TRACE) tr_off[c] = (uint32_t)(rec - stage);
            const uint32_t s = T * kWaveRows + c * 32u + lane;
            if constexpr (F == 1 && !TRACE && kWaveChunks > 2) {
                // a pair of a mixed tile that is itself a width-7 pair: the fast tile's pair code
                if (staged && !(c & 1u) && (R::info4(rec).w & kWavePair7)) {
                    double a0, a1;
                    pair7(stage_s + (uint32_t)(rec - stage) + R::hdr, a0, a1);
                    pair_store(rec, s, a0, a1);
                    rec += 2u * R::affine_bytes;
                    ++c;
                    continue;
                }
            }
            uint32_t L, rr, len, rb;
            double acc = 0.0;
            if (staged && F == 1 && (R::info4(rec).w & kWaveAffine)) {  // an affine chunk: full rows
                const uint4 inf = R::info4(rec);
                L = inf.y;
                rb = inf.z;
                rr = SIGMA ? R::slot(rec, lane) : s;
                len = L;
                const char* body = rec + R::hdr;
                if (L == 7) {
                    double x7[7];
                    affine_gather<7>(body, src_lane, x7);
                    acc = affine_sum<7>(body, x7);
                } else {
                    acc = wave_dot_affine_any(body, L, src_lane);
                }
                if (q != q0 && is_nan_bits(acc)) acc = wave_redo_affine(body, L, src_lane, P.dbg);
            } else if (staged && F == 1 && (R::info4(rec).w & kWaveBanded)) {  // a banded chunk
                const uint4 inf = R::info4(rec);
                L = inf.y;
                rb = inf.z;
                rr = SIGMA ? R::slot(rec, lane) : s;
                len = rr < P.n_rows ? R::len(rec, lane) : 0u;
                const char* body = rec + R::hdr;
                acc = wave_dot_banded(body, lane, src);
                if (q != q0 && is_nan_bits(acc)) acc = wave_row_banded_slow(body, lane, src, false, P.dbg);
            } else if (staged) {  // the record in shared memory (every load below is an LDS)
                const uint4 inf = R::info4(rec);
                L = inf.y;
                rb = inf.z;
                rr = SIGMA ? R::slot(rec, lane) : s;
                len = rr < P.n_rows ? R::len(rec, lane) : 0u;
                const char* body = rec + R::hdr;
                // 7 tested first: the 3D 7-point stencil is the schedule's main customer
                if (__builtin_expect(L == 7, 1)) acc = wave_dot<7, F>(body, lane, len, src, dict);
                else switch (L) {
                    case 0: break;
                    case 1: acc = wave_dot<1, F>(body, lane, len, src, dict); break;
                    case 2: acc = wave_dot<2, F>(body, lane, len, src, dict); break;
                    case 3: acc = wave_dot<3, F>(body, lane, len, src, dict); break;
                    case 4: acc = wave_dot<4, F>(body, lane, len, src, dict); break;
                    case 5: acc = wave_dot<5, F>(body, lane, len, src, dict); break;
                    case 6: acc = wave_dot<6, F>(body, lane, len, src, dict); break;
                    case 7: break;
                    default: acc = wave_dot<8, F>(body, lane, len, src, dict); break;
                }
                // An empty (signalling-NaN) value makes the sum NaN: the row again with every input
                // awaited (slice q0-1 is complete and may hold any bit pattern: never checked).  A
                // NaN in the data takes the same detour and gets the same sum.
                if (L != 0 && q != q0 && is_nan_bits(acc))
                    acc = wave_row_slow<F>(body, L, lane, len, src, false, dict, P.dbg, false);
            } else {  // a tile with a wide chunk: its records from global memory
                const char* h = P.wrec + (uint64_t)d.x * 16u + (uint64_t)(rec - stage);
                const uint4 inf = R::info4(h);
                L = inf.y;
                rb = inf.z;
                rr = SIGMA ? R::slot(h, lane) : s;
                len = rr < P.n_rows ? R::len(h, lane) : 0u;
                if (F == 1 && (inf.w & kWaveBanded))
                    acc = wave_row_banded_slow(h + R::hdr, lane, src, q == q0, P.dbg);
                else
                    acc = wave_row_slow<F>(h + R::hdr, L, lane, len, src, q == q0, dict, P.dbg,
                                           (inf.w & kWaveAffine) != 0);
            }
            if constexpr (TRACE) {  // audit build: every chunk's results are stored after the
                                    // whole tile's inputs are final (one stamp between the two)
                tr_acc[c] = acc;
                if (c + 1 == kWaveChunks) {
                    __syncwarp();
                    if (lane == 0) {
                        const unsigned long long ts = global_ns();
                        P.trace[2ull * ((uint64_t)q * P.n_tiles + T)] = ts;
                        P.trace[2ull * ((uint64_t)q * P.n_tiles + T) + 1] = ts;
                    }
                    __syncwarp();
                    for (uint32_t c2 = 0; c2 < kWaveChunks; ++c2) {
                        const uint32_t s2 = T * kWaveRows + c2 * 32u + lane;
                        const char* h2 = staged ? stage + tr_off[c2] : P.wrec + (uint64_t)d.x * 16u + tr_off[c2];
                        const uint32_t r2 = SIGMA ? R::slot(h2, lane) : s2;
                        if (r2 < P.n_rows) wave_epilogue<KIND, SIGMA>(P, s2, r2, q, q0, src, tr_acc[c2]);
                    }
                }
            } else if (rr < P.n_rows) {
                wave_epilogue<KIND, SIGMA>(P, s, rr, q, q0, src, acc);
            }
            // The tile's last power in this pass also empties its rows of the next pass's in-pass
            // slices (never read by this pass): k_wave_fill runs once per call instead of per pass.
            if (q == q1 && s < (SIGMA ? P.n_slots : P.n_rows)) {
                const double e = __longlong_as_double((long long)kWaveEmpty);
                for (uint32_t f = fill_lo; f < fill_hi; ++f) P.V[(uint64_t)f * P.vstride + s] = e;
            }
            rec += rb;
        }
        }
        __syncwarp();  // every lane is done with the stage: refill it with ticket tnn
        if (lane == 0 && tnn < t1) wave_stage<F, SIGMA>(P, dnn, q0, q1, ring_s + st * SB, bar0 + 8u * st);
        t = tn, d = dn, tn = tnn, dn = dnn;
        ++it;
    }
}

// Value dictionary (setup): the distinct value bit patterns of the SELL arrays (padding entries
// are 0.0 and count), inserted into an open-addressing table of 512 slots (empty = kDictEmpty);
// warps first merge equal values (__match_any_sync), so only warp-unique values hit the table.
// *count = distinct values (stops counting past 512: the dict format is then not used).
constexpr unsigned long long kDictEmpty = 0xfff8dead0000beefull;  // a NaN payload no value takes here
constexpr uint32_t kDictSlots = 512;
__device__ __forceinline__ uint32_t dict_hash(unsigned long long b) {
    b ^= b >> 33;
    b *= 0xff51afd7ed558ccdull;
    b ^= b >> 33;
    return (uint32_t)b & (kDictSlots - 1);
}
__global__ void k_dict_insert(const double* __restrict__ vals, uint64_t n, unsigned long long* table,
                              uint32_t* count) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i - threadIdx.x % 32 < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const bool in = i < n;
        const unsigned long long b = in ? (unsigned long long)__double_as_longlong(vals[i]) : kDictEmpty;
        const uint32_t peers = __match_any_sync(0xffffffffu, b);
        const bool leader = (threadIdx.x & 31u) == (uint32_t)(__ffs(peers) - 1);
        if (!in || !leader || b == kDictEmpty) continue;
        if (*reinterpret_cast<volatile uint32_t*>(count) > kDictSlots / 2) return;
        uint32_t h = dict_hash(b);
        for (uint32_t probe = 0; probe < kDictSlots; ++probe, h = (h + 1) & (kDictSlots - 1)) {
            const unsigned long long cur = table[h];
            if (cur == b) break;
            if (cur == kDictEmpty) {
                const unsigned long long prev = atomicCAS(table + h, kDictEmpty, b);
                if (prev == kDictEmpty) {
                    atomicAdd(count, 1u);
                    break;
                }
                if (prev == b) break;
            }
        }
    }
}
__device__ __forceinline__ uint32_t dict_index(const unsigned long long* table, const uint16_t* slot_ix,
                                               unsigned long long b) {
    uint32_t h = dict_hash(b);
    while (table[h] != b) h = (h + 1) & (kDictSlots - 1);
    return slot_ix[h];
}

// A chunk's rows against at most two row templates (banded records): the lane's keys (column -
// lane) and value bits; template t = the longest row not yet matched (lowest lane on ties); a row
// matches when each of its entries equals a template entry (key and value) at increasing template
// positions.  Returns whether every real row matched; meta = template << 8 | entry mask, tk / tv =
// the templates (unused positions 0), tl[t] = their lengths.
__device__ bool banded_match(const uint32_t* __restrict__ cols, const double* __restrict__ vals, uint64_t o,
                             uint32_t L, uint32_t len, uint32_t lane, uint32_t& meta, uint32_t (&tk)[2][8],
                             unsigned long long (&tv)[2][8], uint32_t (&tl)[2]) {
    uint32_t key[8];
    unsigned long long vb[8];
    const uint32_t Lp = L & ~1u;
#pragma unroll
    for (uint32_t k = 0; k < 8; ++k) {
        key[k] = 0;
        vb[k] = 0;
        if (k < len) {
            const uint32_t e = k < Lp ? (k >> 1) * 64u + lane * 2u + (k & 1u) : Lp * 32u + lane;
            key[k] = cols[o + e] - lane;
            vb[k] = (unsigned long long)__double_as_longlong(vals[o + e]);
        }
    }
    bool open = true;
    meta = 0;
    tl[0] = tl[1] = 0;
#pragma unroll
    for (int t = 0; t < 2; ++t) {
        const uint32_t want = open ? len + 1u : 0u;
        const uint32_t best = __reduce_max_sync(0xffffffffu, want);
        const uint32_t src = best ? (uint32_t)__ffs(__ballot_sync(0xffffffffu, want == best)) - 1u : 0u;
        const uint32_t T_len = best ? best - 1u : 0u;
        tl[t] = T_len;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const uint32_t kk = __shfl_sync(0xffffffffu, key[k], src);
            const unsigned long long vv = __shfl_sync(0xffffffffu, vb[k], src);
            tk[t][k] = (uint32_t)k < T_len ? kk : 0u;
            tv[t][k] = (uint32_t)k < T_len ? vv : 0ull;
        }
        if (open) {
            uint32_t mk = 0;
            int last = -1;
            bool all = true;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                if ((uint32_t)j >= len) continue;
                int at = -1;
#pragma unroll
                for (int k = 0; k < 8; ++k)
                    if ((uint32_t)k < T_len && tk[t][k] == key[j] && tv[t][k] == vb[j] && k > last && at < 0) at = k;
                if (at < 0) all = false;
                else {
                    mk |= 1u << at;
                    last = at;
                }
            }
            if (all) {
                open = false;
                meta = mk | (uint32_t)t << 8;
            }
        }
    }
    return !__any_sync(0xffffffffu, open);
}

// Affine and banded chunks (setup): one warp per SELL chunk; flags[T] = 1 (affine) when the chunk
// has width 1..8, 32 real full rows, and every entry k is column c_k + lane with one value bit
// pattern in all lanes; else 2 (banded) when its rows fit two templates (banded_match); else 0.
__global__ void k_wave_affine(const uint32_t* __restrict__ cols, const double* __restrict__ vals,
                              const uint32_t* __restrict__ row_len, const uint32_t* __restrict__ slot_row,
                              const uint64_t* __restrict__ chunk_off, uint32_t n_chunks, uint32_t n_rows,
                              int banded, uint8_t* __restrict__ flags) {
    const uint32_t lane = threadIdx.x & 31u;
    for (uint64_t T = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5; T < n_chunks;
         T += ((uint64_t)gridDim.x * blockDim.x) >> 5) {
        const uint64_t o = chunk_off[T];
        const uint32_t L = (uint32_t)((chunk_off[T + 1] - o) >> 5);
        const bool narrow = L >= 1 && L <= 8;
        bool ok = narrow;
        uint32_t len = 0;
        bool real = false;
        if (narrow) {
            const uint32_t row = slot_row ? slot_row[T * 32 + lane] : (uint32_t)(T * 32 + lane);
            real = row < n_rows;
            len = real ? row_len[T * 32 + lane] : 0u;
            ok = real && len == L;
            const uint32_t Lp = L & ~1u;
            for (uint32_t k = 0; k < L; ++k) {
                const uint32_t e = k < Lp ? (k >> 1) * 64u + lane * 2u + (k & 1u) : Lp * 32u + lane;
                const uint32_t c = cols[o + e];
                const unsigned long long b = (unsigned long long)__double_as_longlong(vals[o + e]);
                const uint32_t c0 = __shfl_sync(0xffffffffu, c, 0);
                const unsigned long long b0 = __shfl_sync(0xffffffffu, b, 0);
                ok = ok && c0 <= 0xffffffffu - 31u && c == c0 + lane && b == b0;
            }
        }
        ok = __all_sync(0xffffffffu, ok);
        uint32_t f = ok ? 1u : 0u;
        if (!ok && narrow && banded) {
            uint32_t meta, tk[2][8], tl[2];
            unsigned long long tv[2][8];
            if (banded_match(cols, vals, o, L, len, lane, meta, tk, tv, tl)) f = 2u;
        }
        if (lane == 0) flags[T] = (uint8_t)f;
    }
}

// Chunk records from the executor's SELL arrays: one warp per chunk; records past the SELL (the
// last tile's padding) are empty (lengths 0, width 0, slot rows ~0).
template <int F>
__global__ void k_wave_pack(const uint32_t* __restrict__ cols, const double* __restrict__ vals,
                            const uint32_t* __restrict__ row_len, const uint32_t* __restrict__ slot_row,
                            const uint64_t* __restrict__ chunk_off, uint32_t n_chunks, uint32_t n_rec,
                            const uint32_t* __restrict__ rec_off, char* __restrict__ rec,
                            const unsigned long long* __restrict__ table, const uint16_t* __restrict__ slot_ix,
                            const uint8_t* __restrict__ affine) {
    const uint32_t lane = threadIdx.x & 31u;
    const uint32_t lb = F == 0 ? 128u : 32u;
    for (uint64_t T = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5; T < n_rec;
         T += ((uint64_t)gridDim.x * blockDim.x) >> 5) {
        char* r = rec + (uint64_t)rec_off[T] * 16u;
        const bool real = T < n_chunks;
        const uint32_t len = real ? row_len[T * 32 + lane] : 0u;
        if (F == 0) reinterpret_cast<uint32_t*>(r)[lane] = len;
        else reinterpret_cast<uint8_t*>(r)[lane] = (uint8_t)len;
        const uint64_t o = real ? chunk_off[T] : 0, ne = real ? chunk_off[T + 1] - o : 0;
        const uint32_t L = (uint32_t)(ne >> 5);
        const bool aff = F == 1 && real && affine && affine[T] == 1;
        const bool band = F == 1 && real && affine && affine[T] == 2;
        if (lane < 4)  // info: tile, width, this record's bytes, flags
            reinterpret_cast<uint32_t*>(r + lb)[lane] =
                lane == 0 ? (uint32_t)(T / kWaveChunks) : lane == 1 ? L : lane == 2 ? (rec_off[T + 1] - rec_off[T]) * 16u
                                                                               : (aff ? kWaveAffine : band ? kWaveBanded : 0u);
        uint32_t hdr = lb + 16;
        if (slot_row) {
            reinterpret_cast<uint32_t*>(r + hdr)[lane] = real ? slot_row[T * 32 + lane] : 0xffffffffu;
            hdr += 128;
        }
        if (aff) {  // base[8] u32 | v[8] f64: lane 0's entries (every lane's column is base + lane)
            if (lane < 8) {
                const uint32_t k = lane, Lp = L & ~1u;
                const uint64_t e = k < Lp ? (k >> 1) * 64u + (k & 1u) : Lp * 32u;
                reinterpret_cast<uint32_t*>(r + hdr)[k] = k < L ? cols[o + e] : 0u;
                reinterpret_cast<double*>(r + hdr + 32)[k] = k < L ? vals[o + e] : 0.0;
            }
            continue;
        }
        if (band) {  // meta[32] u16 | base[2][8] u32 | v[2][8] f64
            uint32_t meta, tk[2][8], tl[2];
            unsigned long long tv[2][8];
            banded_match(cols, vals, o, L, len, lane, meta, tk, tv, tl);
            reinterpret_cast<uint16_t*>(r + hdr)[lane] = (uint16_t)meta;
            if (lane < 16) {
                uint32_t kv = 0;
                unsigned long long vv = 0;
#pragma unroll
                for (int t = 0; t < 2; ++t)
#pragma unroll
                    for (int k = 0; k < 8; ++k)
                        if (lane == (uint32_t)(t * 8 + k)) {
                            kv = tk[t][k];
                            vv = tv[t][k];
                        }
                reinterpret_cast<uint32_t*>(r + hdr + 64)[lane] = kv;
                reinterpret_cast<unsigned long long*>(r + hdr + 128)[lane] = vv;
            }
            continue;
        }
        uint32_t* rc = reinterpret_cast<uint32_t*>(r + hdr);
        for (uint64_t e = lane; e < ne; e += 32) rc[e] = cols[o + e];
        if (F == 0) {
            double* rv = reinterpret_cast<double*>(r + hdr + 4 * ne);
            for (uint64_t e = lane; e < ne; e += 32) rv[e] = vals[o + e];
        } else {
            uint8_t* ri = reinterpret_cast<uint8_t*>(r + hdr + 4 * ne);
            const uint32_t L8 = (L + 7u) & ~7u;
            for (uint32_t k = 0; k < L8; ++k) {  // lane-major: lane's L8 bytes, padding index of 0.0
                double v = 0.0;
                if (k < L) {
                    const uint32_t Lp = L & ~1u;
                    const uint32_t e = k < Lp ? (k >> 1) * 64u + lane * 2u + (k & 1u) : Lp * 32u + lane;
                    v = vals[o + e];
                }
                ri[lane * L8 + k] = (uint8_t)dict_index(table, slot_ix, (unsigned long long)__double_as_longlong(v));
            }
        }
    }
}

// Pairs (setup, after k_wave_pack): a chunk pair (2i, 2i+1 of a tile) whose records are both
// affine of one width and whose second chunk is the first 32 rows further down the same diagonals
// (bases + 32, the same values) is marked in the first record (info.w |= kWavePair7 when the width
// is 7); a fast tile all of whose pairs are such gets bit 1 of its tile code (pair tile): the
// engine then reads one record per chunk pair.  One thread per tile.
__global__ void k_wave_pairs(char* __restrict__ rec, const uint32_t* __restrict__ rec_off, uint32_t n_tiles,
                             uint32_t len_bytes, uint32_t hdr, uint8_t* __restrict__ code) {
    for (uint64_t T = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; T < n_tiles;
         T += (uint64_t)gridDim.x * blockDim.x) {
        bool all = true;
        for (uint32_t c = 0; c < kWaveChunks; c += 2) {
            char* ra = rec + (uint64_t)rec_off[T * kWaveChunks + c] * 16u;
            const char* rb = rec + (uint64_t)rec_off[T * kWaveChunks + c + 1] * 16u;
            uint32_t* ia = reinterpret_cast<uint32_t*>(ra + len_bytes);
            const uint32_t* ib = reinterpret_cast<const uint32_t*>(rb + len_bytes);
            bool ok = (ia[3] & kWaveAffine) && (ib[3] & kWaveAffine) && ia[1] == ib[1];
            const uint32_t L = ia[1];
            const char *a = ra + hdr, *b = rb + hdr;
            for (int k = 0; k < 8 && ok; ++k) {
                const uint32_t ba = reinterpret_cast<const uint32_t*>(a)[k], bb = reinterpret_cast<const uint32_t*>(b)[k];
                const unsigned long long va = reinterpret_cast<const unsigned long long*>(a + 32)[k];
                const unsigned long long vb = reinterpret_cast<const unsigned long long*>(b + 32)[k];
                ok = va == vb && ((uint32_t)k < L ? bb == ba + 32u : bb == ba);
            }
            if (ok && L == 7) ia[3] |= kWavePair7;
            all = all && ok;
        }
        if (all && (code[T] >> 4) != 0) code[T] |= 2u;
    }
}

// Descriptors of a pass's tickets from the host codes (T | q << 24, kLastUse ignored: the last use
// is q == q1); narrow[T] bit 0: every chunk of the tile is at most 8 entries wide (staged), bits
// 4-7: the width of a fast tile (all chunks affine records of that width), 0 otherwise, bit 1:
// a pair tile (k_wave_pairs).
__global__ void k_wave_desc(const uint32_t* __restrict__ codes, uint64_t n, const uint32_t* __restrict__ rec_off,
                            const uint8_t* __restrict__ narrow, uint32_t q0, uint32_t q1, uint2* __restrict__ out) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t code = codes[i];
        const uint32_t T = code & 0xffffffu, q = (code >> 24) & 63u;
        const uint32_t o = rec_off[(uint64_t)T * kWaveChunks];
        const uint32_t code8 = narrow[T];  // bit 0: staged (narrow chunks); bits 4-7: fast-tile width
        const uint32_t b16 = (code8 & 1u) ? rec_off[(uint64_t)(T + 1) * kWaveChunks] - o : 0u;
        out[i] = make_uint2(o, b16 | (q - q0) << 16 | (code8 >> 4) << 24 | ((code8 >> 1) & 1u) << 28 |
                                   (q == q1 ? 1u << 29 : 0u));
    }
}

__global__ void k_l2_policies(uint64_t* out) {
    out[0] = l2_policy_first();
    out[1] = l2_policy_last();
}

__global__ void k_wave_fill(double* __restrict__ V, uint64_t vstride, uint64_t n, uint32_t q_lo, uint32_t q_hi) {
    const double e = __longlong_as_double((long long)kWaveEmpty);
    for (uint32_t q = q_lo; q < q_hi; ++q)
        for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
            V[q * vstride + i] = e;
}

__device__ __forceinline__ void mbar_init_n(uint64_t* bar, uint32_t n) {
    asm volatile("mbarrier.init.shared.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(n));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                         uint64_t pol) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
        "[%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
        : "memory");
}
// 8-byte asynchronous gather global -> shared (no register destination).
__device__ __forceinline__ void gather8(void* dst, const double* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
// Arrives on `bar` once all of this thread's earlier cp.async copies have landed.
__device__ __forceinline__ void gather_arrive(uint64_t* bar) {
    asm volatile("cp.async.mbarrier.arrive.noinc.shared.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// Asynchronous-gather variant ("kernel" knob 4).  The row loop of the other variants holds its
// in-flight loads in registers, so memory parallelism per SM is capped by the register file and
// a row needs ~len/2 dependent round trips: ~230K rows (~74 MB of C2's matrix) must be in flight
// to cover HBM latency, which leaves no L2 room for reuse across powers.  Here each CTA runs a
// ring of P.stages shared-memory slots, each holding one tile:
//   cols[ne_max] u32 | vals[ne_max] f64 | xs[ne_max] f64   (the tile's SELL entries, in order)
// P.n_prod producer warps fill slots: per ticket, (1) bulk-copy the tile's columns and values
// (TMA, mbarrier complete_tx), (2) poll + acquire the tile's dependencies for power q-1,
// (3) gather every x_{q-1}[col] of the tile into the slot with 8-byte cp.async copies (landing in
// shared memory: no registers held) and (4) signal the slot.  P.n_cgroups consumer groups of
// tile_rows threads (one thread per row) sum their rows' products in stored order straight from
// shared memory (bitwise identical to the row loop) and publish the tile.
// Tickets are assigned statically: iteration i of CTA b is ticket i*gridDim.x + b; producer warp
// j owns iterations i = j mod n_prod, consumer group g owns i = g mod n_cgroups, and every role
// walks its iterations in increasing order.  The lowest unfinished ticket's CTA has finished all
// its earlier iterations, so its producer (slot free, dependencies all lower) and its consumer
// group both make progress: deadlock-free.
constexpr uint32_t kMaxSlots = 16;

template <int KIND, bool SIGMA>
__global__ void __launch_bounds__(512) k_mpk_async(const __grid_constant__ FusedParams P) {
    extern __shared__ __align__(128) char smem[];
    __shared__ __align__(8) uint64_t full_mat[kMaxSlots];
    __shared__ __align__(8) uint64_t full_x[kMaxSlots];
    __shared__ __align__(8) uint64_t empty[kMaxSlots];
    __shared__ uint32_t s_code[kMaxSlots];
    const uint32_t tid = threadIdx.x;
    const uint32_t tr = P.tile_rows;
    const uint32_t nc = P.n_cgroups * tr;  // consumer threads
    const uint32_t S = P.stages;
    const uint32_t ne_max = P.buf_bytes / 20u;
    if (tid == 0) {
        for (uint32_t i = 0; i < S; ++i) {
            mbar_init_n(&full_mat[i], 1);
            mbar_init_n(&full_x[i], 32);
            mbar_init_n(&empty[i], 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const uint32_t b = blockIdx.x;
    const uint32_t i_end = b < P.n_tickets ? (P.n_tickets - b + gridDim.x - 1) / gridDim.x : 0u;
    if (tid >= nc) {
        // ---------------- producer warps ----------------
        // Iteration i: prepare (slot free -> ticket code -> TMA of columns + values), then, one
        // iteration later in this warp's order, dependencies -> gathers.  The next iteration's
        // TMA is issued right after the current gathers, so it overlaps their round trip.
        const uint32_t lane = tid & 31u;
        const uint32_t w = (tid - nc) >> 5;
        struct Prep {
            uint32_t code, T, q, ne;
        };
        auto prepare = [&](uint32_t i) -> Prep {
            const uint32_t slot = i % S;
            if (i >= S) mbar_wait(&empty[slot], ((i / S) - 1u) & 1u);
            Prep pr{kNoTicket, 0, 0, 0};
            if (i >= i_end) {
                if (lane == 0) {
                    s_code[slot] = kNoTicket;
                    mbar_arrive(&full_mat[slot]);
                }
                gather_arrive(&full_x[slot]);
                return pr;
            }
            pr.code = P.tickets[i * gridDim.x + b];
            pr.T = pr.code & 0xffffffu;
            pr.q = (pr.code >> 24) & 63u;
            const uint64_t e0 = P.tile_off[pr.T];
            pr.ne = (uint32_t)(P.tile_off[pr.T + 1] - e0);
            if (lane == 0) {
                char* st = smem + slot * P.buf_bytes;
                s_code[slot] = pr.code;
                const uint64_t pol = l2_policy(pr.code & kLastUse);
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                mbar_expect_tx(&full_mat[slot], pr.ne * 12u);
                if (pr.ne) {
                    bulk_g2s(st, P.cols + e0, pr.ne * 4u, &full_mat[slot], pol);
                    bulk_g2s(st + ne_max * 4u, P.vals + e0, pr.ne * 8u, &full_mat[slot], pol);
                }
            }
            return pr;
        };
        uint32_t i = w;
        Prep cur = prepare(i);
        while (i < i_end) {
            const uint32_t slot = i % S;
            if (cur.q > 1) {
                const uint32_t r0 = P.dep_ptr[cur.T], r1 = P.dep_ptr[cur.T + 1];
                while (!__all_sync(0xffffffffu, deps_ready<false>(P, r0, r1, cur.q - 1, lane, 32u))) __nanosleep(32);
                (void)deps_ready<true>(P, r0, r1, cur.q - 1, lane, 32u);  // acquire each unit once
                __syncwarp();
            }
            // release (cta) after the acquires: consumers waiting on full_mat may read data of the
            // dependency tiles (own-row values, polynomial accumulator) from global memory
            if (lane == 0) mbar_arrive(&full_mat[slot]);
            mbar_wait(&full_mat[slot], (i / S) & 1u);  // columns landed
            const char* st = smem + slot * P.buf_bytes;
            const uint32_t* cs = reinterpret_cast<const uint32_t*>(st);
            double* xs = reinterpret_cast<double*>(const_cast<char*>(st) + ne_max * 12u);
            const double* src = P.V + (uint64_t)(cur.q - 1) * P.vstride;
            uint32_t e = lane;
            for (; e + 7u * 32u < cur.ne; e += 8u * 32u) {  // ne is a multiple of 32
                uint32_t c[8];
#pragma unroll
                for (int j = 0; j < 8; ++j) c[j] = cs[e + j * 32u];
#pragma unroll
                for (int j = 0; j < 8; ++j) gather8(xs + e + j * 32u, src + c[j]);
            }
            for (; e < cur.ne; e += 32u) gather8(xs + e, src + cs[e]);
            gather_arrive(&full_x[slot]);
            i += P.n_prod;
            cur = prepare(i);
        }
        // terminal markers for every consumer group's first iteration past the end
        for (i += P.n_prod; i < i_end + P.n_cgroups; i += P.n_prod) (void)prepare(i);
        return;
    }
    // ---------------- consumer groups: one thread per tile row ----------------
    const uint32_t g = tid / tr, row = tid - g * tr;
    for (uint32_t i = g;; i += P.n_cgroups) {
        const uint32_t slot = i % S;
        const uint32_t ph = (i / S) & 1u;
        mbar_wait(&full_mat[slot], ph);
        const uint32_t code = s_code[slot];
        if (code == kNoTicket) {
            if (row == 0) mbar_arrive(&empty[slot]);
            return;
        }
        const uint32_t T = code & 0xffffffu;
        const uint32_t q = (code >> 24) & 63u;
        const double* src = P.V + (uint64_t)(q - 1) * P.vstride;
        const uint32_t s = T * tr + row;
        const uint32_t r = SIGMA ? (s < P.n_slots ? P.slot_row[s] : 0xffffffffu) : s;
        uint32_t len = 0, rb = 0, L = 0;
        if (r < P.n_rows) {
            len = P.row_len[s];
            const uint64_t off = P.chunk_off[s >> 5];
            L = (uint32_t)((P.chunk_off[(s >> 5) + 1] - off) >> 5);
            rb = (uint32_t)(off - P.tile_off[T]);
        }
        mbar_wait(&full_x[slot], ph);
        if (r < P.n_rows) {
            const char* st = smem + slot * P.buf_bytes;
            const double* vs = reinterpret_cast<const double*>(st + ne_max * 4u) + rb;
            const double* xs = vs + ne_max;
            const uint32_t lane = s & 31u;
            const uint32_t Lp = L & ~1u;
            double acc = 0.0;
            uint32_t k = 0;
            for (; k + 1 < len && k < Lp; k += 2) {  // whole pairs
                const double2 v = *reinterpret_cast<const double2*>(vs + (k >> 1) * 64u + lane * 2u);
                const double2 x = *reinterpret_cast<const double2*>(xs + (k >> 1) * 64u + lane * 2u);
                acc = __dadd_rn(acc, __dmul_rn(v.x, x.x));
                acc = __dadd_rn(acc, __dmul_rn(v.y, x.y));
            }
            for (; k < len; ++k) {
                const uint32_t e = sell_pos(k, Lp, lane);
                acc = __dadd_rn(acc, __dmul_rn(vs[e], xs[e]));
            }
            row_epilogue<KIND, SIGMA>(P, s, r, q, src, acc);
        }
        asm volatile("bar.sync %0, %1;" ::"r"(1u + g), "r"(tr) : "memory");  // group done with the slot
        if (row == 0) {
            mbar_arrive(&empty[slot]);  // the slot can be refilled while the publish fence drains
            publish(P, T, q);
        }
    }
}

// Warp-tile variant ("kernel" knob 2): each warp owns one 32-row SELL chunk of the tile.
// Phase 1 walks the chunk's entries FLAT (lane l takes entries l, l+32, ...: coalesced column /
// value loads, all x-gathers independent, software-pipelined in batches of U) and writes every
// product v*x[col] to the warp's shared-memory slice at the same flat position; after
// __syncwarp, phase 2 lets lane r sum ITS row's products in stored order (bitwise identical to
// the row loop: same products, same additions, same order).  A row costs ~L/(32U) pipelined
// round trips instead of ~L/2 dependent ones; no CTA-wide barrier inside the tile.  Chunks wider
// than `wt_lmax` fall back to the row loop.
template <int KIND, bool SIGMA, int U>
__global__ void __launch_bounds__(128) k_mpk_warptile(const __grid_constant__ FusedParams P) {
    extern __shared__ __align__(16) double prod[];  // [4 warps][32 * wt_lmax]
    __shared__ uint32_t s_ticket[2];
    const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
    double* my = prod + (uint64_t)warp * 32u * P.wt_lmax;
    if (tid == 0) s_ticket[0] = atomicAdd(P.counter, 1u);
    __syncthreads();
    for (uint32_t buf = 0;; buf ^= 1u) {
        const uint32_t t = s_ticket[buf];
        if (t >= P.n_tickets) return;
        if (tid == 0) s_ticket[buf ^ 1u] = atomicAdd(P.counter, 1u);
        const uint32_t code = P.tickets[t];
        const uint32_t T = code & 0xffffffu;
        const uint32_t q = (code >> 24) & 63u;
        if (q > 1) {
            const uint32_t r0 = P.dep_ptr[T], r1 = P.dep_ptr[T + 1];
            while (!__syncthreads_and(deps_ready<false>(P, r0, r1, q - 1, tid, 128u))) __nanosleep(32);
            (void)deps_ready<true>(P, r0, r1, q - 1, tid, 128u);  // acquire each unit once
            __syncthreads();
        }
        const double* src = P.V + (uint64_t)(q - 1) * P.vstride;
        const uint64_t pol = l2_policy(code & kLastUse);
        const uint32_t s = T * 128u + tid;  // this lane's row slot; the warp's chunk = s >> 5
        const uint32_t r = SIGMA ? (s < P.n_slots ? P.slot_row[s] : 0xffffffffu) : s;
        const bool chunk_ok = (T * 128u + warp * 32u) < P.n_slots;
        uint64_t off = 0;
        uint32_t L = 0;
        if (chunk_ok) {
            off = P.chunk_off[s >> 5];
            L = (uint32_t)((P.chunk_off[(s >> 5) + 1] - off) >> 5);
        }
        double acc = 0.0;
        const uint32_t len = (r < P.n_rows) ? P.row_len[s] : 0u;
        if (chunk_ok && L <= P.wt_lmax) {
            // phase 1: flat products of the chunk (32*L entries), U gathers in flight per lane
            const uint32_t ne = 32u * L;
            const uint32_t* cc = P.cols + off;
            const double* vv = P.vals + off;
            for (uint32_t e0 = 0; e0 < ne; e0 += 32u * U) {
                uint32_t c[U];
                double v[U], x[U];
#pragma unroll
                for (int j = 0; j < U; ++j) {
                    const uint32_t e = e0 + j * 32u + lane;
                    c[j] = e < ne ? ld_mat_u32(cc + e, pol) : 0u;
                    v[j] = e < ne ? ld_mat_d(vv + e, pol) : 0.0;
                }
#pragma unroll
                for (int j = 0; j < U; ++j) {
                    const uint32_t e = e0 + j * 32u + lane;
                    x[j] = e < ne ? (q == 1 ? ld_vec<true>(src + c[j]) : ld_vec<false>(src + c[j])) : 0.0;
                }
#pragma unroll
                for (int j = 0; j < U; ++j) {
                    const uint32_t e = e0 + j * 32u + lane;
                    if (e < ne) my[e] = __dmul_rn(v[j], x[j]);
                }
            }
            __syncwarp();
            // phase 2: lane = row, stored-order sum of its products
            if (r < P.n_rows) acc = sell_row_sum_smem(my, 0u, L, lane, len);
            __syncwarp();
        } else if (r < P.n_rows) {
            acc = q == 1 ? sell_row_dot_pipe<true>(P.cols, P.vals, off, L, lane, len, src, pol)
                         : sell_row_dot_pipe<false>(P.cols, P.vals, off, L, lane, len, src, pol);
        }
        if (r < P.n_rows) {
            if constexpr (KIND == 1) {
                const double a = P.shift_a[q - 1], b2 = P.shift_b2[q - 1];
                const double own = src[s];
                const double own2 = b2 != 0.0 ? P.V[(uint64_t)(q - 2) * P.vstride + s] : 0.0;
                acc = shift_epilogue(acc, a, b2, own, own2);
            }
            P.V[(uint64_t)q * P.vstride + s] = acc;
            if constexpr (SIGMA) P.out[(uint64_t)q * P.rows + r] = acc;
            if constexpr (KIND == 2) {
                double zr;
                if (q == 1)
                    zr = __dadd_rn(__dmul_rn(P.coef[0], src[s]), __dmul_rn(P.coef[1], acc));
                else
                    zr = __dadd_rn(P.zs[s], __dmul_rn(P.coef[q], acc));
                P.zs[s] = zr;
                if (SIGMA && q == P.p) P.z[r] = zr;
            }
        }
        __syncthreads();
        if (tid == 0) publish(P, T, q);
    }
}

// Sparse-table range maximum over r[0..n).
struct RangeMax {
    std::vector<std::vector<int64_t>> t;
    explicit RangeMax(const std::vector<int64_t>& r) {
        const size_t n = r.size();
        t.push_back(r);
        for (size_t w = 1; (w << 1) <= n; w <<= 1) {
            const auto& prev = t.back();
            std::vector<int64_t> cur(n - (w << 1) + 1);
            for (size_t i = 0; i < cur.size(); ++i) cur[i] = std::max(prev[i], prev[i + w]);
            t.push_back(std::move(cur));
        }
    }
    int64_t query(uint32_t lo, uint32_t hi) const {  // inclusive
        const uint32_t len = hi - lo + 1;
        const int k = 31 - __builtin_clz(len);
        return std::max(t[k][lo], t[k][hi - (1u << k) + 1]);
    }
};

template <int G>
void configure_kernels(uint32_t smem_bytes) {
    const void* ks[] = {(const void*)k_mpk_fused<0, false, G>, (const void*)k_mpk_fused<0, true, G>,
                        (const void*)k_mpk_fused<1, false, G>, (const void*)k_mpk_fused<1, true, G>,
                        (const void*)k_mpk_fused<2, false, G>, (const void*)k_mpk_fused<2, true, G>};
    for (const void* k : ks)
        MPKG_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_bytes));
}

void configure_warptile(uint32_t lmax) {
    const int smem = (int)(128 * lmax * 8);
    const void* ks[] = {
        (const void*)k_mpk_warptile<0, false, 4>, (const void*)k_mpk_warptile<0, true, 4>,
        (const void*)k_mpk_warptile<1, false, 4>, (const void*)k_mpk_warptile<1, true, 4>,
        (const void*)k_mpk_warptile<2, false, 4>, (const void*)k_mpk_warptile<2, true, 4>,
        (const void*)k_mpk_warptile<0, false, 8>, (const void*)k_mpk_warptile<0, true, 8>,
        (const void*)k_mpk_warptile<1, false, 8>, (const void*)k_mpk_warptile<1, true, 8>,
        (const void*)k_mpk_warptile<2, false, 8>, (const void*)k_mpk_warptile<2, true, 8>};
    for (const void* k : ks)
        MPKG_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
}

// Variable tiles (long rows) always come with wide dependency runs (superblock counters).
template <bool SIGMA, bool VT, bool SB>
std::array<const void*, 3> lean_kinds() {
    return {(const void*)k_mpk_lean<0, SIGMA, VT, SB>, (const void*)k_mpk_lean<1, SIGMA, VT, SB>,
            (const void*)k_mpk_lean<2, SIGMA, VT, SB>};
}
std::array<const void*, 3> lean_variants(bool sigma, bool vt, bool sb) {
    if (sigma) return vt ? lean_kinds<true, true, true>() : sb ? lean_kinds<true, false, true>() : lean_kinds<true, false, false>();
    return vt ? lean_kinds<false, true, true>() : sb ? lean_kinds<false, false, true>() : lean_kinds<false, false, false>();
}

template <int KIND, bool SIGMA>
void launch_lean(bool sb, int grid, int nt, cudaStream_t st, const FusedParams& P) {
    if (P.tile_start)
        k_mpk_lean<KIND, SIGMA, true, true><<<grid, nt, kLeanRingBytes, st>>>(P);
    else if (sb)
        k_mpk_lean<KIND, SIGMA, false, true><<<grid, nt, 0, st>>>(P);
    else
        k_mpk_lean<KIND, SIGMA, false, false><<<grid, nt, 0, st>>>(P);
}


template <int U>
void launch_warptile(int kind, bool sigma, int grid, uint32_t smem, cudaStream_t st,
                     const FusedParams& P) {
    switch (kind * 2 + (sigma ? 1 : 0)) {
        case 0: k_mpk_warptile<0, false, U><<<grid, 128, smem, st>>>(P); break;
        case 1: k_mpk_warptile<0, true, U><<<grid, 128, smem, st>>>(P); break;
        case 2: k_mpk_warptile<1, false, U><<<grid, 128, smem, st>>>(P); break;
        case 3: k_mpk_warptile<1, true, U><<<grid, 128, smem, st>>>(P); break;
        case 4: k_mpk_warptile<2, false, U><<<grid, 128, smem, st>>>(P); break;
        default: k_mpk_warptile<2, true, U><<<grid, 128, smem, st>>>(P); break;
    }
}

Executor& get_executor(mpkg_ctx_s* ctx, mpkg_plan_s* P, mpkg_csr_s* A) {
    if (P->exec && P->exec_csr == A && P->exec->order_knob == ctx->order &&
        P->exec->group == (ctx->group == 8 ? 8 : 16) && P->exec->stage_knob == ctx->stages &&
        P->exec->tile_knob == ctx->tile_rows && P->exec->thread_knob == ctx->threads &&
        P->exec->kernel_knob == ctx->kernel &&
        P->exec->prod_knob == ctx->producers &&
        P->exec->cg_knob == ctx->cgroups && P->exec->sched_knob == ctx->schedule) {
        Executor& E = *P->exec;
        const std::array<int64_t, 4> k = {ctx->slack, ctx->pass_powers, ctx->l2_budget, ctx->ctas_per_sm};
        if (E.knobs != k && E.fused_ready) {
            E.tickets.clear();  // schedule knobs changed: re-plan the ticket order
            E.pass_len.clear();
            E.wave.clear();
            const int occ = ctx->ctas_per_sm > 0 ? std::min<int>(E.occ_max, (int)ctx->ctas_per_sm) : E.occ_max;
            E.grid = occ * ctx->sm_count;
            E.slack = ctx->slack >= 0 ? ctx->slack : (int64_t)E.grid * E.stages;
            E.knobs = k;
        }
        return E;
    }
    auto E = std::make_shared<Executor>();
    E->knobs = {ctx->slack, ctx->pass_powers, ctx->l2_budget, ctx->ctas_per_sm};
    E->order_knob = ctx->order;
    E->kernel_knob = ctx->kernel;
    E->sched_knob = ctx->schedule;
    cudaStream_t st = ctx->stream;
    E->n_rows = A->n_rows;
    E->n_slots = (A->n_rows + 31u) & ~31u;
    // Row order: explicit, or auto: longest-rows-first (SELL-C-sigma) for power-law row lengths,
    // Cuthill-McKee inside levels otherwise.
    // Auto schedule: the wave (cross-power L2 reuse) for short-row matrices larger than the L2 --
    // every row a single 8-entry group (7-point Laplacians, p = 8, tools/wave_threshold.py: 128^3 /
    // 175 MB 146 vs 288 us for the sweeps, 256^3 0.77 vs 2.58 ms, C5 5.4 vs 20.2 ms; 64^3, which
    // sits in L2, 69 vs 46 us); one launch per power otherwise.
    const uint32_t mx_len = gpu_max_row_len(ctx, A);
    E->wave_auto = ctx->schedule == 0 && mx_len <= 8 && 12ull * A->nnz > 1ull * ctx->l2_bytes;
    if (ctx->order >= 0 && ctx->order <= 2) {
        E->order = (int)ctx->order;
    } else {
        const uint32_t mx = mx_len;
        const double avg = A->n_rows ? (double)A->nnz / A->n_rows : 0.0;
        if (mx > 64 && mx > 16.0 * avg)
            E->order = 2;
        else  // A_perm order already local (e.g. lexicographic grids): keep it, no private copies
            E->order = gpu_mean_first_col_jump(ctx, A) > 256.0 ? 1 : 0;
    }
    E->prod_knob = ctx->producers;
    E->cg_knob = ctx->cgroups;
    // every knob the cache check in this function compares (build_fused reads them later)
    E->group = ctx->group == 8 ? 8 : 16;
    E->stage_knob = ctx->stages;
    E->tile_knob = ctx->tile_rows;
    E->thread_knob = ctx->threads;
    E->tile_rows = ctx->tile_rows == 32 ? 32u : ctx->tile_rows == 64 ? 64u : (ctx->tile_rows == 256 ? 256u : 128u);
    if (E->tile_rows == 32 && ctx->kernel != 4) E->tile_rows = 64;  // 32-row tiles: async kernel only
    if (ctx->kernel == 2) E->tile_rows = 128;  // warp-tile: 4 warps x 32-row chunks
    if (ctx->schedule == 3 || E->wave_auto) E->tile_rows = kWaveRows;  // wave: one SELL chunk per ticket
    // consumer threads: one per tile row unless forced
    E->threads = ctx->threads == 256 || ctx->threads == 512 ? (uint32_t)ctx->threads : E->tile_rows;
    if (E->threads < E->tile_rows) E->threads = E->tile_rows;
    if (E->order >= 1) {
        gpu_level_cm_order(ctx, A, P->level_ptr, E->n_slots, E->slot_row, E->pos, E->order);
        build_sell(ctx, A, E->slot_row.p, E->pos.p, E->own, kLongCap);
        E->S = &E->own;
    } else {
        E->S = &csr_sell(A);
    }
    E->long_cap = E->S->long_cap;
    {  // tiles: fixed tile_rows slots, except that a 32-row chunk holding a long row is split
       // into single-row tiles (each long row gets its own ticket and the whole CTA).
        std::vector<uint32_t> rl(E->S->n_slots);
        bool has_long = false;
        if (E->long_cap != 0xffffffffu && E->S->n_slots) {
            MPKG_CUDA(cudaMemcpyAsync(rl.data(), E->S->row_len.p, 4ull * rl.size(), cudaMemcpyDeviceToHost, st));
            MPKG_CUDA(cudaStreamSynchronize(st));
            for (uint32_t v : rl)
                if (v > E->long_cap) {
                    has_long = true;
                    break;
                }
        }
        E->h_tile_start.clear();
        if (has_long) {
            const uint32_t per = E->tile_rows / 32;
            uint32_t c = 0, nch = E->S->n_chunks;
            while (c < nch) {
                bool lg = false;
                for (uint32_t i = 0; i < 32; ++i) lg |= rl[c * 32 + i] > E->long_cap;
                if (lg) {
                    for (uint32_t i = 0; i < 32; ++i) E->h_tile_start.push_back(c * 32 + i);
                    ++c;
                    continue;
                }
                E->h_tile_start.push_back(c * 32);
                uint32_t k = 1;
                ++c;
                while (k < per && c < nch) {
                    bool lg2 = false;
                    for (uint32_t i = 0; i < 32; ++i) lg2 |= rl[c * 32 + i] > E->long_cap;
                    if (lg2) break;
                    ++k;
                    ++c;
                }
            }
            E->h_tile_start.push_back(E->S->n_slots);
            E->n_tiles = (uint32_t)E->h_tile_start.size() - 1;
            E->tile_start.alloc(E->h_tile_start.size());
            MPKG_CUDA(cudaMemcpyAsync(E->tile_start.p, E->h_tile_start.data(), 4ull * E->h_tile_start.size(),
                                      cudaMemcpyHostToDevice, st));
            E->long_rows = 0;
            std::vector<uint32_t> ls;
            for (uint32_t i = 0; i < (uint32_t)rl.size(); ++i)
                if (rl[i] > E->long_cap) ls.push_back(i);
            E->long_rows = ls.size();
            E->long_slots.alloc(std::max<size_t>(ls.size(), 1));
            if (!ls.empty())
                MPKG_CUDA(cudaMemcpyAsync(E->long_slots.p, ls.data(), 4ull * ls.size(), cudaMemcpyHostToDevice, st));
            std::stable_sort(ls.begin(), ls.end(), [&](uint32_t x, uint32_t y) { return rl[x] > rl[y]; });
            E->long_sorted.alloc(std::max<size_t>(ls.size(), 1));
            if (!ls.empty())
                MPKG_CUDA(cudaMemcpyAsync(E->long_sorted.p, ls.data(), 4ull * ls.size(), cudaMemcpyHostToDevice, st));
        } else {
            E->n_tiles = (A->n_rows + E->tile_rows - 1) / E->tile_rows;
        }
    }
    if (E->n_tiles >= (1u << 24)) fail(MPKG_EINVAL, "mpk: more than 2^24 tiles");
    if (!E->h_tile_start.empty()) E->kernel_forced_lean = true;
    MPKG_CUDA(cudaStreamSynchronize(st));
    P->exec = E;
    P->exec_csr = A;
    return *E;
}

// Fused-kernel state (first fused run only: the sweep schedule never needs it): tile extents in
// the SELL arrays, tile dependency runs, kernel variant, occupancy, grid.
void build_fused(mpkg_ctx_s* ctx, mpkg_plan_s* P, mpkg_csr_s* A, Executor* E) {
    cudaStream_t st = ctx->stream;
    const uint32_t nt = E->n_tiles;
    auto tile_first = [&](uint32_t T) -> uint32_t {
        return E->h_tile_start.empty() ? std::min<uint64_t>((uint64_t)T * E->tile_rows, E->n_slots)
                                       : E->h_tile_start[T];
    };
    {  // tile extents in the SELL arrays; staging buffer size; oversized tiles
        std::vector<uint64_t> off(E->S->n_chunks + 1);
        MPKG_CUDA(cudaMemcpyAsync(off.data(), E->S->chunk_off.p, 8 * off.size(), cudaMemcpyDeviceToHost, st));
        MPKG_CUDA(cudaStreamSynchronize(st));
        std::vector<uint64_t> toff(nt + 1);
        E->tile_bytes.assign(nt, 0);
        E->big.assign(nt, 0);
        uint64_t max_buf = 256;
        for (uint32_t T = 0; T <= nt; ++T) toff[T] = off[std::min<uint64_t>((tile_first(T) + 31) / 32, E->S->n_chunks)];
        for (uint32_t T = 0; T < nt; ++T) {
            const uint64_t ne = toff[T + 1] >= toff[T] ? toff[T + 1] - toff[T] : 0;
            E->ne_max = std::max(E->ne_max, ne);
            const uint64_t bytes = (4 * ne + 127) & ~127ull;  // staged: column indices
            E->tile_bytes[T] = 12 * ne + (uint64_t)(tile_first(T + 1) - tile_first(T)) * 8 * 3;
            if (bytes > kMaxBufBytes)
                E->big[T] = 1;
            else
                max_buf = std::max(max_buf, bytes);
        }
        E->buf_bytes = (uint32_t)((max_buf + 127) & ~127ull);
        uint64_t lmax = 1;  // widest chunk (entries per lane), capped for the warp-tile slice
        for (uint32_t c = 0; c < E->S->n_chunks; ++c)
            lmax = std::max<uint64_t>(lmax, std::min<uint64_t>((off[c + 1] - off[c]) / 32, 64));
        E->wt_lmax = (uint32_t)lmax;
        E->tile_off.alloc(nt + 1);
        MPKG_CUDA(cudaMemcpyAsync(E->tile_off.p, toff.data(), 8ull * (nt + 1), cudaMemcpyHostToDevice, st));
    }
    // dependency runs
    std::vector<uint32_t> lp = P->level_ptr;
    if (lp.empty() || lp.back() != A->n_rows) lp = {0, A->n_rows};  // no level info: one level
    const uint32_t nl = (uint32_t)lp.size() - 1;
    DevBuf<uint32_t> d_lp(lp.size()), bmin((uint64_t)nt * kBuckets), bmax((uint64_t)nt * kBuckets);
    MPKG_CUDA(cudaMemcpyAsync(d_lp.p, lp.data(), 4 * lp.size(), cudaMemcpyHostToDevice, st));
    MPKG_CUDA(cudaMemsetAsync(bmin.p, 0xff, bmin.bytes(), st));
    MPKG_CUDA(cudaMemsetAsync(bmax.p, 0, bmax.bytes(), st));
    if (nt) {
        k_dep_buckets<<<grid_for(A->n_rows, 256), 256, 0, st>>>(
            A->row_ptr.p, A->col_idx.p, A->n_rows, E->order ? E->slot_row.p : nullptr,
            E->order ? E->pos.p : nullptr, d_lp.p, nl, E->tile_rows,
            E->h_tile_start.empty() ? nullptr : E->tile_start.p, nt, bmin.p, bmax.p);
        MPKG_LAUNCH_CHECK();
        ctx->launches += 1;
    }
    std::vector<uint32_t> hmin((uint64_t)nt * kBuckets), hmax((uint64_t)nt * kBuckets);
    MPKG_CUDA(cudaMemcpyAsync(hmin.data(), bmin.p, bmin.bytes(), cudaMemcpyDeviceToHost, st));
    MPKG_CUDA(cudaMemcpyAsync(hmax.data(), bmax.p, bmax.bytes(), cudaMemcpyDeviceToHost, st));
    MPKG_CUDA(cudaStreamSynchronize(st));
    E->h_ptr.assign(nt + 1, 0);
    E->h_lo.clear();
    E->h_hi.clear();
    auto slot_tile = [&](uint32_t sl) -> uint32_t {
        if (E->h_tile_start.empty()) return sl / E->tile_rows;
        return (uint32_t)(std::upper_bound(E->h_tile_start.begin(), E->h_tile_start.end(), sl) -
                          E->h_tile_start.begin()) - 1;
    };
    std::vector<std::pair<uint32_t, uint32_t>> runs;
    for (uint32_t T = 0; T < nt; ++T) {
        runs.clear();
        runs.push_back({T, T});
        for (int b = 0; b < kBuckets; ++b) {
            const uint64_t i = (uint64_t)T * kBuckets + b;
            if (hmin[i] <= hmax[i]) runs.push_back({slot_tile(hmin[i]), slot_tile(hmax[i])});
        }
        std::sort(runs.begin(), runs.end());
        uint32_t lo = runs[0].first, hi = runs[0].second;
        for (size_t k = 1; k < runs.size(); ++k) {
            if (runs[k].first <= hi + 1) {
                hi = std::max(hi, runs[k].second);
            } else {
                E->h_lo.push_back(lo);
                E->h_hi.push_back(hi);
                lo = runs[k].first;
                hi = runs[k].second;
            }
        }
        E->h_lo.push_back(lo);
        E->h_hi.push_back(hi);
        E->h_ptr[T + 1] = (uint32_t)E->h_lo.size();
    }
    {  // superblock polling pays when tiles wait on many tiles on average (R-MAT hubs: ~10^4);
       // a 3D stencil has ~30 and a few wide runs, which the tile-flag loop handles fine
        uint64_t dep_tiles = 0;
        for (size_t k = 0; k < E->h_lo.size(); ++k) dep_tiles += E->h_hi[k] - E->h_lo[k] + 1;
        E->sb = nt && dep_tiles > (uint64_t)nt * 4 * kSB;
    }
    // Stages: enough staged bytes per SM to cover DRAM latency (~200 KB of the 228 KB), at
    // least 2 (prefetch), at most kMaxStages; "stages" knob overrides.
    if (ctx->stages > 0)
        E->stages = (uint32_t)std::min<int64_t>(ctx->stages, kMaxStages);
    else
        E->stages = std::max<uint32_t>(2, std::min<uint32_t>(kMaxStages, (200u << 10) / E->buf_bytes));
    while (E->stages > 1 && E->stages * E->buf_bytes > (220u << 10)) --E->stages;
    const uint32_t smem = E->stages * E->buf_bytes;
    int occ = 0;
    // variable tiles (long rows): the lean kernel
    E->kernel = E->kernel_forced_lean ? 0 : (int)ctx->kernel;
    const uint64_t async_stage = ((E->ne_max + 31) & ~31ull) * 20;  // cols + vals + gathered x
    if (E->kernel == 4 && (async_stage > (110u << 10) || E->tile_rows > 256)) E->kernel = 0;
    if (E->kernel == 4) {
        E->buf_bytes = (uint32_t)std::max<uint64_t>(async_stage, 640);
        E->n_prod = ctx->producers > 0 ? (uint32_t)ctx->producers : 4u;
        E->n_cgroups = ctx->cgroups > 0 ? (uint32_t)ctx->cgroups : std::max<uint32_t>(1u, 128u / E->tile_rows);
        while (E->n_cgroups * E->tile_rows + 32 * E->n_prod > 512) E->n_cgroups > 1 ? --E->n_cgroups : --E->n_prod;
        const uint32_t fit = std::max<uint32_t>(1u, (225u << 10) / E->buf_bytes);  // slots that fit
        E->n_prod = std::min(E->n_prod, fit);
        E->n_cgroups = std::min(E->n_cgroups, fit);
        const uint32_t unit = std::max(E->n_prod, E->n_cgroups);
        uint32_t S = ctx->stages > 0 ? (uint32_t)ctx->stages : (210u << 10) / E->buf_bytes;
        S = std::min<uint32_t>(S, kMaxSlots) / unit * unit;
        while (S > unit && S * E->buf_bytes > (225u << 10)) S -= unit;
        E->stages = std::max(S, unit);
        E->threads = E->n_cgroups * E->tile_rows + 32 * E->n_prod;
        const int sm = (int)(E->stages * E->buf_bytes);
        if (sm > (225 << 10)) fail(MPKG_EINVAL, "mpk: async kernel stages do not fit shared memory");
        const void* ks[] = {(const void*)k_mpk_async<0, false>, (const void*)k_mpk_async<0, true>,
                            (const void*)k_mpk_async<1, false>, (const void*)k_mpk_async<1, true>,
                            (const void*)k_mpk_async<2, false>, (const void*)k_mpk_async<2, true>};
        for (const void* k : ks)
            MPKG_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
        MPKG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_mpk_async<0, true>, (int)E->threads, sm));
    } else if (E->kernel == 2) {
        E->threads = 128;
        E->stages = 1;
        configure_warptile(E->wt_lmax);
        if (E->group == 16)
            MPKG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_mpk_warptile<0, true, 8>, 128, 128 * E->wt_lmax * 8));
        else
            MPKG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_mpk_warptile<0, true, 4>, 128, 128 * E->wt_lmax * 8));
    } else if (E->kernel == 0) {
        E->threads = E->tile_rows;
        E->stages = 1;
        // resident CTAs of the variant this executor launches (all three kinds)
        const int nt = (int)std::min<uint32_t>(E->tile_rows, 128u);
        const bool vt = !E->h_tile_start.empty();
        occ = 1 << 30;
        for (const void* k : lean_variants(E->order >= 1, vt, vt || E->sb)) {
            int o = 0;
            MPKG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, k, nt, vt ? kLeanRingBytes : 0));
            occ = std::min(occ, o);
        }
    } else if (E->group == 8) {
        configure_kernels<8>(smem);
        MPKG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_mpk_fused<0, true, 8>, (int)E->threads + 32, smem));
    } else {
        configure_kernels<16>(smem);
        MPKG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_mpk_fused<0, true, 16>, (int)E->threads + 32, smem));
    }
    occ = std::max(1, occ);
    E->occ_max = occ;
    if (ctx->ctas_per_sm > 0) occ = std::min<int>(occ, (int)ctx->ctas_per_sm);
    E->grid = occ * ctx->sm_count;
    E->slack = ctx->slack >= 0 ? ctx->slack : (int64_t)E->grid * E->stages;
    E->dep_ptr.alloc(nt + 1);
    E->dep_lo.alloc(std::max<size_t>(E->h_lo.size(), 1));
    E->dep_hi.alloc(std::max<size_t>(E->h_hi.size(), 1));
    MPKG_CUDA(cudaMemcpyAsync(E->dep_ptr.p, E->h_ptr.data(), 4ull * (nt + 1), cudaMemcpyHostToDevice, st));
    if (!E->h_lo.empty()) {
        MPKG_CUDA(cudaMemcpyAsync(E->dep_lo.p, E->h_lo.data(), 4 * E->h_lo.size(), cudaMemcpyHostToDevice, st));
        MPKG_CUDA(cudaMemcpyAsync(E->dep_hi.p, E->h_hi.data(), 4 * E->h_hi.size(), cudaMemcpyHostToDevice, st));
    }
    E->done.alloc(std::max<uint32_t>(nt, 1));
    E->counter.alloc(1);
    MPKG_CUDA(cudaStreamSynchronize(st));
    E->knobs = {ctx->slack, ctx->pass_powers, ctx->l2_budget, ctx->ctas_per_sm};
    E->fused_ready = true;
}

// One pass of the list schedule over powers q0..q1: keys (pass, ready time, q, tile), unsorted.
void pass_keys(const Executor& E, uint32_t pass, int q0, int q1, std::vector<uint64_t>& keys) {
    const uint32_t nt = E.n_tiles;
    std::vector<int64_t> r(nt), rn(nt);
    for (uint32_t T = 0; T < nt; ++T) r[T] = T;
    for (int q = q0; q <= q1; ++q) {
        if (q > q0) {
            RangeMax rm(r);
            for (uint32_t T = 0; T < nt; ++T) {
                int64_t m = r[T] + 1;
                for (uint32_t k = E.h_ptr[T]; k < E.h_ptr[T + 1]; ++k)
                    // strictly later than every dependency: keeps the order topological
                    m = std::max(m, rm.query(E.h_lo[k], E.h_hi[k]) + std::max<int64_t>(E.slack, 1));
                rn[T] = m;
            }
            r.swap(rn);
        }
        const uint64_t last = q == q1 ? kLastUse : 0;
        for (uint32_t T = 0; T < nt; ++T)
            keys.push_back(((uint64_t)pass << 59) | ((uint64_t)r[T] << 32) |
                           (last | (E.big[T] ? kBig : 0) | ((uint64_t)q << 24) | T));
    }
}

// Peak bytes of matrix + working vectors that one pass of P powers keeps live, measured on the
// ticket order: tile T is live from its first to its last ticket of the pass.
uint64_t pass_window_bytes(const Executor& E, int P) {
    std::vector<uint64_t> keys;
    keys.reserve((uint64_t)E.n_tiles * P);
    pass_keys(E, 0, 1, P, keys);
    __gnu_parallel::sort(keys.begin(), keys.end());
    const uint32_t nt = E.n_tiles;
    std::vector<int64_t> first(nt, -1), last(nt, -1);
    for (size_t i = 0; i < keys.size(); ++i) {
        const uint32_t T = (uint32_t)(keys[i] & 0xffffffu);
        if (first[T] < 0) first[T] = (int64_t)i;
        last[T] = (int64_t)i;
    }
    std::vector<int64_t> diff(keys.size() + 1, 0);
    for (uint32_t T = 0; T < nt; ++T) {
        const int64_t b = (int64_t)E.tile_bytes[T];
        diff[first[T]] += b;
        diff[last[T] + 1] -= b;
    }
    int64_t cur = 0, peak = 0;
    for (size_t i = 0; i < keys.size(); ++i) peak = std::max(peak, cur += diff[i]);
    return (uint64_t)peak;
}

const DevBuf<uint32_t>& get_tickets(mpkg_ctx_s* ctx, Executor& E, int p) {
    auto it = E.tickets.find(p);
    if (it != E.tickets.end()) return it->second;
    const uint32_t nt = E.n_tiles;
    // Pass length: the largest P whose live window fits the L2 budget (the paper's p_opt
    // slicing into ceil(p/P) consecutive MPKs, chosen here by simulating the
    // schedule instead of by timing), unless forced with the "pass" knob.
    int P = p;
    if (ctx->pass_powers > 0) {
        P = std::min<int>({p, (int)ctx->pass_powers, kWaveMaxPass});
    } else {
        const uint64_t budget =
            ctx->l2_budget > 0 ? (uint64_t)ctx->l2_budget : ctx->l2_bytes * 6 / 10;
        while (P > 1 && pass_window_bytes(E, P) > budget) --P;
    }
    const int n_pass = (p + P - 1) / P;
    std::vector<uint64_t> keys;
    keys.reserve((uint64_t)nt * p);
    int q0 = 1;
    for (int j = 0; j < n_pass; ++j) {
        const int len = p / n_pass + (j < p % n_pass ? 1 : 0);  // balanced passes
        pass_keys(E, (uint32_t)j, q0, q0 + len - 1, keys);
        q0 += len;
    }
    E.pass_len[p] = (p + n_pass - 1) / n_pass;
    __gnu_parallel::sort(keys.begin(), keys.end());
    std::vector<uint32_t> codes(keys.size());
    for (size_t i = 0; i < keys.size(); ++i) codes[i] = (uint32_t)(keys[i] & 0xffffffffu);
    DevBuf<uint32_t> d(codes.size());
    MPKG_CUDA(cudaMemcpyAsync(d.p, codes.data(), sizeof(uint32_t) * codes.size(),
                              cudaMemcpyHostToDevice, ctx->stream));
    MPKG_CUDA(cudaStreamSynchronize(ctx->stream));
    return E.tickets.emplace(p, std::move(d)).first->second;
}

// Wave schedule, host side.  reach(T) = the furthest tile read by the rows of tiles <= T (a prefix
// maximum, so ready times stay monotone in T), from six buckets per tile: (row level - tile's first
// level in {0, >=1}) x (column level - row level in {-1, 0, +1}), each the min / max tile its
// columns fall in (wave_dep_tiles, the bucket spans, is reported by mpkg_plan_exec_info).
constexpr int kWaveBuckets = 6;
#ifndef MPKG_WAVE_SLACK_NUM
#define MPKG_WAVE_SLACK_NUM 5
#endif
constexpr int64_t kWaveSlackNum = MPKG_WAVE_SLACK_NUM, kWaveSlackDen = 1;

__global__ void k_wave_buckets(const uint32_t* __restrict__ rp, const uint32_t* __restrict__ ci, uint32_t n,
                               const uint32_t* __restrict__ slot_row, const uint32_t* __restrict__ pos,
                               const uint32_t* __restrict__ lp, uint32_t nl, uint32_t n_slots,
                               uint32_t* __restrict__ bmin, uint32_t* __restrict__ bmax) {
    for (uint64_t s = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; s < n_slots;
         s += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t r = slot_row ? slot_row[s] : (uint32_t)s;
        if (r >= n) continue;
        const uint32_t T = (uint32_t)(s / kWaveRows);
        const uint32_t lt = level_of(lp, nl, T * kWaveRows);
        const uint32_t L = level_of(lp, nl, (uint32_t)s);
        const uint32_t rb = L > lt ? 1u : 0u;
        const uint32_t lb = lp[L], le = lp[L + 1];
        for (uint32_t k = rp[r]; k < rp[r + 1]; ++k) {
            const uint32_t c = ci[k];
            const uint32_t d = c < lb ? 0u : (c >= le ? 2u : 1u);
            const uint32_t tc = (pos ? pos[c] : c) / kWaveRows;
            atomicMin(bmin + (uint64_t)T * kWaveBuckets + rb * 3 + d, tc);
            atomicMax(bmax + (uint64_t)T * kWaveBuckets + rb * 3 + d, tc);
        }
    }
}

uint32_t wave_stage_for(int fmt, bool sigma);

void build_wave(mpkg_ctx_s* ctx, mpkg_plan_s* Pl, mpkg_csr_s* A, Executor& E) {
    cudaStream_t st = ctx->stream;
    const uint32_t nt = E.n_tiles;
    {  // the chunk records (one per tile) and the bytes one tile-power touches (record + x read + y
       // written: the live-window model of wave_order)
        const uint32_t nc = E.S->n_chunks;
        const uint64_t nrec = (uint64_t)nt * kWaveChunks;  // the last tile padded with empty records
        if (nrec < nc) fail(MPKG_EINTERNAL, "wave: tiles do not cover the SELL chunks");
        std::vector<uint64_t> off((uint64_t)nc + 1);
        MPKG_CUDA(cudaMemcpyAsync(off.data(), E.S->chunk_off.p, 8 * off.size(), cudaMemcpyDeviceToHost, st));
        MPKG_CUDA(cudaStreamSynchronize(st));
        uint64_t max_l = 0;
        for (uint32_t c = 0; c < nc; ++c) max_l = std::max<uint64_t>(max_l, (off[c + 1] - off[c]) >> 5);
        // value dictionary: at most kWaveDictMax distinct values and rows of at most 255 entries
        DevBuf<unsigned long long> table(kDictSlots);
        DevBuf<uint16_t> slot_ix(kDictSlots);
        std::vector<double> dict;
        E.wave_fmt = 0;
        if (ctx->wave_dict && max_l <= 255 && E.S->n_entries) {
            DevBuf<uint32_t> count(1);
            std::vector<unsigned long long> empty(kDictSlots, kDictEmpty);
            MPKG_CUDA(cudaMemcpyAsync(table.p, empty.data(), 8 * kDictSlots, cudaMemcpyHostToDevice, st));
            MPKG_CUDA(cudaMemsetAsync(count.p, 0, 4, st));
            k_dict_insert<<<grid_for(E.S->n_entries, 256, (unsigned)ctx->sm_count * 8u), 256, 0, st>>>(
                E.S->vals.p, E.S->n_entries, table.p, count.p);
            MPKG_LAUNCH_CHECK();
            ctx->launches += 1;
            uint32_t cnt = 0;
            std::vector<unsigned long long> h(kDictSlots);
            MPKG_CUDA(cudaMemcpyAsync(&cnt, count.p, 4, cudaMemcpyDeviceToHost, st));
            MPKG_CUDA(cudaMemcpyAsync(h.data(), table.p, 8 * kDictSlots, cudaMemcpyDeviceToHost, st));
            MPKG_CUDA(cudaStreamSynchronize(st));
            if (cnt <= kWaveDictMax) {
                std::vector<uint16_t> ix(kDictSlots, 0);
                for (uint32_t i = 0; i < kDictSlots; ++i)
                    if (h[i] != kDictEmpty) {
                        ix[i] = (uint16_t)dict.size();
                        double v;
                        std::memcpy(&v, &h[i], 8);
                        dict.push_back(v);
                    }
                MPKG_CUDA(cudaMemcpyAsync(slot_ix.p, ix.data(), 2 * kDictSlots, cudaMemcpyHostToDevice, st));
                E.wave_dict.alloc(std::max<size_t>(dict.size(), 1));
                if (!dict.empty())
                    MPKG_CUDA(cudaMemcpyAsync(E.wave_dict.p, dict.data(), 8 * dict.size(), cudaMemcpyHostToDevice, st));
                E.n_dict = (uint32_t)dict.size();
                E.wave_fmt = 1;
            }
        }
        const bool sigma = E.order >= 1;
        // affine chunks (dict format only)
        std::vector<uint8_t> aff;
        DevBuf<uint8_t> d_aff(std::max<uint32_t>(nc, 1));
        E.wave_affine_chunks = 0;
        E.wave_banded_chunks = 0;
        if (E.wave_fmt == 1 && ctx->wave_affine && nc) {
            k_wave_affine<<<grid_for((uint64_t)nc * 32, 256, (unsigned)ctx->sm_count * 8u), 256, 0, st>>>(
                E.S->cols.p, E.S->vals.p, E.S->row_len.p, sigma ? E.slot_row.p : nullptr, E.S->chunk_off.p, nc,
                A->n_rows, ctx->wave_affine >= 2 ? 1 : 0, d_aff.p);
            MPKG_LAUNCH_CHECK();
            ctx->launches += 1;
            aff.resize(nc);
            MPKG_CUDA(cudaMemcpyAsync(aff.data(), d_aff.p, nc, cudaMemcpyDeviceToHost, st));
            MPKG_CUDA(cudaStreamSynchronize(st));
        }
        E.tile_bytes.assign(nt, 0);
        const uint32_t stage_cap = wave_stage_for(E.wave_fmt, sigma);
        std::vector<uint32_t> ro(nrec + 1);
        std::vector<uint8_t> narrow(nt, 1);
        std::vector<uint32_t> trec(nt, 0);
        uint64_t acc = 0;
        for (uint64_t c = 0; c < nrec; ++c) {
            ro[c] = (uint32_t)acc;
            const uint32_t L = c < nc ? (uint32_t)((off[c + 1] - off[c]) >> 5) : 0u;
            const bool is_aff = c < aff.size() && aff[c] == 1;
            const bool is_band = c < aff.size() && aff[c] == 2;
            const uint32_t rb = is_aff ? wave_affine_bytes(sigma)
                                : is_band ? wave_banded_bytes(sigma) : wave_rec_bytes(E.wave_fmt, sigma, L);
            E.wave_affine_chunks += is_aff;
            E.wave_banded_chunks += is_band;
            acc += rb / 16;
            if (acc > 0xffffffffull) fail(MPKG_EINVAL, "mpk: matrix too large for the wave schedule's records");
            E.tile_bytes[c / kWaveChunks] += rb + 16ull * 32;
            if (L > 8) narrow[c / kWaveChunks] &= ~1u;
            // fast tile: all chunks affine with one width (bits 4-7; 0 = not fast)
            uint8_t& code = narrow[c / kWaveChunks];
            if (c % kWaveChunks == 0) code = (uint8_t)((code & 1u) | (is_aff ? L << 4 : 0u));
            else if (!is_aff || (code >> 4) != L) code &= 1u;
            trec[c / kWaveChunks] += rb;
        }
        for (uint32_t T = 0; T < nt; ++T)  // records larger than a stage: not staged (nor fast)
            if (trec[T] > stage_cap) narrow[T] = 0;
        ro[nrec] = (uint32_t)acc;
        E.wave_rec_total = acc * 16;
        E.wrec_off.alloc(nrec + 1);
        E.wrec.alloc(std::max<uint64_t>(acc * 16, 16));
        E.wave_narrow.alloc(std::max<uint64_t>(nt, 1));
        MPKG_CUDA(cudaMemcpyAsync(E.wrec_off.p, ro.data(), 4 * ro.size(), cudaMemcpyHostToDevice, st));
        if (nt) MPKG_CUDA(cudaMemcpyAsync(E.wave_narrow.p, narrow.data(), nt, cudaMemcpyHostToDevice, st));
        if (nrec) {
            const unsigned g = grid_for(nrec * 32, 256, (unsigned)ctx->sm_count * 8u);
            if (E.wave_fmt == 1)
                k_wave_pack<1><<<g, 256, 0, st>>>(E.S->cols.p, E.S->vals.p, E.S->row_len.p,
                                                  sigma ? E.slot_row.p : nullptr, E.S->chunk_off.p, nc,
                                                  (uint32_t)nrec, E.wrec_off.p, E.wrec.p, table.p, slot_ix.p,
                                                  aff.empty() ? nullptr : d_aff.p);
            else
                k_wave_pack<0><<<g, 256, 0, st>>>(E.S->cols.p, E.S->vals.p, E.S->row_len.p,
                                                  sigma ? E.slot_row.p : nullptr, E.S->chunk_off.p, nc,
                                                  (uint32_t)nrec, E.wrec_off.p, E.wrec.p, nullptr, nullptr, nullptr);
            MPKG_LAUNCH_CHECK();
            ctx->launches += 1;
        }
        if (nt && !aff.empty()) {
            k_wave_pairs<<<grid_for(nt, 256, (unsigned)ctx->sm_count * 8u), 256, 0, st>>>(
                E.wrec.p, E.wrec_off.p, nt, WaveRec<1, false>::len_bytes,
                sigma ? WaveRec<1, true>::hdr : WaveRec<1, false>::hdr, E.wave_narrow.p);
            MPKG_LAUNCH_CHECK();
            ctx->launches += 1;
        }
        DevBuf<uint64_t> pol(2);
        k_l2_policies<<<1, 1, 0, st>>>(pol.p);
        MPKG_LAUNCH_CHECK();
        MPKG_CUDA(cudaMemcpyAsync(E.wave_pol, pol.p, 16, cudaMemcpyDeviceToHost, st));
        MPKG_CUDA(cudaStreamSynchronize(st));
    }
    std::vector<uint32_t> lp = Pl->level_ptr;
    if (lp.empty() || lp.back() != A->n_rows) lp = {0, A->n_rows};  // no level info: one level
    const uint32_t nl = (uint32_t)lp.size() - 1;
    DevBuf<uint32_t> d_lp(lp.size()), bmin((uint64_t)nt * kWaveBuckets), bmax((uint64_t)nt * kWaveBuckets);
    MPKG_CUDA(cudaMemcpyAsync(d_lp.p, lp.data(), 4 * lp.size(), cudaMemcpyHostToDevice, st));
    MPKG_CUDA(cudaMemsetAsync(bmin.p, 0xff, bmin.bytes(), st));
    MPKG_CUDA(cudaMemsetAsync(bmax.p, 0, bmax.bytes(), st));
    if (nt) {
        k_wave_buckets<<<grid_for(E.n_slots, 256, (unsigned)ctx->sm_count * 8u), 256, 0, st>>>(
            A->row_ptr.p, A->col_idx.p, A->n_rows, E.order ? E.slot_row.p : nullptr,
            E.order ? E.pos.p : nullptr, d_lp.p, nl, E.n_slots, bmin.p, bmax.p);
        MPKG_LAUNCH_CHECK();
        ctx->launches += 1;
    }
    std::vector<uint32_t> hmin((uint64_t)nt * kWaveBuckets), hmax((uint64_t)nt * kWaveBuckets);
    MPKG_CUDA(cudaMemcpyAsync(hmin.data(), bmin.p, bmin.bytes(), cudaMemcpyDeviceToHost, st));
    MPKG_CUDA(cudaMemcpyAsync(hmax.data(), bmax.p, bmax.bytes(), cudaMemcpyDeviceToHost, st));
    MPKG_CUDA(cudaStreamSynchronize(st));
    E.wave_reach.assign(nt, 0);
    E.wave_dep_tiles = 0;
    uint32_t reach = 0;
    for (uint32_t T = 0; T < nt; ++T) {
        uint32_t hi = T;
        for (int b = 0; b < kWaveBuckets; ++b) {
            const uint64_t i = (uint64_t)T * kWaveBuckets + b;
            if (hmin[i] <= hmax[i]) {
                hi = std::max(hi, hmax[i]);
                E.wave_dep_tiles += hmax[i] - hmin[i] + 1;
            }
        }
        reach = std::max(reach, hi);
        E.wave_reach[T] = reach;
    }
}

// Ticket order of one pass over powers q0..q1: ready(T, q0) = T, ready(T, q) = ready(reach(T),
// q-1) + slack (monotone in T, so each power's list is sorted and the pass is their merge, ties
// broken by power then tile).  Returns the pass's live window: the most matrix + vector bytes of
// tiles between their first and last ticket, at any point of the order.
uint64_t wave_order(const Executor& E, int q0, int q1, int64_t slack, std::vector<uint32_t>* codes) {
    const uint32_t nt = E.n_tiles;
    const int np = q1 - q0 + 1;
    std::vector<std::vector<int64_t>> rdy(np, std::vector<int64_t>(nt));
    for (uint32_t T = 0; T < nt; ++T) rdy[0][T] = T;
    for (int j = 1; j < np; ++j)
        for (uint32_t T = 0; T < nt; ++T) rdy[j][T] = rdy[j - 1][E.wave_reach[T]] + slack;
    std::vector<uint32_t> pos(np, 0);
    std::vector<int64_t> diff;
    diff.reserve((uint64_t)nt * np + 1);
    int64_t cur = 0, peak = 0;
    // live bytes: tile T enters at its q0 ticket and leaves after its q1 ticket
    for (;;) {
        int best = -1;
        for (int j = np - 1; j >= 0; --j)  // ties: the higher power first (older front)
            if (pos[j] < nt && (best < 0 || rdy[j][pos[j]] < rdy[best][pos[best]])) best = j;
        if (best < 0) break;
        const uint32_t T = pos[best]++;
        const int q = q0 + best;
        if (best == 0) cur += (int64_t)E.tile_bytes[T];
        peak = std::max(peak, cur);
        if (best == np - 1) cur -= (int64_t)E.tile_bytes[T];
        if (codes) codes->push_back((q == q1 ? kLastUse : 0u) | ((uint32_t)q << 24) | T);
    }
    return (uint64_t)peak;
}

// Pass length p' = the longest pass whose live window fits the budget (0.6 x L2 unless the
// l2_budget knob says otherwise; the "pass" knob forces p'); slack (ready-time units, ~p'
// tickets each) = 5 x the warps / p': a ticket runs two claims after its warp took it and its
// producer needs a ticket's time to store, so producer and consumer sit ~5 x warps tickets apart
// in the order and a ticket's inputs are almost always stored when its warp reaches it (C5 p = 8:
// 2.2 x warps left 13% of the rows waiting on a producer, 9.0 ms; 5 x warps none, 6.8 ms).
// Passes are balanced (ceil(p / p') of them).
const Executor::Wave& get_wave(mpkg_ctx_s* ctx, Executor& E, int p) {
    auto it = E.wave.find(p);
    if (it != E.wave.end()) return it->second;
    Executor::Wave W;
    const uint64_t budget = ctx->l2_budget > 0 ? (uint64_t)ctx->l2_budget : ctx->l2_bytes * 6 / 10;
    const int64_t warps = (int64_t)E.wave_grid * kWaveWarps;
    auto slack_for = [&](int len) -> int64_t {
        if (ctx->slack >= 0) return std::max<int64_t>(ctx->slack, 1);
        return std::max<int64_t>(1, (warps * kWaveSlackNum / kWaveSlackDen + len - 1) / len);
    };
    // auto: at most kWaveAutoPass powers per pass (C5, chunk records in the dict format: p' = 2..4
    // within 4%, 8 is 15% slower: the fronts' lag grows with p')
    int P = std::min(p, kWaveAutoPass);
    if (ctx->pass_powers > 0) {
        P = std::min<int>({p, (int)ctx->pass_powers, kWaveMaxPass});
        W.window = wave_order(E, 1, P, slack_for(P), nullptr);
    } else {
        for (; P >= 1; --P) {
            W.window = wave_order(E, 1, P, slack_for(P), nullptr);
            if (P == 1 || W.window <= budget) break;
        }
    }
    const int n_pass = (p + P - 1) / P;
    std::vector<uint32_t> codes;
    codes.reserve((uint64_t)E.n_tiles * p);
    int q0 = 1;
    W.t_begin.push_back(0);
    for (int j = 0; j < n_pass; ++j) {
        // the shorter passes first: the first pass's in-pass slices are the ones k_wave_fill has to
        // empty (every later pass's are emptied by the pass before it)
        const int len = p / n_pass + (j >= n_pass - p % n_pass ? 1 : 0);
        W.slack = slack_for(len);
        wave_order(E, q0, q0 + len - 1, W.slack, &codes);
        W.q_begin.push_back(q0);
        q0 += len;
        W.t_begin.push_back((uint32_t)codes.size());
    }
    W.q_begin.push_back(q0);
    W.pass_len = (p + n_pass - 1) / n_pass;
    W.tickets.alloc(std::max<size_t>(codes.size(), 1));
    W.desc.alloc(std::max<size_t>(codes.size(), 1));
    if (!codes.empty())
        MPKG_CUDA(cudaMemcpyAsync(W.tickets.p, codes.data(), sizeof(uint32_t) * codes.size(),
                                  cudaMemcpyHostToDevice, ctx->stream));
    for (int j = 0; j < n_pass; ++j) {
        const uint64_t b = W.t_begin[j], e = W.t_begin[j + 1];
        if (e > b) {
            k_wave_desc<<<grid_for(e - b, 256, (unsigned)ctx->sm_count * 8u), 256, 0, ctx->stream>>>(
                W.tickets.p + b, e - b, E.wrec_off.p, E.wave_narrow.p, (uint32_t)W.q_begin[j],
                (uint32_t)W.q_begin[j + 1] - 1u, W.desc.p + b);
            MPKG_LAUNCH_CHECK();
            ctx->launches += 1;
        }
    }
    MPKG_CUDA(cudaStreamSynchronize(ctx->stream));
    E.pass_len[p] = W.pass_len;
    return E.wave.emplace(p, std::move(W)).first->second;
}

// The coefficient polynomial from finished slices (wave schedule): z = c_0 x + c_1 y_1, then
// z += c_q y_q for q = 2..p, the order and the separate multiply / add of row_epilogue<2> (and of
// the reference harness): bit-identical to the sweeps' running accumulator.
__global__ void k_poly_combine(const double* __restrict__ blk, uint64_t stride, uint32_t n, uint32_t p,
                               const double* __restrict__ coef, double* __restrict__ z) {
    for (uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r < n; r += (uint64_t)gridDim.x * blockDim.x) {
        double zr = __dadd_rn(__dmul_rn(coef[0], blk[r]), __dmul_rn(coef[1], blk[stride + r]));
        for (uint32_t q = 2; q <= p; ++q) zr = __dadd_rn(zr, __dmul_rn(coef[q], blk[(uint64_t)q * stride + r]));
        z[r] = zr;
    }
}

void* wave_fn(int kind, bool sigma, int fmt, bool trace) {
#define MPKG_WAVE_FNS(F, TR)                                                                         \
    {(void*)k_mpk_wave<0, false, F, TR>, (void*)k_mpk_wave<0, true, F, TR>, (void*)k_mpk_wave<1, false, F, TR>, \
     (void*)k_mpk_wave<1, true, F, TR>}
    static void* const fns[2][2][4] = {{MPKG_WAVE_FNS(0, false), MPKG_WAVE_FNS(0, true)},
                                       {MPKG_WAVE_FNS(1, false), MPKG_WAVE_FNS(1, true)}};
#undef MPKG_WAVE_FNS
    return fns[fmt][trace ? 1 : 0][kind * 2 + (sigma ? 1 : 0)];
}
uint32_t wave_stage_for(int fmt, bool sigma) {
    return fmt == 1 ? (sigma ? wave_stage_bytes<1, true>() : wave_stage_bytes<1, false>())
                    : (sigma ? wave_stage_bytes<0, true>() : wave_stage_bytes<0, false>());
}
uint32_t wave_smem_for(int fmt, bool sigma) {
    return fmt == 1 ? (sigma ? wave_smem<1, true>() : wave_smem<1, false>())
                    : (sigma ? wave_smem<0, true>() : wave_smem<0, false>());
}

template <int KIND, int G>
void launch_g(bool sigma, int grid, int threads, uint32_t smem, cudaStream_t st,
              const FusedParams& P) {
    if (sigma)
        k_mpk_fused<KIND, true, G><<<grid, threads, smem, st>>>(P);
    else
        k_mpk_fused<KIND, false, G><<<grid, threads, smem, st>>>(P);
}

template <int KIND>
void launch_kind(bool sigma, const Executor& E, uint32_t smem, cudaStream_t st,
                 const FusedParams& P) {
    if (E.group == 8)
        launch_g<KIND, 8>(sigma, E.grid, (int)E.threads + 32, smem, st, P);
    else
        launch_g<KIND, 16>(sigma, E.grid, (int)E.threads + 32, smem, st, P);
}

}  // namespace

// Schedule choice ("schedule" knob: 0 auto, 1 fused, 2 sweeps).  Measured on B200 (DESIGN.md
// §5): the fused tile-DAG kernel never reuses L2 across powers at C2..C5 sizes (the in-flight
// window needed to saturate HBM plus the level lag exceeds the 126 MB L2) and even at C1 its
// level-by-level critical path costs more than p launches, so auto runs one launch per power
// over the executor's SELL -- except for matrices with long rows, whose CTA-cooperative path
// exists only in the fused kernel.
// Fast mode: work items of k_coop_rows for every row longer than kMedCap (none for stencils), the
// longest first so the tail of the side-stream launch is short.
void build_coop(mpkg_ctx_s* ctx, Executor& E, mpkg_csr_s* A) {
    E.coop_ready = true;
    E.coop_min = ctx->coop_min > 0 ? (uint32_t)ctx->coop_min : kMedCap;
    const Sell& S = *E.S;
    cudaStream_t st = ctx->stream;
    const bool sigma = E.order >= 1;
    std::vector<uint32_t> rl(S.n_slots), sr, rp((uint64_t)A->n_rows + 1);
    if (S.n_slots) MPKG_CUDA(cudaMemcpyAsync(rl.data(), S.row_len.p, 4ull * rl.size(), cudaMemcpyDeviceToHost, st));
    if (sigma) {
        sr.resize(E.n_slots);
        MPKG_CUDA(cudaMemcpyAsync(sr.data(), E.slot_row.p, 4ull * sr.size(), cudaMemcpyDeviceToHost, st));
    }
    MPKG_CUDA(cudaMemcpyAsync(rp.data(), A->row_ptr.p, 4ull * rp.size(), cudaMemcpyDeviceToHost, st));
    MPKG_CUDA(cudaStreamSynchronize(st));
    std::vector<std::pair<uint32_t, uint32_t>> rows;  // (length, slot)
    for (uint32_t sl = 0; sl < (uint32_t)rl.size(); ++sl) {
        const uint32_t r = sigma ? sr[sl] : sl;
        if (r < A->n_rows && rl[sl] > E.coop_min) rows.emplace_back(rl[sl], sl);
    }
    std::stable_sort(rows.begin(), rows.end(), [](const auto& x, const auto& y) { return x.first > y.first; });
    std::vector<uint4> items, multi;
    uint32_t part = 0;
    for (const auto& [len, sl] : rows) {
        const uint32_t r = sigma ? sr[sl] : sl;
        const uint32_t b = rp[r], e = rp[r + 1];
        if (len <= kCoopSeg) {
            items.push_back(make_uint4(sl, b, e, 0xffffffffu));
        } else {
            const uint32_t cnt = (len + kCoopSeg - 1) / kCoopSeg;
            multi.push_back(make_uint4(sl, part, cnt, 0u));
            for (uint32_t i = 0; i < cnt; ++i)
                items.push_back(make_uint4(sl, b + i * kCoopSeg, std::min(e, b + (i + 1) * kCoopSeg), part++));
        }
    }
    E.n_coop = (uint32_t)items.size();
    E.n_multi = (uint32_t)multi.size();
    E.coop_items.alloc(std::max<size_t>(items.size(), 1));
    E.coop_multi.alloc(std::max<size_t>(multi.size(), 1));
    E.coop_part.alloc(std::max<uint32_t>(part, 1));
    if (!items.empty())
        MPKG_CUDA(cudaMemcpyAsync(E.coop_items.p, items.data(), sizeof(uint4) * items.size(), cudaMemcpyHostToDevice, st));
    if (!multi.empty())
        MPKG_CUDA(cudaMemcpyAsync(E.coop_multi.p, multi.data(), sizeof(uint4) * multi.size(), cudaMemcpyHostToDevice, st));
    MPKG_CUDA(cudaStreamSynchronize(st));
}

bool use_sweeps(const mpkg_ctx_s* ctx, const Executor& E, int p, int kind) {
    if (ctx->schedule == 1) return false;
    if ((ctx->schedule == 3 || (ctx->schedule == 0 && E.wave_auto && p >= 2)) && E.h_tile_start.empty() &&
        E.tile_rows == kWaveRows)
        return false;
    // Long rows live outside the SELL arrays.  Fast mode reduces them in k_coop_rows beside the
    // sweeps; bitwise mode adds them in stored order in k_long_rows_bitwise beside the sweeps
    // (R-MAT scale 21: 2.79 ms vs 2.93 ms for the fused kernel's CTA-cooperative path; both are
    // bounded by the hub row's chain of 102,493 dependent adds).
    return true;
}

void run_fused(mpkg_ctx_s* ctx, mpkg_plan_s* Pl, mpkg_csr_s* A, const FusedArgs& a) {
    if (a.p > kMaxFusedP) fail(MPKG_EINVAL, "mpk: at most 32 powers per fused launch");
    Executor& E = get_executor(ctx, Pl, A);
    if (E.n_tiles == 0) return;
    const bool sweep = use_sweeps(ctx, E, a.p, a.kind);
    const bool wave = !sweep && ctx->schedule != 1;
    if (!sweep && !wave && !E.fused_ready) build_fused(ctx, Pl, A, &E);
    if (wave && !E.wave_grid) {
        build_wave(ctx, Pl, A, E);  // picks the record format
        int occ = 1 << 30;
        for (int k = 0; k < 4; ++k) {
            int o = 0;
            void* fn = wave_fn(k / 2, k % 2, E.wave_fmt, false);
            const uint32_t sm = wave_smem_for(E.wave_fmt, k % 2 != 0);
            MPKG_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
            MPKG_CUDA(cudaFuncSetAttribute(wave_fn(k / 2, k % 2, E.wave_fmt, true),
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
            MPKG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, fn, kWaveThreads, sm));
            occ = std::min(occ, o);
        }
        if (ctx->ctas_per_sm > 0) occ = std::min<int>(occ, (int)ctx->ctas_per_sm);
        E.wave_grid = std::max(1, occ) * ctx->sm_count;
        E.wave.clear();  // the slack follows the warps in flight
        E.counter.alloc(kWaveStreams * 32 + 32);
    }
    static const DevBuf<uint32_t> no_tickets;
    const Executor::Wave* W = wave ? &get_wave(ctx, E, a.p) : nullptr;
    const DevBuf<uint32_t>& tk = sweep ? no_tickets : wave ? W->tickets : get_tickets(ctx, E, a.p);
    const Sell& S = *E.S;
    cudaStream_t st = ctx->stream;
    const bool sigma = E.order >= 1;  // any private order (CM or length-sorted)
    FusedParams P;
    std::memset(&P, 0, sizeof(P));  // padding too: the bytes key the CUDA-graph cache
    P.cols = S.cols.p;
    P.vals = S.vals.p;
    P.chunk_off = S.chunk_off.p;
    P.tile_off = E.tile_off.p;
    P.row_len = S.row_len.p;
    P.slot_row = sigma ? E.slot_row.p : nullptr;
    P.tickets = tk.p;
    P.wdesc = wave ? W->desc.p : nullptr;
    P.wrec = E.wrec.p;
    P.wrec_off = E.wrec_off.p;
    P.dict = E.wave_dict.p;
    P.n_dict = E.n_dict;
    P.pol_first = E.wave_pol[0];
    P.pol_last = E.wave_pol[1];
    P.dep_ptr = E.dep_ptr.p;
    P.dep_lo = E.dep_lo.p;
    P.dep_hi = E.dep_hi.p;
    P.done = E.done.p;
    P.counter = E.counter.p;
    P.n_tickets = (uint32_t)tk.n;
    P.n_rows = A->n_rows;
    P.n_slots = E.n_slots;
    P.p = (uint32_t)a.p;
    P.buf_bytes = E.buf_bytes;
    P.stages = E.stages;
    P.tile_rows = E.tile_rows;
    P.wt_lmax = E.wt_lmax;
    P.tile_start = E.h_tile_start.empty() ? nullptr : E.tile_start.p;
    P.long_cap = E.long_cap;
    P.csr_rp = A->row_ptr.p;
    P.csr_ci = A->col_idx.p;
    P.csr_v = A->values.p;
    P.n_tiles = E.n_tiles;
    P.long_slots = E.long_slots.p;
    if (ctx->trace && !sweep) {
        E.trace_n = 2ull * E.n_tiles * (a.p + 1);
        E.trace.ensure(E.trace_n);
        MPKG_CUDA(cudaMemsetAsync(E.trace.p, 0, 8 * E.trace_n, st));
        P.trace = E.trace.p;
    } else {
        E.trace_n = 0;
    }
    P.n_long = (uint32_t)E.long_rows;
    // fast-mode sweeps over a matrix with rows longer than kMedCap: those rows (long ones
    // included) run in k_coop_rows on a side stream, concurrently with each power's sweep
    if (sweep && ctx->mode == MPKG_MODE_FAST &&
        (!E.coop_ready || E.coop_min != (ctx->coop_min > 0 ? (uint32_t)ctx->coop_min : kMedCap)))
        build_coop(ctx, E, A);
    const bool coop = sweep && ctx->mode == MPKG_MODE_FAST && E.n_coop > 0;
    const bool bw_long = sweep && ctx->mode != MPKG_MODE_FAST && E.long_rows > 0;
    P.sweep_cap = coop ? E.coop_min : E.long_cap;
    // matrix + the p+1 working vectors within half the L2: one cooperative launch (k_mpk_resident)
    const uint64_t res_bytes = 12ull * A->nnz + 4ull * (A->n_rows + 1) + 8ull * E.n_slots * (a.p + 1);
    const bool resident = sweep && ctx->resident && !coop && !E.long_rows && a.host_block == nullptr &&
                          res_bytes <= ctx->l2_bytes / 2 && a.p >= 2;
    P.coop_items = coop ? E.coop_items.p : nullptr;
    P.coop_multi = coop ? E.coop_multi.p : nullptr;
    P.coop_part = coop ? E.coop_part.p : nullptr;
    P.n_coop = coop ? E.n_coop : 0;
    P.n_multi = coop ? E.n_multi : 0;
    P.n_prod = E.n_prod;
    P.n_cgroups = E.n_cgroups;
    P.n_sb = (E.n_tiles + kSB - 1) / kSB;
    if (!sweep && !wave) {
        E.sb_count.ensure((uint64_t)(kMaxFusedP + 1) * P.n_sb + 1);
        P.sb_count = E.sb_count.p;
        MPKG_CUDA(cudaMemsetAsync(E.sb_count.p, 0, 4ull * (a.p + 1) * P.n_sb, st));
    }
    P.rows = a.rows;
    P.out = a.block;
    P.z = a.z;
    // slice 0 = x (mpk.hpp:62).  On the graph-replayed sweep path the copy is a node of the graph
    // (one API call less per MPK on launch-bound matrices); otherwise it is issued up front.
    bool x_pending = a.x != nullptr && a.x != a.block;
    auto copy_x = [&]() {
        MPKG_CUDA(cudaMemcpyAsync(a.block, a.x, sizeof(double) * A->n_rows, cudaMemcpyDeviceToDevice, st));
        x_pending = false;
    };
    if (sigma && x_pending) copy_x();  // the sigma gather below reads slice 0
    if (sigma) {
        E.V.ensure((uint64_t)E.n_slots * (a.p + 1));
        P.V = E.V.p;
        P.vstride = E.n_slots;
        if (a.kind == 2) {
            E.zs.ensure(E.n_slots);
            P.zs = E.zs.p;
        }
        k_gather_x<<<grid_for(E.n_slots, 256), 256, 0, st>>>(a.block, E.slot_row.p, E.n_slots,
                                                             A->n_rows, E.V.p);
        MPKG_LAUNCH_CHECK();
        ctx->launches += 1;
    } else {
        P.V = a.block;
        P.vstride = a.rows;
        P.zs = a.z;
    }
    for (int i = 0; i < a.p; ++i) {
        P.shift_a[i] = a.shift_a ? a.shift_a[i] : 0.0;
        P.shift_b2[i] = a.shift_b2 ? a.shift_b2[i] : 0.0;
    }
    for (int i = 0; i <= a.p; ++i) P.coef[i] = a.coef ? a.coef[i] : 0.0;
    if (!sweep && !wave) {
        MPKG_CUDA(cudaMemsetAsync(E.done.p, 0, E.done.bytes(), st));
        MPKG_CUDA(cudaMemsetAsync(E.counter.p, 0, sizeof(uint32_t), st));
    }
    const uint32_t smem = E.stages * E.buf_bytes;
    E.last_sweep = sweep;
    E.last_wave = wave;
    const int sv = (int)ctx->sweep_variant;
    // One power of the sweep schedule.  A_perm order with plain or shifted powers and no long
    // rows is exactly the baseline's row kernel (k_spmv_sell, fewest instructions per row); every
    // other case runs k_mpk_sweep (private order, polynomial accumulator, long rows skipped).
    // programmatic dependent launch between consecutive powers on the context stream; not when a
    // side stream joins between them (the event wait must stay a full dependency)
    const bool pdl = ctx->pdl && sweep && !coop && !bw_long;
    auto sweep_power = [&](uint32_t q) {
        const unsigned g = grid_for(E.n_slots, 256, (unsigned)ctx->sm_count * 8u);
        if (!sigma && a.kind <= 1 && !E.long_rows && !coop && sv == 0) {  // (bw_long implies long rows)
            const double* src = a.block + (uint64_t)(q - 1) * a.rows;
            const double* src2 = q >= 2 ? a.block + (uint64_t)(q - 2) * a.rows : src;
            launch_spmv_sell_raw(ctx, S, a.kind == 1, src, a.block + (uint64_t)q * a.rows, src2,
                                 P.shift_a[q - 1], P.shift_b2[q - 1], pdl);
            ctx->launches -= 1;  // counted with the step below
            return;
        }
        switch (a.kind * 2 + (sigma ? 1 : 0)) {
            case 0: launch_sweep<0, false>(sv, g, st, P, q, pdl); break;
            case 1: launch_sweep<0, true>(sv, g, st, P, q, pdl); break;
            case 2: launch_sweep<1, false>(sv, g, st, P, q, pdl); break;
            case 3: launch_sweep<1, true>(sv, g, st, P, q, pdl); break;
            case 4: launch_sweep<2, false>(sv, g, st, P, q, pdl); break;
            default: launch_sweep<2, true>(sv, g, st, P, q, pdl); break;
        }
    };
    // One power: the sweep, plus the rows it skips in fast mode -- k_coop_rows on the side stream
    // (forked from and joined back into the context stream, so a CUDA-graph capture records both
    // branches) or, without cooperative items, k_long_rows_fast after the sweep.
    const unsigned gl = (unsigned)std::min<uint64_t>(std::max<uint64_t>(E.long_rows, 1), (uint64_t)ctx->sm_count * 8u);
    const unsigned gc = (unsigned)std::min<uint64_t>(std::max<uint64_t>((E.n_coop + 7) / 8, 1), (uint64_t)ctx->sm_count * 8u);
    if ((coop || bw_long) && !ctx->aux) {
        const void* fns[6] = {(const void*)k_long_rows_bitwise<0, false>, (const void*)k_long_rows_bitwise<0, true>,
                              (const void*)k_long_rows_bitwise<1, false>, (const void*)k_long_rows_bitwise<1, true>,
                              (const void*)k_long_rows_bitwise<2, false>, (const void*)k_long_rows_bitwise<2, true>};
        for (const void* f : fns)  // once per context (device)
            MPKG_CUDA(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(kBwSlots * kBwChunk * 8)));
        MPKG_CUDA(cudaStreamCreateWithFlags(&ctx->aux, cudaStreamNonBlocking));
        MPKG_CUDA(cudaEventCreateWithFlags(&ctx->fork_ev, cudaEventDisableTiming));
        MPKG_CUDA(cudaEventCreateWithFlags(&ctx->join_ev, cudaEventDisableTiming));
    }
    // bitwise sweeps over a matrix with rows longer than the SELL cap: k_long_rows_bitwise beside
    // the sweep, one CTA per long row, longest first
    FusedParams Pb = P;
    Pb.long_slots = E.long_sorted.p;
    auto power = [&](uint32_t q) {
        const int kk = a.kind * 2 + (sigma ? 1 : 0);
        if (bw_long) {
            cudaStream_t ax = ctx->aux;
            MPKG_CUDA(cudaEventRecord(ctx->fork_ev, st));
            MPKG_CUDA(cudaStreamWaitEvent(ax, ctx->fork_ev, 0));
            const unsigned gb = (unsigned)E.long_rows;  // one CTA per long row, longest first
            const size_t sm = kBwSlots * kBwChunk * 8;
            switch (kk) {
                case 0: k_long_rows_bitwise<0, false><<<gb, 256, sm, ax>>>(Pb, q); break;
                case 1: k_long_rows_bitwise<0, true><<<gb, 256, sm, ax>>>(Pb, q); break;
                case 2: k_long_rows_bitwise<1, false><<<gb, 256, sm, ax>>>(Pb, q); break;
                case 3: k_long_rows_bitwise<1, true><<<gb, 256, sm, ax>>>(Pb, q); break;
                case 4: k_long_rows_bitwise<2, false><<<gb, 256, sm, ax>>>(Pb, q); break;
                default: k_long_rows_bitwise<2, true><<<gb, 256, sm, ax>>>(Pb, q); break;
            }
            MPKG_LAUNCH_CHECK();
            MPKG_CUDA(cudaEventRecord(ctx->join_ev, ax));
            sweep_power(q);
            MPKG_LAUNCH_CHECK();
            MPKG_CUDA(cudaStreamWaitEvent(st, ctx->join_ev, 0));
            return;
        }
        if (coop) {
            cudaStream_t ax = ctx->aux;
            MPKG_CUDA(cudaEventRecord(ctx->fork_ev, st));
            MPKG_CUDA(cudaStreamWaitEvent(ax, ctx->fork_ev, 0));
            switch (kk * 4 + (int)(ctx->coop_variant & 3)) {
#define MPKG_COOP_CASE(K, S)                                                        \
    case (K * 2 + S) * 4 + 0: k_coop_rows<K, S, 8, false><<<gc, 256, 0, ax>>>(P, q); break; \
    case (K * 2 + S) * 4 + 1: k_coop_rows<K, S, 16, false><<<gc, 256, 0, ax>>>(P, q); break; \
    case (K * 2 + S) * 4 + 2: k_coop_rows<K, S, 8, true><<<gc, 256, 0, ax>>>(P, q); break; \
    case (K * 2 + S) * 4 + 3: k_coop_rows<K, S, 16, true><<<gc, 256, 0, ax>>>(P, q); break;
                MPKG_COOP_CASE(0, 0) MPKG_COOP_CASE(0, 1) MPKG_COOP_CASE(1, 0)
                MPKG_COOP_CASE(1, 1) MPKG_COOP_CASE(2, 0) MPKG_COOP_CASE(2, 1)
#undef MPKG_COOP_CASE
            }
            MPKG_LAUNCH_CHECK();
            if (E.n_multi) {
                const unsigned gm = grid_for(E.n_multi, 128, (unsigned)ctx->sm_count * 4u);
                switch (kk) {
                    case 0: k_coop_finish<0, false><<<gm, 128, 0, ax>>>(P, q); break;
                    case 1: k_coop_finish<0, true><<<gm, 128, 0, ax>>>(P, q); break;
                    case 2: k_coop_finish<1, false><<<gm, 128, 0, ax>>>(P, q); break;
                    case 3: k_coop_finish<1, true><<<gm, 128, 0, ax>>>(P, q); break;
                    case 4: k_coop_finish<2, false><<<gm, 128, 0, ax>>>(P, q); break;
                    default: k_coop_finish<2, true><<<gm, 128, 0, ax>>>(P, q); break;
                }
                MPKG_LAUNCH_CHECK();
            }
            MPKG_CUDA(cudaEventRecord(ctx->join_ev, ax));
            sweep_power(q);
            MPKG_LAUNCH_CHECK();
            MPKG_CUDA(cudaStreamWaitEvent(st, ctx->join_ev, 0));
            return;
        }
        sweep_power(q);
        MPKG_LAUNCH_CHECK();
        if (E.long_rows) {  // fast mode only (use_sweeps)
            switch (kk) {
                case 0: k_long_rows_fast<0, false><<<gl, 256, 0, st>>>(P, q); break;
                case 1: k_long_rows_fast<0, true><<<gl, 256, 0, st>>>(P, q); break;
                case 2: k_long_rows_fast<1, false><<<gl, 256, 0, st>>>(P, q); break;
                case 3: k_long_rows_fast<1, true><<<gl, 256, 0, st>>>(P, q); break;
                case 4: k_long_rows_fast<2, false><<<gl, 256, 0, st>>>(P, q); break;
                default: k_long_rows_fast<2, true><<<gl, 256, 0, st>>>(P, q); break;
            }
            MPKG_LAUNCH_CHECK();
        }
    };
    const uint64_t per_power = 1 + (coop ? 1 + (E.n_multi ? 1 : 0) : (E.long_rows ? 1 : 0));
    if (x_pending && !(sweep && !resident && ctx->graphs && a.host_block == nullptr)) copy_x();
    const auto ev = timing_begin(ctx);
    // host-pointer calls: slice q goes to the host on the copy stream once power q is written
    const bool to_host = a.host_block != nullptr;
    auto copy_slice = [&](uint32_t q) {
        if (!to_host || a.rows == 0 || q == 0) return;  // slice 0 (= x): the host copies it
        if (!ctx->d2h) MPKG_CUDA(cudaStreamCreateWithFlags(&ctx->d2h, cudaStreamNonBlocking));
        while (ctx->d2h_events.size() <= q) {
            cudaEvent_t e;
            MPKG_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
            ctx->d2h_events.push_back(e);
        }
        MPKG_CUDA(cudaEventRecord(ctx->d2h_events[q], st));
        MPKG_CUDA(cudaStreamWaitEvent(ctx->d2h, ctx->d2h_events[q], 0));
        MPKG_CUDA(cudaMemcpyAsync(a.host_block + (uint64_t)q * a.rows, a.block + (uint64_t)q * a.rows,
                                  8ull * a.rows, cudaMemcpyDeviceToHost, ctx->d2h));
    };
    auto join_copies = [&]() {  // the context stream (and so the caller's sync) covers the copies
        if (!to_host || a.rows == 0 || a.p < 1) return;
        MPKG_CUDA(cudaEventRecord(ctx->d2h_events[0], ctx->d2h));
        MPKG_CUDA(cudaStreamWaitEvent(st, ctx->d2h_events[0], 0));
    };
    if (sweep && to_host) {
        // one launch per power with the copies interleaved (no graph: the copy stream waits on
        // per-power events); the PCIe transfer of slice q overlaps the sweeps q+1..p
        for (uint32_t q = 1; q <= (uint32_t)a.p; ++q) {
            power(q);
            copy_slice(q);
        }
        join_copies();
        ctx->launches += (uint64_t)a.p * per_power - 1;
    } else if (sweep && resident) {
        const int kk = a.kind * 2 + (sigma ? 1 : 0);
        static void* const fns[6] = {(void*)k_mpk_resident<0, false>, (void*)k_mpk_resident<0, true>,
                                     (void*)k_mpk_resident<1, false>, (void*)k_mpk_resident<1, true>,
                                     (void*)k_mpk_resident<2, false>, (void*)k_mpk_resident<2, true>};
        if (!E.res_bar.p) {
            E.res_bar.alloc(2);
            MPKG_CUDA(cudaMemsetAsync(E.res_bar.p, 0, 8, st));
        }
        if (!E.res_grid[kk]) {
            int per_sm = 0;
            MPKG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fns[kk], 256, 0));
            const uint64_t need = (E.n_slots + 255) / 256;
            E.res_grid[kk] = (int)std::max<uint64_t>(1, std::min<uint64_t>((uint64_t)per_sm * ctx->sm_count, need));
        }
        uint32_t* bar = E.res_bar.p;
        void* args[] = {(void*)&P, (void*)&bar};
        MPKG_CUDA(cudaLaunchCooperativeKernel(fns[kk], dim3(E.res_grid[kk]), dim3(256), args, 0, st));
    } else if (sweep) {
        const bool graph_x = x_pending;
        auto launch_all = [&]() {
            if (graph_x) copy_x();
            for (uint32_t q = 1; q <= (uint32_t)a.p; ++q) power(q);
        };
        if (ctx->graphs) {
            // One CUDA graph per distinct launch set (parameters, p, kind): repeated calls with
            // the same buffers replay all p sweeps with a single launch (C1 is launch-bound).
            std::vector<unsigned char> key(sizeof(FusedParams) + 16 + sizeof(void*));
            std::memcpy(key.data(), &P, sizeof(FusedParams));
            const int32_t extra[4] = {a.kind, a.p, sigma ? 1 : 0, (int32_t)E.long_rows};
            std::memcpy(key.data() + sizeof(FusedParams), extra, sizeof(extra));
            const void* xk = graph_x ? (const void*)a.x : nullptr;  // the captured copy's source
            std::memcpy(key.data() + sizeof(FusedParams) + 16, &xk, sizeof(xk));
            cudaGraphExec_t exec = nullptr;
            for (auto& gr : E.graphs)
                if (gr.first == key) exec = gr.second;
            if (!exec) {
                MPKG_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
                cudaGraph_t graph = nullptr;
                try {
                    launch_all();
                } catch (...) {
                    (void)cudaStreamEndCapture(st, &graph);
                    if (graph) cudaGraphDestroy(graph);
                    throw;
                }
                MPKG_CUDA(cudaStreamEndCapture(st, &graph));
                const cudaError_t e = cudaGraphInstantiate(&exec, graph, 0);
                cudaGraphDestroy(graph);
                MPKG_CUDA(e);
                if (E.graphs.size() >= 8) {
                    cudaGraphExecDestroy(E.graphs.front().second);
                    E.graphs.erase(E.graphs.begin());
                }
                E.graphs.emplace_back(std::move(key), exec);
            }
            MPKG_CUDA(cudaGraphLaunch(exec, st));
        } else {
            launch_all();
        }
        ctx->launches += (uint64_t)a.p * per_power - 1;  // kernels the step ran
    } else if (wave) {
        // one cooperative launch per pass (all CTAs resident: static ticket assignment); with a
        // host block, the pass's slices go to the host while the next pass runs
        // (the polynomial: plain powers here, then z from the finished slices, k_poly_combine)
        void* fn = wave_fn(a.kind == 2 ? 0 : a.kind, sigma, E.wave_fmt, P.trace != nullptr);
        P.counter = E.counter.p;
        P.dbg = getenv("MPKG_WAVE_DEBUG") ? E.counter.p + kWaveStreams * 32 : nullptr;
        for (size_t j = 0; j + 1 < W->t_begin.size(); ++j) {
            uint32_t t0 = W->t_begin[j], t1 = W->t_begin[j + 1], q0 = (uint32_t)W->q_begin[j];
            const uint32_t q1 = (uint32_t)W->q_begin[j + 1] - 1;
            MPKG_CUDA(cudaMemsetAsync(E.counter.p, 0, 4ull * kWaveStreams * 32, st));
            if (j == 0 && q1 > q0) {  // the slices read inside the pass start out empty (later
                                      // passes: filled by the pass before, fill_lo..fill_hi)
                k_wave_fill<<<grid_for(P.vstride, 256, (unsigned)ctx->sm_count * 8u), 256, 0, st>>>(
                    P.V, P.vstride, sigma ? E.n_slots : A->n_rows, q0, q1);
                MPKG_LAUNCH_CHECK();
                ctx->launches += 1;
            }
            uint32_t fill_lo = 0, fill_hi = 0;
            if (j + 2 < W->t_begin.size()) {
                fill_lo = (uint32_t)W->q_begin[j + 1];
                fill_hi = (uint32_t)W->q_begin[j + 2] - 1;
            }
            const unsigned g = (unsigned)std::max<uint64_t>(
                1, std::min<uint64_t>(E.wave_grid, (t1 - t0 + kWaveWarps - 1) / kWaveWarps));
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3(g);
            cfg.blockDim = dim3(kWaveThreads);
            cfg.dynamicSmemBytes = wave_smem_for(E.wave_fmt, sigma);
            cfg.stream = st;
            cudaLaunchAttribute attr[1];
            attr[0].id = cudaLaunchAttributeCooperative;
            attr[0].val.cooperative = 1;
            cfg.attrs = attr;
            cfg.numAttrs = 1;
            uint32_t q1a = q1;
            void* args[] = {(void*)&P, (void*)&t0, (void*)&t1, (void*)&q0, (void*)&q1a, (void*)&fill_lo, (void*)&fill_hi};
            MPKG_CUDA(cudaLaunchKernelExC(&cfg, fn, args));
            if (j + 2 < W->t_begin.size()) ctx->launches += 1;
            if (to_host)
                for (int q = W->q_begin[j]; q < W->q_begin[j + 1]; ++q) copy_slice((uint32_t)q);
        }
        if (a.kind == 2) {
            DevBuf<double>& cf = E.poly_coef;
            cf.ensure(kMaxFusedP + 1);
            MPKG_CUDA(cudaMemcpyAsync(cf.p, P.coef, sizeof(double) * (a.p + 1), cudaMemcpyHostToDevice, st));
            k_poly_combine<<<grid_for(A->n_rows, 256, (unsigned)ctx->sm_count * 8u), 256, 0, st>>>(
                a.block, a.rows, A->n_rows, (uint32_t)a.p, cf.p, a.z);
            MPKG_LAUNCH_CHECK();
            ctx->launches += 1;
        }
        if (to_host) join_copies();
        if (getenv("MPKG_WAVE_DEBUG")) {
            uint32_t misses = 0;
            MPKG_CUDA(cudaMemcpyAsync(&misses, E.counter.p + kWaveStreams * 32, 4, cudaMemcpyDeviceToHost, st));
            MPKG_CUDA(cudaStreamSynchronize(st));
            fprintf(stderr, "wave: p=%d passes=%zu tickets=%zu slack=%lld window=%llu misses=%u\n", a.p,
                    W->t_begin.size() - 1, (size_t)W->t_begin.back(), (long long)W->slack,
                    (unsigned long long)W->window, misses);
            MPKG_CUDA(cudaMemsetAsync(E.counter.p + kWaveStreams * 32, 0, 4, st));
        }
    } else if (E.kernel == 4) {
        const int nt = (int)E.threads;
        const uint32_t sm = E.stages * E.buf_bytes;
        switch (a.kind * 2 + (sigma ? 1 : 0)) {
            case 0: k_mpk_async<0, false><<<E.grid, nt, sm, st>>>(P); break;
            case 1: k_mpk_async<0, true><<<E.grid, nt, sm, st>>>(P); break;
            case 2: k_mpk_async<1, false><<<E.grid, nt, sm, st>>>(P); break;
            case 3: k_mpk_async<1, true><<<E.grid, nt, sm, st>>>(P); break;
            case 4: k_mpk_async<2, false><<<E.grid, nt, sm, st>>>(P); break;
            default: k_mpk_async<2, true><<<E.grid, nt, sm, st>>>(P); break;
        }
    } else if (E.kernel == 2) {
        const uint32_t wsmem = 128 * E.wt_lmax * 8;
        if (E.group == 16)
            launch_warptile<8>(a.kind, sigma, E.grid, wsmem, st, P);
        else
            launch_warptile<4>(a.kind, sigma, E.grid, wsmem, st, P);
    } else if (E.kernel == 0) {
        const int nt = (int)std::min<uint32_t>(E.tile_rows, 128u);
        switch (a.kind * 2 + (sigma ? 1 : 0)) {
            case 0: launch_lean<0, false>(E.sb, E.grid, nt, st, P); break;
            case 1: launch_lean<0, true>(E.sb, E.grid, nt, st, P); break;
            case 2: launch_lean<1, false>(E.sb, E.grid, nt, st, P); break;
            case 3: launch_lean<1, true>(E.sb, E.grid, nt, st, P); break;
            case 4: launch_lean<2, false>(E.sb, E.grid, nt, st, P); break;
            default: launch_lean<2, true>(E.sb, E.grid, nt, st, P); break;
        }
    } else {
        switch (a.kind) {
            case 0: launch_kind<0>(sigma, E, smem, st, P); break;
            case 1: launch_kind<1>(sigma, E, smem, st, P); break;
            default: launch_kind<2>(sigma, E, smem, st, P); break;
        }
    }
    MPKG_LAUNCH_CHECK();
    timing_end(ctx, ev);
    ctx->launches += 1;
    if (to_host && !sweep && !wave) {  // fused kernel: one copy at the end
        for (uint32_t q = 1; q <= (uint32_t)a.p; ++q) copy_slice(q);
        join_copies();
    }
}

void exec_info(const mpkg_plan_s* P, uint32_t* n_tiles, uint64_t* n_tickets, uint64_t* n_deps,
               uint32_t* pass_powers) {
    uint32_t t = 0, pp = 0;
    uint64_t k = 0, d = 0;
    if (P->exec) {
        t = P->exec->n_tiles;
        for (const auto& kv : P->exec->tickets) k = std::max<uint64_t>(k, kv.second.n);
        for (const auto& kv : P->exec->pass_len) pp = (uint32_t)kv.second;
        for (size_t i = 0; i < P->exec->h_lo.size(); ++i) d += P->exec->h_hi[i] - P->exec->h_lo[i] + 1;
        if (P->exec->last_wave) {
            d = P->exec->wave_dep_tiles;
            for (const auto& kv : P->exec->wave) k = std::max<uint64_t>(k, kv.second.tickets.n);
        }
    }
    if (n_tiles) *n_tiles = t;
    if (n_tickets) *n_tickets = k;
    if (n_deps) *n_deps = d;
    if (pass_powers) *pass_powers = pp;
}

void exec_wave(const mpkg_plan_s* P, int* format, uint64_t* n_chunks, uint64_t* n_affine, uint64_t* n_banded,
               uint64_t* record_bytes) {
    const Executor* E = P->exec.get();
    const bool w = E && E->wrec.p != nullptr;
    if (format) *format = w ? E->wave_fmt : 0;
    if (n_chunks) *n_chunks = w ? (uint64_t)E->n_tiles * kWaveChunks : 0;
    if (n_affine) *n_affine = w ? E->wave_affine_chunks : 0;
    if (n_banded) *n_banded = w ? E->wave_banded_chunks : 0;
    if (record_bytes) *record_bytes = w ? E->wave_rec_total : 0;
}

void exec_trace(const mpkg_plan_s* P, uint64_t* out, uint64_t cap, uint64_t* n, uint32_t* tile_rows) {
    const Executor* E = P->exec.get();
    const uint64_t m = E ? E->trace_n : 0;
    if (n) *n = m;
    if (tile_rows) *tile_rows = E ? E->tile_rows : 0;
    if (out && m) {
        if (cap < m) fail(MPKG_EINVAL, "plan_exec_trace: buffer too small");
        MPKG_CUDA(cudaMemcpy(out, E->trace.p, 8 * m, cudaMemcpyDeviceToHost));
    }
}

void exec_mode(const mpkg_plan_s* P, int* order, int* sweeps, int* kernel, uint64_t* long_rows) {
    const Executor* E = P->exec.get();
    if (order) *order = E ? E->order : -1;
    if (sweeps) *sweeps = E ? (E->last_sweep ? 1 : E->last_wave ? 2 : 0) : 0;
    if (kernel) *kernel = E ? E->kernel : -1;
    if (long_rows) *long_rows = E ? E->long_rows : 0;
}

}  // namespace mpkg_detail
