// Multi-GPU level-range shards behind the C ABI: the partition and halo plan
// (pure host functions), an NCCL communicator, the one-time scatter of the matrix blocks and of
// x from a root rank, and the per-step halo exchange of x (grouped ncclSend / ncclRecv on the
// context's stream into a preallocated buffer) followed by the local MPK.
//
// The partition (rank r owns the BFS levels [bounds[r], bounds[r+1]), balanced by nnz) and the
// p-deep ghost levels on each side follow from the level adjacency property (levels.hpp:17-24,
// SPEC.md:144): row i's columns lie in levels level(i)-1 .. level(i)+1, so power k is valid on the
// own rows plus ghost depth p-k (redundant-compute, communication-avoiding MPK) and ONE exchange
// of x per MPK call suffices.  Own rows are computed by the same formula from the same inputs as
// on one GPU: bit-identical results for any number of ranks.  multi.py is the Python mirror (the
// gloo path of the CPU tests); tests/test_dist_abi.py checks the two plans agree.
//
// NCCL is loaded at run time (libnccl.so.2, the one already in the process if the host loaded
// one): only the mpkg_dist_* entries need it.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstring>
#include <mutex>
#include <vector>

#include "common.h"
#include "device.h"

using namespace mpkg_detail;

namespace {

void use_device(mpkg_ctx_s* ctx) { MPKG_CUDA(cudaSetDevice(ctx->device)); }

struct Nccl {
    bool ok = false;
    std::string why;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Bcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char* (*ErrorString)(ncclResult_t) = nullptr;
};

const Nccl& nccl() {
    static Nccl N;
    static std::once_flag once;
    std::call_once(once, [] {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            N.why = std::string("libnccl.so.2 not found: ") + dlerror();
            return;
        }
        auto sym = [&](const char* name) {
            void* s = dlsym(h, name);
            if (!s) N.why += std::string(" missing ") + name;
            return s;
        };
        N.GetUniqueId = reinterpret_cast<decltype(N.GetUniqueId)>(sym("ncclGetUniqueId"));
        N.CommInitRank = reinterpret_cast<decltype(N.CommInitRank)>(sym("ncclCommInitRank"));
        N.CommDestroy = reinterpret_cast<decltype(N.CommDestroy)>(sym("ncclCommDestroy"));
        N.Send = reinterpret_cast<decltype(N.Send)>(sym("ncclSend"));
        N.Recv = reinterpret_cast<decltype(N.Recv)>(sym("ncclRecv"));
        N.Bcast = reinterpret_cast<decltype(N.Bcast)>(sym("ncclBroadcast"));
        N.GroupStart = reinterpret_cast<decltype(N.GroupStart)>(sym("ncclGroupStart"));
        N.GroupEnd = reinterpret_cast<decltype(N.GroupEnd)>(sym("ncclGroupEnd"));
        N.ErrorString = reinterpret_cast<decltype(N.ErrorString)>(sym("ncclGetErrorString"));
        N.ok = N.why.empty();
    });
    return N;
}

void nccl_check(ncclResult_t r, const char* what) {
    if (r != ncclSuccess)
        fail(MPKG_ECUDA, std::string(what) + ": " + (nccl().ErrorString ? nccl().ErrorString(r) : "NCCL error"));
}
const Nccl& need_nccl() {
    const Nccl& N = nccl();
    if (!N.ok) fail(MPKG_EINTERNAL, "dist: NCCL unavailable (" + N.why + ")");
    return N;
}

// Halo plan of one rank (global A_perm rows).  send[r] / recv[r]: the row range this rank sends to
// / receives from rank r (empty: lo == hi).  Mirrors multi.halo_plan.
struct Halo {
    uint32_t own[2] = {0, 0};
    uint32_t local[2] = {0, 0};
    std::vector<uint32_t> send, recv;  // 2 * world
};

void own_rows(const uint32_t* lp, const uint32_t* bounds, int r, uint32_t* o) {
    o[0] = lp[bounds[r]];
    o[1] = lp[bounds[r + 1]];
}
void local_rows(const uint32_t* lp, uint32_t nl, const uint32_t* bounds, int r, int p, uint32_t* g) {
    const uint32_t L0 = bounds[r], L1 = bounds[r + 1];
    if (lp[L0] == lp[L1]) {  // empty rank: holds nothing
        g[0] = g[1] = lp[L0];
        return;
    }
    g[0] = lp[L0 >= (uint32_t)p ? L0 - p : 0u];
    g[1] = lp[std::min<uint64_t>(nl, (uint64_t)L1 + p)];
}

Halo make_halo(const uint32_t* lp, uint32_t nl, const uint32_t* bounds, int world, int rank, int p) {
    require(world >= 1 && rank >= 0 && rank < world, "dist: rank outside [0, world)");
    require(p >= 0, "dist: p must be >= 0");
    require(bounds[0] == 0 && bounds[world] == nl, "dist: bounds must start at 0 and end at n_levels");
    for (int r = 0; r < world; ++r) require(bounds[r] <= bounds[r + 1], "dist: bounds must be monotone");
    Halo H;
    own_rows(lp, bounds, rank, H.own);
    local_rows(lp, nl, bounds, rank, p, H.local);
    H.send.assign(2 * world, 0);
    H.recv.assign(2 * world, 0);
    for (int r = 0; r < world; ++r) {
        if (r == rank) continue;
        uint32_t o[2], g[2];
        own_rows(lp, bounds, r, o);
        local_rows(lp, nl, bounds, r, p, g);
        // I receive r's own rows that fall inside my local range
        const uint32_t a = std::max(o[0], H.local[0]), b = std::min(o[1], H.local[1]);
        if (a < b) H.recv[2 * r] = a, H.recv[2 * r + 1] = b;
        // I send my own rows that fall inside r's local range
        const uint32_t c = std::max(H.own[0], g[0]), d = std::min(H.own[1], g[1]);
        if (c < d) H.send[2 * r] = c, H.send[2 * r + 1] = d;
    }
    return H;
}

}  // namespace

struct mpkg_dist_s {
    mpkg_ctx_s* ctx = nullptr;
    ncclComm_t comm = nullptr;
    int world = 1, rank = 0, p = 0;
    bool planned = false;
    std::vector<uint32_t> level_ptr;
    std::vector<uint32_t> bounds;
    Halo halo;
    DevBuf<double> x_local;  // preallocated local x (rows local[0] .. local[1])
    uint64_t send_bytes = 0, recv_bytes = 0;
};

extern "C" {

int mpkg_dist_partition(const uint32_t* level_ptr, uint32_t n_levels, const uint64_t* nnz_before, int world,
                        uint32_t* bounds) {
    return guarded([&] {
        require(level_ptr && nnz_before && bounds, "dist_partition: null argument");
        require(world >= 1, "dist_partition: world must be >= 1");
        const uint64_t total = nnz_before[n_levels];
        bounds[0] = 0;
        for (int r = 1; r < world; ++r) {  // first level boundary with nnz_before >= total * r / world
            const double target = (double)total * r / world;
            const uint64_t* it = std::lower_bound(nnz_before, nnz_before + n_levels + 1, target,
                                                  [](uint64_t v, double t) { return (double)v < t; });
            uint32_t L = (uint32_t)(it - nnz_before);
            L = std::max(L, bounds[r - 1]);
            bounds[r] = std::min(L, n_levels);
        }
        bounds[world] = n_levels;
    });
}

int mpkg_dist_halo(const uint32_t* level_ptr, uint32_t n_levels, const uint32_t* bounds, int world, int rank,
                   int p, uint32_t* own, uint32_t* local, uint32_t* send, uint32_t* recv) {
    return guarded([&] {
        require(level_ptr && bounds && own && local && send && recv, "dist_halo: null argument");
        const Halo H = make_halo(level_ptr, n_levels, bounds, world, rank, p);
        own[0] = H.own[0], own[1] = H.own[1];
        local[0] = H.local[0], local[1] = H.local[1];
        std::copy(H.send.begin(), H.send.end(), send);
        std::copy(H.recv.begin(), H.recv.end(), recv);
    });
}

int mpkg_dist_unique_id(void* id) {
    return guarded([&] {
        require(id != nullptr, "dist_unique_id: null argument");
        ncclUniqueId u;
        nccl_check(need_nccl().GetUniqueId(&u), "ncclGetUniqueId");
        std::memcpy(id, &u, sizeof(u));
    });
}

int mpkg_dist_create(mpkg_ctx_t ctx, const void* id, int world, int rank, mpkg_dist_t* out) {
    return guarded([&] {
        require(ctx && id && out, "dist_create: null argument");
        require(world >= 1 && rank >= 0 && rank < world, "dist_create: rank outside [0, world)");
        const Nccl& N = need_nccl();
        use_device(ctx);
        auto* D = new mpkg_dist_s();
        D->ctx = ctx;
        D->world = world;
        D->rank = rank;
        ncclUniqueId u;
        std::memcpy(&u, id, sizeof(u));
        const ncclResult_t r = N.CommInitRank(&D->comm, world, u, rank);
        if (r != ncclSuccess) {
            delete D;
            nccl_check(r, "ncclCommInitRank");
        }
        *out = D;
    });
}

int mpkg_dist_destroy(mpkg_dist_t D) {
    return guarded([&] {
        if (!D) return;
        use_device(D->ctx);
        if (D->comm) nccl().CommDestroy(D->comm);
        delete D;
    });
}

int mpkg_dist_bcast_host(mpkg_dist_t D, void* buf, uint64_t bytes, int root) {
    return guarded([&] {
        require(D && (buf || bytes == 0), "dist_bcast_host: null argument");
        require(root >= 0 && root < D->world, "dist_bcast_host: root outside [0, world)");
        if (bytes == 0) return;
        use_device(D->ctx);
        DevBuf<uint8_t> tmp(bytes);
        cudaStream_t st = D->ctx->stream;
        if (D->rank == root) MPKG_CUDA(cudaMemcpyAsync(tmp.p, buf, bytes, cudaMemcpyHostToDevice, st));
        nccl_check(need_nccl().Bcast(tmp.p, tmp.p, bytes, ncclUint8, root, D->comm, st), "ncclBroadcast");
        MPKG_CUDA(cudaMemcpyAsync(buf, tmp.p, bytes, cudaMemcpyDeviceToHost, st));
        MPKG_CUDA(cudaStreamSynchronize(st));
    });
}

int mpkg_dist_set_plan(mpkg_dist_t D, const uint32_t* level_ptr, uint32_t n_levels, const uint32_t* bounds,
                       int p) {
    return guarded([&] {
        require(D && level_ptr && bounds, "dist_set_plan: null argument");
        D->halo = make_halo(level_ptr, n_levels, bounds, D->world, D->rank, p);
        D->level_ptr.assign(level_ptr, level_ptr + n_levels + 1);
        D->bounds.assign(bounds, bounds + D->world + 1);
        D->p = p;
        use_device(D->ctx);
        D->x_local.alloc(std::max<uint64_t>(1, D->halo.local[1] - D->halo.local[0]));
        D->send_bytes = D->recv_bytes = 0;
        for (int r = 0; r < D->world; ++r) {
            D->send_bytes += 8ull * (D->halo.send[2 * r + 1] - D->halo.send[2 * r]);
            D->recv_bytes += 8ull * (D->halo.recv[2 * r + 1] - D->halo.recv[2 * r]);
        }
        D->planned = true;
    });
}

int mpkg_dist_info(mpkg_dist_t D, uint32_t* own, uint32_t* local, uint64_t* send_bytes, uint64_t* recv_bytes) {
    return guarded([&] {
        require(D && D->planned, "dist_info: no plan (mpkg_dist_set_plan)");
        if (own) own[0] = D->halo.own[0], own[1] = D->halo.own[1];
        if (local) local[0] = D->halo.local[0], local[1] = D->halo.local[1];
        if (send_bytes) *send_bytes = D->send_bytes;
        if (recv_bytes) *recv_bytes = D->recv_bytes;
    });
}

// Root: every rank's local block A_perm[g0:g1, g0:g1] (cut on the root's GPU, kept entries in
// stored order) goes to its rank; the others receive theirs.  One-time setup, not per step.
int mpkg_dist_scatter_blocks(mpkg_dist_t D, int root, mpkg_csr_t A_perm, mpkg_csr_t* out) {
    return guarded([&] {
        require(D && D->planned && out, "dist_scatter_blocks: null argument or no plan");
        require(root >= 0 && root < D->world, "dist_scatter_blocks: root outside [0, world)");
        const Nccl& N = need_nccl();
        use_device(D->ctx);
        cudaStream_t st = D->ctx->stream;
        const uint32_t nl = (uint32_t)D->level_ptr.size() - 1;
        std::vector<mpkg_csr_s*> blocks;
        DevBuf<uint64_t> hdr(2);
        auto* B = new mpkg_csr_s();
        try {
            if (D->rank == root) {
                require(A_perm && A_perm->n_rows == D->level_ptr.back(), "dist_scatter_blocks: root needs A_perm");
                for (int r = 0; r < D->world; ++r) {
                    uint32_t g[2];
                    local_rows(D->level_ptr.data(), nl, D->bounds.data(), r, D->p, g);
                    auto* Br = r == root ? B : new mpkg_csr_s();
                    if (r != root) blocks.push_back(Br);
                    gpu_csr_block(D->ctx, A_perm, g[0], g[1], g[0], g[1], Br);
                }
                size_t bi = 0;
                for (int r = 0; r < D->world; ++r) {
                    if (r == root) continue;
                    mpkg_csr_s* Br = blocks[bi++];
                    const uint64_t h[2] = {Br->n_rows, Br->nnz};
                    MPKG_CUDA(cudaMemcpyAsync(hdr.p, h, 16, cudaMemcpyHostToDevice, st));
                    nccl_check(N.Send(hdr.p, 2, ncclUint64, r, D->comm, st), "ncclSend");
                    nccl_check(N.GroupStart(), "ncclGroupStart");
                    nccl_check(N.Send(Br->row_ptr.p, Br->n_rows + 1ull, ncclUint32, r, D->comm, st), "ncclSend");
                    if (Br->nnz) {
                        nccl_check(N.Send(Br->col_idx.p, Br->nnz, ncclUint32, r, D->comm, st), "ncclSend");
                        nccl_check(N.Send(Br->values.p, Br->nnz, ncclFloat64, r, D->comm, st), "ncclSend");
                    }
                    nccl_check(N.GroupEnd(), "ncclGroupEnd");
                }
                MPKG_CUDA(cudaStreamSynchronize(st));
            } else {
                nccl_check(N.Recv(hdr.p, 2, ncclUint64, root, D->comm, st), "ncclRecv");
                uint64_t h[2];
                MPKG_CUDA(cudaMemcpyAsync(h, hdr.p, 16, cudaMemcpyDeviceToHost, st));
                MPKG_CUDA(cudaStreamSynchronize(st));
                B->ctx = D->ctx;
                B->device = D->ctx->device;
                B->n_rows = B->n_cols = (uint32_t)h[0];
                B->nnz = (uint32_t)h[1];
                B->row_ptr.alloc(h[0] + 1);
                B->col_idx.alloc(h[1] + 1);
                B->values.alloc(h[1] + 1);
                nccl_check(N.GroupStart(), "ncclGroupStart");
                nccl_check(N.Recv(B->row_ptr.p, h[0] + 1, ncclUint32, root, D->comm, st), "ncclRecv");
                if (h[1]) {
                    nccl_check(N.Recv(B->col_idx.p, h[1], ncclUint32, root, D->comm, st), "ncclRecv");
                    nccl_check(N.Recv(B->values.p, h[1], ncclFloat64, root, D->comm, st), "ncclRecv");
                }
                nccl_check(N.GroupEnd(), "ncclGroupEnd");
                MPKG_CUDA(cudaStreamSynchronize(st));
            }
        } catch (...) {
            for (auto* b : blocks) delete b;
            delete B;
            throw;
        }
        for (auto* b : blocks) delete b;
        *out = B;
    });
}

// Root: every rank's own rows of a global device vector (A_perm order) go to its rank.
int mpkg_dist_scatter_rows(mpkg_dist_t D, int root, const double* d_full, double* d_own) {
    return guarded([&] {
        require(D && D->planned && (d_own || D->halo.own[0] == D->halo.own[1]), "dist_scatter_rows: null argument or no plan");
        const Nccl& N = need_nccl();
        use_device(D->ctx);
        cudaStream_t st = D->ctx->stream;
        nccl_check(N.GroupStart(), "ncclGroupStart");
        if (D->rank == root) {
            require(d_full != nullptr, "dist_scatter_rows: root needs the full vector");
            for (int r = 0; r < D->world; ++r) {
                uint32_t o[2];
                own_rows(D->level_ptr.data(), D->bounds.data(), r, o);
                if (o[0] == o[1]) continue;
                if (r == root)
                    MPKG_CUDA(cudaMemcpyAsync(d_own, d_full + o[0], 8ull * (o[1] - o[0]), cudaMemcpyDeviceToDevice, st));
                else
                    nccl_check(N.Send(d_full + o[0], o[1] - o[0], ncclFloat64, r, D->comm, st), "ncclSend");
            }
        } else if (D->halo.own[1] > D->halo.own[0]) {
            nccl_check(N.Recv(d_own, D->halo.own[1] - D->halo.own[0], ncclFloat64, root, D->comm, st), "ncclRecv");
        }
        nccl_check(N.GroupEnd(), "ncclGroupEnd");
        MPKG_CUDA(cudaStreamSynchronize(st));
    });
}

// The halo exchange: the local x (rows local[0] .. local[1]) from this rank's own rows and the
// peers' pieces, one grouped set of ncclSend / ncclRecv on the context's stream (asynchronous).
int mpkg_dist_exchange(mpkg_dist_t D, const double* d_x_own, double** d_x_local) {
    return guarded([&] {
        require(D && D->planned, "dist_exchange: no plan (mpkg_dist_set_plan)");
        const Halo& H = D->halo;
        require(d_x_own || H.own[0] == H.own[1], "dist_exchange: null x");
        use_device(D->ctx);
        cudaStream_t st = D->ctx->stream;
        double* xl = D->x_local.p;
        const uint32_t g0 = H.local[0];
        if (H.own[1] > H.own[0])
            MPKG_CUDA(cudaMemcpyAsync(xl + (H.own[0] - g0), d_x_own, 8ull * (H.own[1] - H.own[0]),
                                      cudaMemcpyDeviceToDevice, st));
        if (D->world > 1) {
            const Nccl& N = need_nccl();
            nccl_check(N.GroupStart(), "ncclGroupStart");
            for (int r = 0; r < D->world; ++r) {
                const uint32_t s0 = H.send[2 * r], s1 = H.send[2 * r + 1];
                if (s1 > s0) nccl_check(N.Send(d_x_own + (s0 - H.own[0]), s1 - s0, ncclFloat64, r, D->comm, st), "ncclSend");
                const uint32_t r0 = H.recv[2 * r], r1 = H.recv[2 * r + 1];
                if (r1 > r0) nccl_check(N.Recv(xl + (r0 - g0), r1 - r0, ncclFloat64, r, D->comm, st), "ncclRecv");
            }
            nccl_check(N.GroupEnd(), "ncclGroupEnd");
        }
        if (d_x_local) *d_x_local = xl;
    });
}

int mpkg_dist_mpk(mpkg_dist_t D, mpkg_plan_t P, mpkg_csr_t A_local, const double* d_x_own, int p,
                  double* d_block, uint64_t block_rows, uint64_t block_slices) {
    double* xl = nullptr;
    int rc = mpkg_dist_exchange(D, d_x_own, &xl);
    if (rc != MPKG_OK) return rc;
    if (D->halo.local[1] == D->halo.local[0]) return MPKG_OK;
    return mpkg_mpk_dev(D->ctx, P, A_local, xl, p, d_block, block_rows, block_slices);
}

}  // extern "C"
