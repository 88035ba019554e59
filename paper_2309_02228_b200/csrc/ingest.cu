// Matrix ingestion: from_coo on the GPU and the Matrix Market
// reader feeding it.
//
//   from_coo (csr.hpp:72-110): stable sort of the entries by (row, col) -- an LSD radix sort of
//   the 64-bit key (row << 32 | col) carrying the input index, which keeps equal keys in input
//   order -- then every run of equal keys is summed in that order starting from 0.0 (so a lone
//   -0.0 becomes +0.0, exactly like the reference), and empty rows inherit the previous offset.
//   Bit-identical to the reference.
//
//   read_matrix_market (matrix_market.hpp:48-113): banner / size-line / entry-line rules and error
//   messages of the reference; decimal values parsed with strtod (what the reference's
//   istream >> double does in libstdc++), symmetric / skew-symmetric expansion in line order; the
//   triplets then go through the GPU from_coo.  Parsing is host work (text), assembly is device
//   work (the sort and dedupe that make the reference's from_coo the memory bottleneck at 512^3).
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include <cctype>
#include <cerrno>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <limits>
#include <sstream>
#include <string>
#include <vector>

#include "device.h"

namespace mpkg_detail {

namespace {

__global__ void k_coo_check(const uint32_t* __restrict__ r, const uint32_t* __restrict__ c, uint64_t m,
                            uint32_t n_rows, uint32_t n_cols, unsigned long long* __restrict__ bad) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m; i += (uint64_t)gridDim.x * blockDim.x)
        if (r[i] >= n_rows || c[i] >= n_cols) atomicMin(bad, (unsigned long long)i);
}

__global__ void k_coo_keys(const uint32_t* __restrict__ r, const uint32_t* __restrict__ c, uint64_t m,
                           uint64_t* __restrict__ key, uint32_t* __restrict__ idx) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m; i += (uint64_t)gridDim.x * blockDim.x) {
        key[i] = ((uint64_t)r[i] << 32) | c[i];
        idx[i] = (uint32_t)i;
    }
}

__global__ void k_coo_heads(const uint64_t* __restrict__ key, uint64_t m, uint32_t* __restrict__ head) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m; i += (uint64_t)gridDim.x * blockDim.x)
        head[i] = (i == 0 || key[i] != key[i - 1]) ? 1u : 0u;
}

__global__ void k_coo_starts(const uint32_t* __restrict__ head, const uint32_t* __restrict__ gid, uint64_t m,
                             uint32_t* __restrict__ start) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m; i += (uint64_t)gridDim.x * blockDim.x)
        if (head[i]) start[gid[i] - 1] = (uint32_t)i;
}

// One thread per unique (row, col): the input-order sum from 0.0 (csr.hpp:97-99).
__global__ void k_coo_sum(const uint64_t* __restrict__ key, const uint32_t* __restrict__ idx,
                          const double* __restrict__ v, const uint32_t* __restrict__ start, uint32_t u,
                          uint32_t* __restrict__ col, double* __restrict__ val, uint32_t* __restrict__ cnt) {
    for (uint64_t g = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; g < u; g += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t b = start[g], e = start[g + 1];
        double sum = 0.0;
        for (uint32_t i = b; i < e; ++i) sum = __dadd_rn(sum, v[idx[i]]);
        col[g] = (uint32_t)(key[b] & 0xffffffffu);
        val[g] = sum;
        atomicAdd(cnt + (key[b] >> 32), 1u);
    }
}

}  // namespace

void gpu_from_coo(mpkg_ctx_s* ctx, uint32_t n_rows, uint32_t n_cols, uint64_t m, const uint32_t* d_r,
                  const uint32_t* d_c, const double* d_v, mpkg_csr_s* B) {
    cudaStream_t st = ctx->stream;
    if (m >= (1ull << 31)) fail(MPKG_EINVAL, "from_coo: entry count exceeds 32-bit index range");
    B->ctx = ctx;
    B->device = ctx->device;
    B->n_rows = n_rows;
    B->n_cols = n_cols;
    B->row_ptr.alloc((uint64_t)n_rows + 1);
    const unsigned grid = grid_for(std::max<uint64_t>(m, 1), 256, (unsigned)ctx->sm_count * 8u);
    if (m) {  // csr.hpp:76-82: the first offending entry in input order
        DevBuf<unsigned long long> bad(1);
        MPKG_CUDA(cudaMemsetAsync(bad.p, 0xff, 8, st));
        k_coo_check<<<grid, 256, 0, st>>>(d_r, d_c, m, n_rows, n_cols, bad.p);
        MPKG_LAUNCH_CHECK();
        unsigned long long h = 0;
        MPKG_CUDA(cudaMemcpyAsync(&h, bad.p, 8, cudaMemcpyDeviceToHost, st));
        MPKG_CUDA(cudaStreamSynchronize(st));
        if (h != ~0ull) {
            uint32_t rc[2];
            MPKG_CUDA(cudaMemcpy(&rc[0], d_r + h, 4, cudaMemcpyDeviceToHost));
            MPKG_CUDA(cudaMemcpy(&rc[1], d_c + h, 4, cudaMemcpyDeviceToHost));
            fail(MPKG_EINVAL, "from_coo: entry index out of range at (" + std::to_string(rc[0]) + ", " +
                                  std::to_string(rc[1]) + ")");
        }
    }
    DevBuf<uint32_t> cnt((uint64_t)n_rows + 1);
    MPKG_CUDA(cudaMemsetAsync(cnt.p, 0, cnt.bytes(), st));
    uint32_t u = 0;
    if (m) {
        DevBuf<uint64_t> key(m), key_s(m);
        DevBuf<uint32_t> idx(m), idx_s(m), head(m), gid(m);
        k_coo_keys<<<grid, 256, 0, st>>>(d_r, d_c, m, key.p, idx.p);
        MPKG_LAUNCH_CHECK();
        int end_bit = 32;
        while (end_bit < 64 && (1ull << (end_bit - 32)) < (uint64_t)n_rows) ++end_bit;
        size_t tb = 0;
        MPKG_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, key.p, key_s.p, idx.p, idx_s.p, (int)m, 0, end_bit, st));
        DevBuf<uint8_t> tmp(tb);
        MPKG_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, tb, key.p, key_s.p, idx.p, idx_s.p, (int)m, 0, end_bit, st));
        k_coo_heads<<<grid, 256, 0, st>>>(key_s.p, m, head.p);
        MPKG_LAUNCH_CHECK();
        size_t tb2 = 0;
        MPKG_CUDA(cub::DeviceScan::InclusiveSum(nullptr, tb2, head.p, gid.p, (int)m, st));
        tmp.ensure(tb2);
        MPKG_CUDA(cub::DeviceScan::InclusiveSum(tmp.p, tb2, head.p, gid.p, (int)m, st));
        MPKG_CUDA(cudaMemcpyAsync(&u, gid.p + m - 1, 4, cudaMemcpyDeviceToHost, st));
        MPKG_CUDA(cudaStreamSynchronize(st));
        DevBuf<uint32_t> start((uint64_t)u + 1);
        const uint32_t mm = (uint32_t)m;
        MPKG_CUDA(cudaMemcpyAsync(start.p + u, &mm, 4, cudaMemcpyHostToDevice, st));
        k_coo_starts<<<grid, 256, 0, st>>>(head.p, gid.p, m, start.p);
        MPKG_LAUNCH_CHECK();
        B->col_idx.alloc((uint64_t)u + 1);
        B->values.alloc((uint64_t)u + 1);
        k_coo_sum<<<grid_for(u, 256, (unsigned)ctx->sm_count * 8u), 256, 0, st>>>(
            key_s.p, idx_s.p, d_v, start.p, u, B->col_idx.p, B->values.p, cnt.p);
        MPKG_LAUNCH_CHECK();
        ctx->launches += 7;
        MPKG_CUDA(cudaStreamSynchronize(st));  // scratch above is freed on scope exit
    } else {
        B->col_idx.alloc(1);
        B->values.alloc(1);
    }
    B->nnz = u;
    size_t tb3 = 0;
    MPKG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb3, cnt.p, B->row_ptr.p, (int)(n_rows + 1), st));
    DevBuf<uint8_t> tmp3(tb3);
    MPKG_CUDA(cub::DeviceScan::ExclusiveSum(tmp3.p, tb3, cnt.p, B->row_ptr.p, (int)(n_rows + 1), st));
    MPKG_CUDA(cudaStreamSynchronize(st));
}

// ---- Matrix Market (matrix_market.hpp:48-113) ------------------------------------------------------
namespace {
std::string lower(std::string s) {
    for (char& ch : s) ch = (char)std::tolower((unsigned char)ch);
    return s;
}
[[noreturn]] void mtx_fail(const std::string& m) { fail(MPKG_EINTERNAL, "read_matrix_market: " + m); }

// istream >> uint64_t on a line: skip whitespace, strtoull (accepts a sign, like num_get)
bool next_u64(const char*& p, const char* end, uint64_t& out) {
    while (p < end && std::isspace((unsigned char)*p)) ++p;
    if (p >= end) return false;
    std::string tok;
    const char* q = p;
    while (q < end && !std::isspace((unsigned char)*q)) ++q;
    tok.assign(p, q);
    char* e = nullptr;
    errno = 0;
    const unsigned long long v = std::strtoull(tok.c_str(), &e, 10);
    if (e == tok.c_str() || errno == ERANGE) return false;
    p += (e - tok.c_str());
    out = v;
    return true;
}
// istream >> double (libstdc++ num_get): decimal syntax only -- no "inf" / "nan" / hex -- and the
// token stops at the first character outside [0-9+-.eE]; overflow fails, underflow does not.
bool next_double(const char*& p, const char* end, double& out) {
    while (p < end && std::isspace((unsigned char)*p)) ++p;
    if (p >= end) return false;
    std::string tok;
    const char* q = p;
    while (q < end && (std::isdigit((unsigned char)*q) || *q == '+' || *q == '-' || *q == '.' ||
                       *q == 'e' || *q == 'E'))
        ++q;
    tok.assign(p, q);
    char* e = nullptr;
    errno = 0;
    const double v = std::strtod(tok.c_str(), &e);
    if (e == tok.c_str() || (errno == ERANGE && std::fabs(v) > 1.0)) return false;  // overflow fails
    p += (e - tok.c_str());
    out = v;
    return true;
}
}  // namespace

void read_matrix_market(mpkg_ctx_s* ctx, const char* path, mpkg_csr_s* B) {
    std::ifstream in(path);
    if (!in) mtx_fail(std::string("cannot open ") + path);
    std::string line;
    if (!std::getline(in, line)) mtx_fail(std::string("empty file ") + path);
    std::istringstream banner(line);
    std::string tag, object, format, field, symmetry;
    banner >> tag >> object >> format >> field >> symmetry;
    if (tag != "%%MatrixMarket") mtx_fail(std::string("missing banner in ") + path);
    object = lower(object), format = lower(format), field = lower(field), symmetry = lower(symmetry);
    if (object != "matrix" || format != "coordinate") mtx_fail("unsupported banner '" + line + "'");
    const bool pattern = field == "pattern";
    if (field != "real" && field != "integer" && !pattern) mtx_fail("unsupported field '" + field + "'");
    const bool symmetric = symmetry == "symmetric", skew = symmetry == "skew-symmetric";
    if (symmetry != "general" && !symmetric && !skew) mtx_fail("unsupported symmetry '" + symmetry + "'");
    uint64_t rows = 0, cols = 0, count = 0;
    while (std::getline(in, line)) {  // size line: first non-comment, non-blank line
        if (line.empty() || line[0] == '%') continue;
        const char* p = line.data();
        const char* e = p + line.size();
        if (!(next_u64(p, e, rows) && next_u64(p, e, cols) && next_u64(p, e, count)))
            mtx_fail("malformed size line");
        break;
    }
    if (rows == 0 || cols == 0) mtx_fail("empty dimensions");
    constexpr uint64_t kMaxDim = std::numeric_limits<uint32_t>::max();
    if (rows > kMaxDim || cols > kMaxDim) mtx_fail("dimensions exceed 32-bit range");
    std::vector<uint32_t> ri, ci;
    std::vector<double> vv;
    const uint64_t cap = symmetric || skew ? 2 * count : count;
    ri.reserve(cap), ci.reserve(cap), vv.reserve(cap);
    uint64_t seen = 0;
    while (seen < count && std::getline(in, line)) {
        if (line.empty() || line[0] == '%') continue;
        const char* p = line.data();
        const char* e = p + line.size();
        uint64_t r1 = 0, c1 = 0;
        double v = 1.0;
        if (!(next_u64(p, e, r1) && next_u64(p, e, c1))) mtx_fail("malformed entry line '" + line + "'");
        if (!pattern && !next_double(p, e, v)) mtx_fail("missing value in '" + line + "'");
        if (r1 == 0 || c1 == 0 || r1 > rows || c1 > cols) mtx_fail("entry index out of range");
        const uint32_t r = (uint32_t)(r1 - 1), c = (uint32_t)(c1 - 1);
        ri.push_back(r), ci.push_back(c), vv.push_back(v);
        if ((symmetric || skew) && r != c) ri.push_back(c), ci.push_back(r), vv.push_back(skew ? -v : v);
        ++seen;
    }
    if (seen != count) mtx_fail("fewer entries than declared");
    const uint64_t m = ri.size();
    DevBuf<uint32_t> dr(std::max<uint64_t>(m, 1)), dc(std::max<uint64_t>(m, 1));
    DevBuf<double> dv(std::max<uint64_t>(m, 1));
    if (m) {
        MPKG_CUDA(cudaMemcpyAsync(dr.p, ri.data(), 4 * m, cudaMemcpyHostToDevice, ctx->stream));
        MPKG_CUDA(cudaMemcpyAsync(dc.p, ci.data(), 4 * m, cudaMemcpyHostToDevice, ctx->stream));
        MPKG_CUDA(cudaMemcpyAsync(dv.p, vv.data(), 8 * m, cudaMemcpyHostToDevice, ctx->stream));
    }
    gpu_from_coo(ctx, (uint32_t)rows, (uint32_t)cols, m, dr.p, dc.p, dv.p, B);
}

}  // namespace mpkg_detail
