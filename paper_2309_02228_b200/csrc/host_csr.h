// Host-side CSR container used by the generators (harness inputs) and the upload path.
#pragma once

#include <cstdint>
#include <cstdlib>
#include <new>

// Plain malloc-backed array: no value-initialisation (the generators fill every entry in
// parallel, so first touch is spread across the host cores).
template <class T>
struct HostArray {
    T* p = nullptr;
    uint64_t n = 0;
    HostArray() = default;
    explicit HostArray(uint64_t count) { reset(count); }
    HostArray(const HostArray&) = delete;
    HostArray& operator=(const HostArray&) = delete;
    HostArray(HostArray&& o) noexcept : p(o.p), n(o.n) {
        o.p = nullptr;
        o.n = 0;
    }
    HostArray& operator=(HostArray&& o) noexcept {
        if (this != &o) {
            std::free(p);
            p = o.p;
            n = o.n;
            o.p = nullptr;
            o.n = 0;
        }
        return *this;
    }
    ~HostArray() { std::free(p); }
    void reset(uint64_t count) {
        std::free(p);
        p = count ? static_cast<T*>(std::malloc(sizeof(T) * count)) : nullptr;
        if (count && !p) throw std::bad_alloc();
        n = count;
    }
    T& operator[](uint64_t i) { return p[i]; }
    const T& operator[](uint64_t i) const { return p[i]; }
};

struct mpkg_host_csr_s {
    uint32_t n_rows = 0;
    uint32_t n_cols = 0;
    HostArray<uint32_t> row_ptr;
    HostArray<uint32_t> col_idx;
    HostArray<double> values;
    uint64_t nnz() const { return n_rows ? row_ptr[n_rows] : 0; }
};
