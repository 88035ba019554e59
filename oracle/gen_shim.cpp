// TEST / HARNESS INFRASTRUCTURE ONLY — host-only generator library for the reference arm.
//
// bench.py's `--impl reference` leg and tests/golden/make_config_digests.py need the BASELINE.json
// inputs (C2 scrambled 27-point, C3 R-MAT, C4 27-point, C5 7-point) without loading the product
// library.  This translation unit compiles the harness generators (the same source the product's
// mpkg_gen uses, paper_2309_02228_b200/csrc/generators.cpp, bit-identical to the reference's
// generators.hpp where one exists: tests/test_generators.py) into oracle/_gen/libmpkgen.so, with
// only the error plumbing the generators need.  No kernel, no CUDA, no reference header.
#include <cstdarg>
#include <cstdio>
#include <string>

#include "../paper_2309_02228_b200/csrc/generators.cpp"

namespace mpkg_detail {
thread_local std::string g_gen_error;
void set_error(const char* fmt, ...) {
    char buf[1024];
    va_list ap;
    va_start(ap, fmt);
    std::vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_gen_error = buf;
}
}  // namespace mpkg_detail

extern "C" const char* gen_last_error(void) { return mpkg_detail::g_gen_error.c_str(); }
