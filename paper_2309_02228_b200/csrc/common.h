// Shared status / error plumbing for the mpkg C ABI (no exception ever crosses the ABI).
#pragma once

#include <cstdarg>
#include <cstdint>
#include <exception>
#include <new>
#include <stdexcept>
#include <string>

#include "mpkg.h"

namespace mpkg_detail {

// Thread-local last-error message (mpkg_last_error).
void set_error(const char* fmt, ...);

// Internal exception carrying an ABI status code.
struct Status : std::runtime_error {
    int code;
    Status(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] inline void fail(int code, const std::string& msg) { throw Status(code, msg); }
inline void require(bool cond, const std::string& msg) {
    if (!cond) fail(MPKG_EINVAL, msg);
}

// Runs f() and maps every exception to a status code + message.
template <class F>
int guarded(F&& f) {
    try {
        f();
        return MPKG_OK;
    } catch (const Status& s) {
        set_error("%s", s.what());
        return s.code;
    } catch (const std::bad_alloc&) {
        set_error("host allocation failed");
        return MPKG_ENOMEM;
    } catch (const std::exception& e) {
        set_error("%s", e.what());
        return MPKG_EINTERNAL;
    } catch (...) {
        set_error("unknown error");
        return MPKG_EINTERNAL;
    }
}

}  // namespace mpkg_detail
