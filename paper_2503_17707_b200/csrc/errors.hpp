// errors.hpp — thread-local error reporting for the C ABI (pb_last_error).
#pragma once
#include <cstdarg>
#include <cstdio>
#include <exception>
#include <new>

#include "../../include/pipeboost.h"

namespace pb {

void set_error(const char* msg);

inline pb_status fail(pb_status st, const char* fmt, ...) __attribute__((format(printf, 2, 3)));
inline pb_status fail(pb_status st, const char* fmt, ...) {
    char buf[1024];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    set_error(buf);
    return st;
}

}  // namespace pb

// Every extern "C" entry point that may allocate wraps its body so no C++
// exception crosses the ABI.
#define PB_TRY_BEGIN try {
#define PB_TRY_END                                                                  \
    }                                                                               \
    catch (const std::bad_alloc&) { return pb::fail(PB_ENOMEM, "host allocation failed"); } \
    catch (const std::exception& e) { return pb::fail(PB_EINVAL, "internal: %s", e.what()); } \
    catch (...) { return pb::fail(PB_EINVAL, "internal: unknown exception"); }
