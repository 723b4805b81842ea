// errors.cpp — pb_last_error storage.
#include <cstring>

#include "errors.hpp"

namespace pb {
static thread_local char g_last_error[1024] = "";
void set_error(const char* msg) {
    strncpy(g_last_error, msg, sizeof g_last_error - 1);
    g_last_error[sizeof g_last_error - 1] = '\0';
}
}  // namespace pb

extern "C" const char* pb_last_error(void) { return pb::g_last_error; }
