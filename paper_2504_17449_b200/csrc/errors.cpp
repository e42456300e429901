// SPDX-License-Identifier: Apache-2.0
// Thread-local last-error text for the C ABI (hmi_gpu_last_error).
#include <string>

#include "host_util.hpp"

namespace hmi_b200 {
namespace {
thread_local std::string g_last_error;
}
void set_last_error(const std::string& msg) { g_last_error = msg; }
const char* g_last_error_ptr() { return g_last_error.c_str(); }
}  // namespace hmi_b200

extern "C" const char* hmi_gpu_last_error(void) { return hmi_b200::g_last_error_ptr(); }
