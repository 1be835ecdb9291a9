#include <string>

#include "capi_util.hpp"

namespace iolmh {
namespace {
thread_local std::string g_last_error;
}
void set_last_error(const std::string& msg) { g_last_error = msg; }
}  // namespace iolmh

extern "C" const char* iolm_cuda_last_error(void) { return iolmh::g_last_error.c_str(); }
