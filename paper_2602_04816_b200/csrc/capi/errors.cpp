// Thread-local last-error message behind hlm_cuda_last_error().
#include <string>

#include "hlm_cuda.h"
#include "capi_util.h"

namespace hlm_capi {
thread_local std::string g_last_error;
void set_error(const std::string& msg) { g_last_error = msg; }
}  // namespace hlm_capi

extern "C" const char* hlm_cuda_last_error(void) { return hlm_capi::g_last_error.c_str(); }
