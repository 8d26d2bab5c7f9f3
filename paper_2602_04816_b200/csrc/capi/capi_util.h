// Helpers shared by the C-ABI translation units.
#pragma once

#include <string>

namespace hlm_capi {
void set_error(const std::string& msg);
// ktimer.cpp: event pair around one launch (no-op unless hlm_ktimer_enable(1))
int ktimer_begin(void* stream);
void ktimer_end(int token, void* stream, int kind, double work);
}  // namespace hlm_capi
