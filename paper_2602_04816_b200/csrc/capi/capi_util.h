// Helpers shared by the C-ABI translation units.
#pragma once

#include <string>

namespace hlm_capi {
void set_error(const std::string& msg);
}  // namespace hlm_capi
