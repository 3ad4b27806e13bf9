// Library-internal exception carrying an nds_status; mapped to return codes at the C-ABI.
#pragma once

#include <stdexcept>
#include <string>

#include "ndsylv_b200.h"

namespace nds {

struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

}  // namespace nds
