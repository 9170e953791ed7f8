// runtime.hpp — process-wide libswg context for the C++ API layer.
#pragma once

#include "swg.h"
#include "swih/errors.hpp"

namespace swih::detail {

// Context of the device named by SWIH_GPU (default 0), created on first use.
swg_ctx* context();
// Throw the reference exception class for a non-OK status.
inline void check(swg_status st) {
  if (st != SWG_OK) raise(int(st));
}

}  // namespace swih::detail
