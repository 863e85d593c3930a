// fluxattn/b200.hpp -- device control for the C++ drop-in (not in the
// reference): which GPU the reference-API calls run on and the per-thread
// C-ABI context they use.  Defaults: device from FLUXATTN_DEVICE (else 0), one
// fx_ctx per host thread (the reference's executed mode calls execute_task from
// many threads; each gets its own stream).
#pragma once

#include <stdexcept>
#include <string>

#include "fluxattn_b200.h"

namespace fluxattn::b200 {

// The calling thread's context (created on first use).
fx_ctx* context();
void set_device(int device);

// C-ABI status -> std::runtime_error carrying the reference error code text.
inline void check(int status) {
    if (status != FX_OK) throw std::runtime_error(fx_last_error());
}

}  // namespace fluxattn::b200
