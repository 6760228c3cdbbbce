// Shared host/device definitions for the B200 batched step engine.
#pragma once

#include <cstddef>
#include <cstdint>
#include <cstdio>
#include <cstring>

#include "bfsim_gpu.h"

// Largest prefill class the class structures support (3-level 64-ary bitmap).
#define BFSIM_MAX_CLASSES 262143

namespace bfsim {

inline int fail(char* err, size_t errlen, int code, const char* msg) {
  if (err && errlen) {
    std::snprintf(err, errlen, "%s", msg);
  }
  return code;
}

}  // namespace bfsim
