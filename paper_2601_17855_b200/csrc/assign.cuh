// Batched policy operator (assign, policies.hpp:372-382): launch parameters.
#pragma once

#include <cstdint>

#include "bfsim_gpu.h"

namespace bfsim {

struct AssignParams {
  const bfsim_assign_call_t* calls;
  int32_t n_calls;
  int32_t n_max, h_max;  // largest waiting list / horizon over the calls
  int32_t ex_n;          // largest waiting list over the bfio-exact calls (lane scratch)
  const int64_t* previews;  // exact integer copies of the reference's doubles
  const int64_t* futures;
  const int32_t* caps;
  const int32_t* counts;
  int32_t* pairs;
  int64_t* n_pairs;
  double* cost;
  int32_t* status;
  unsigned char* ws;  // per call: ws_stride bytes
  int64_t ws_stride;
  int64_t i64_offset;                                   // F[32*(H+1)], wrow[H+1]
  int64_t lane_offset, lane_stride, lane_i64_offset;    // per-lane exact-search scratch
  int64_t limit;
};

int launch_assign(const AssignParams& p, void* stream);

}  // namespace bfsim
