// Launch plan shared by the host planner (capi.cu) and the step kernels (engine.cu).
#pragma once

#include <cstdint>

#include "bfsim_gpu.h"

namespace bfsim {

constexpr int kWarpsPerCta = 1;  // one warp (trajectory) per CTA: the planner always launches wpc = 1
constexpr uint32_t kEmpty = 0xFFFFFFFFu;

// Per-launch-group plan: every scenario in the group fits these maxima. Every
// o_* is an array placement code: >= 0 is a byte offset into the warp's
// shared-memory arena; < 0 encodes byte (-code - 1) of the warp's slice of the
// global workspace (ws_stride bytes per warp slot).
struct Plan {
  int G, B, H, S;  // maxima over the group: workers, batch, horizon, prefill classes
  int R;           // clock ring entries (power of two > max decode)
  int umax;        // max admissions in one step (G*B)
  int smem_per_warp;
  int all_smem;  // every array placed in shared memory (32-bit addressing variant)
  int64_t ws_stride;
  // slots
  int64_t o_f, o_a, o_x, o_id, o_stk, o_capb, o_asum, o_cap;
  // per-step accounting ring (32 steps) and clock ring
  int64_t o_rl, o_rdt, o_rcs, o_rmx, o_rac, o_ring;
  // FCFS/JSQ level tables
  int64_t o_lvT, o_lvV, o_lvK, o_lvM;
  // class structures: int4 records {front, back, picks, base} + int32 chain start, S+2 each; 2 bitmaps;
  // o_deq (per-class waiting deques) is always in the global workspace
  int64_t o_cls, o_bm, o_pbm, o_deq;
  // picks / chain results / prefetch stage (int2 per admission)
  int64_t o_stage, o_pcl, o_pt, o_res;
  // lookahead window (H > 0)
  int64_t o_F, o_M, o_Wc, o_Wa, o_oc, o_oo, o_oid;
  // TPOT completion buffer (cbuf entries) + misc counters
  int64_t o_cbuf, o_misc;
  // noisy lookahead: mt19937_64 state, draw -> worker prefix, per-item draws
  // (hot); per-worker active lists of {finish step, a} (o_lst) and the ids of
  // appended entries (o_eid), the admitted waiting draws, admitted-id bitmap
  // and its word prefix (cold)
  int64_t o_mt, o_lst, o_onz, o_nzb, o_abits, o_zpre, o_selb, o_eid, o_pre;
  int64_t o_nring;  // noisy: the producer warp's ring of draws (kRing int32)
  int64_t o_admc;   // per-worker admissions of the step (int32 chain)
  // bfio-greedy with WPL >= 16: per-worker argmin keys
  int64_t o_key;
  // completion calendar (cal != 0, large G*B): list heads [R][32], per-slot links
  int64_t o_calh, o_calnx;
  int cal, reserved3;
  int cbuf, noisy;
};

struct KParams {
  const bfsim_scenario_t* scen;
  const int32_t* order;
  int32_t n;
  const bfsim_input_t* inputs;
  const int32_t* class_base;
  const bfsim_request_t* traces;
  const bfsim_sample_t* streams;
  bfsim_step_sink_t steps;  // device pointers, NULL when absent
  bfsim_req_sink_t reqs;
  bfsim_req_sink_t reqs_host;  // optional page-locked mirror, filled per trajectory at its end
  bfsim_result_t* results;
  unsigned char* ws;
  int32_t* queue;
  Plan plan;
};

// Launch one group (grid CTAs of wpc warps) or, when occupancy != NULL, only
// query CTAs per SM. Returns cudaError_t as int.
int launch_step_kernel(int mode, int policy, int wpl, int small_classes, int noisy, int hr,
                       const KParams& kp, int grid, int wpc, void* stream, int* occupancy);

}  // namespace bfsim
