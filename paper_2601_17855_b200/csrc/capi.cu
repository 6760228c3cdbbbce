// C ABI of the batched step engine (include/bfsim_gpu.h): context, scenario
// validation (mirroring the reference's exceptions), launch planning and the
// host <-> device plumbing. No exception crosses this boundary.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cstring>
#include <map>
#include <string>
#include <tuple>
#include <vector>

#include "bfsim_gpu.h"
#include "common.h"
#include "assign.cuh"
#include "engine.cuh"

using bfsim::fail;
using bfsim::KParams;
using bfsim::Plan;

namespace {

struct DevBuf {
  void* p = nullptr;
  size_t n = 0;
  cudaError_t ensure(size_t bytes) {
    if (bytes <= n) return cudaSuccess;
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
    size_t want = bytes + bytes / 4 + 256;
    cudaError_t e = cudaMalloc(&p, want);
    if (e == cudaSuccess) n = want;
    return e;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
};

constexpr int kMaxGroups = 16;  // side streams; kernel groups beyond this share them round-robin

}  // namespace

struct bfsim_ctx {
  int device = 0;
  int sm_count = 0;
  int smem_optin = 0;
  cudaStream_t side[kMaxGroups] = {};
  cudaEvent_t fork = nullptr, join[kMaxGroups] = {}, t0 = nullptr, t1 = nullptr;
  // device buffers for the host-pointer entry
  DevBuf scen, inputs, cbase, traces, streams, results, st_cs, st_dt, st_mx, st_ac, st_ld, rq_as,
      rq_ss, rq_wk, rq_ac, rq_fc;
  // planner-owned buffers
  DevBuf order, ws, queue;
  // batched assign()
  DevBuf a_calls, a_pv, a_fut, a_caps, a_cnt, a_pairs, a_np, a_cost, a_st, a_ws;
  // dyadic-drift inputs: prefill-scaled copies of traces / streams / class_base
  DevBuf dy_tr, dy_sm, dy_cb;
  int64_t last_launches = 0;
  bool timed = false;

};

namespace {

int cuda_fail(char* err, size_t errlen, cudaError_t e, const char* what) {
  std::string m = std::string(what) + ": " + cudaGetErrorString(e);
  return fail(err, errlen, BFSIM_ECUDA, m.c_str());
}

bool is_int_drift(double v) { return v >= 0.0 && v == std::floor(v) && v < 1e9; }

// Dyadic constant drift d = m / 2^e (SURVEY hard part 2). The reference
// accumulates the profile sequentially in fp64 (drift_profile,
// workload.hpp:73-85); with a dyadic d every partial sum s + j*d is exact, so
// the run equals the integer problem with every workload scaled by 2^e
// (prefill s*2^e, drift m): loads, maxima and the policies' sums scale
// exactly, every comparison and tie is unchanged, t_ell*2^-e times the scaled
// maximum is the reference's dt bit for bit, and the kernel scales the loads
// back on the way out (engine_impl.cuh, lsc).
constexpr int kMaxDriftShift = 16;
constexpr int kMaxScaledClasses = 262143;  // ClassSet<false>: 3-level 64-ary bitmap
bool dyadic_drift(double v, int64_t* m, int* e) {
  if (!(v >= 0.0) || !std::isfinite(v)) return false;
  for (int k = 0; k <= kMaxDriftShift; ++k) {
    const double x = std::ldexp(v, k);
    if (x == std::floor(x)) {
      if (x >= 1e9) return false;
      *m = static_cast<int64_t>(x);
      *e = k;
      return true;
    }
  }
  return false;
}

template <class R>
__global__ void scale_prefill_kernel(const R* __restrict__ src, R* __restrict__ dst, int64_t n, int e) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    R r = src[i];
    r.prefill <<= e;
    dst[i] = r;
  }
}

// class_base of the scaled input: #records with s*2^e < c = #records with s < ceil(c / 2^e)
__global__ void scale_class_base_kernel(const int32_t* __restrict__ src, int32_t* __restrict__ dst, int64_t n,
                                        int e) {
  for (int64_t c = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; c < n;
       c += static_cast<int64_t>(gridDim.x) * blockDim.x)
    dst[c] = src[(c + (int64_t{1} << e) - 1) >> e];
}

// SimConfig::validate (engine.hpp:31-36), PowerModel::validate
// (metrics_power.hpp:17-21), DriftSpec::validate (workload.hpp:52-60), plus the
// GPU path's own limits. Returns a BFSIM_* code.
int validate_scenario(const bfsim_scenario_t& s, const bfsim_input_t* inputs, int32_t n_inputs,
                      const std::vector<int>* single_class_inputs, char* err, size_t errlen) {
  if (s.workers < 1 || s.batch < 1)
    return fail(err, errlen, BFSIM_EINVAL, "config: workers and batch must be >= 1");
  if (s.overhead < 0.0 || s.per_token <= 0.0)
    return fail(err, errlen, BFSIM_EINVAL, "config: bad time constants");
  if (s.horizon < 0 || (s.mode == BFSIM_MODE_POISSON && s.max_steps < 1))
    return fail(err, errlen, BFSIM_EINVAL, "config: bad horizon or max_steps");
  if (!(s.p_idle > 0.0 && s.p_idle < s.p_max))
    return fail(err, errlen, BFSIM_EINVAL, "power: need 0 < p_idle < p_max");
  if (!(s.mfu_sat > 0.0 && s.mfu_sat <= 1.0))
    return fail(err, errlen, BFSIM_EINVAL, "power: mfu_sat out of (0,1]");
  if (!(s.gamma > 0.0 && s.gamma < 1.0))
    return fail(err, errlen, BFSIM_EINVAL, "power: gamma out of (0,1)");
  if (s.drift < 0.0) return fail(err, errlen, BFSIM_EINVAL, "drift: increment out of [0, delta_max]");
  int64_t d = 0;
  int dshift = 0;
  if (!dyadic_drift(s.drift, &d, &dshift))
    return fail(err, errlen, BFSIM_EINVAL,
                "drift: the GPU path is bit-exact only for integer or dyadic (m / 2^e, e <= 16) constant drift "
                "(SURVEY F5)");
  if (s.policy == BFSIM_POLICY_BFIO_EXACT)
    return fail(err, errlen, BFSIM_EINVAL,
                "bfio-exact is an exponential search; it runs on the CPU reference only");
  if (s.policy != BFSIM_POLICY_FCFS && s.policy != BFSIM_POLICY_JSQ &&
      s.policy != BFSIM_POLICY_BFIO_GREEDY)
    return fail(err, errlen, BFSIM_EINVAL, "unknown policy");
  if (s.mode != BFSIM_MODE_POISSON && s.mode != BFSIM_MODE_OVERLOADED)
    return fail(err, errlen, BFSIM_EINVAL, "unknown mode");
  if (s.lookahead < 0 || s.lookahead > 2) return fail(err, errlen, BFSIM_EINVAL, "unknown lookahead");
  // sigma <= 0 (or NaN) previews perfectly, as make_preview does (policies.hpp:74);
  // an infinite sigma has no lround (the reference's result is undefined)
  if (s.lookahead == BFSIM_LOOKAHEAD_NOISY && std::isinf(s.noise_sigma))
    return fail(err, errlen, BFSIM_EINVAL, "noisy lookahead: infinite noise_sigma");
  if (s.input_id < 0 || s.input_id >= n_inputs)
    return fail(err, errlen, BFSIM_EINVAL, "scenario: input_id out of range");
  if (s.workers > 1024) return fail(err, errlen, BFSIM_EINVAL, "GPU path: workers > 1024 not supported");
  if (s.batch > 65535) return fail(err, errlen, BFSIM_EINVAL, "GPU path: batch > 65535");
  if (static_cast<int64_t>(s.workers) * s.batch > (1 << 24))
    return fail(err, errlen, BFSIM_EINVAL, "GPU path: workers*batch too large");
  if (s.mode == BFSIM_MODE_OVERLOADED) {
    if (s.steps < 0 || s.warmup < 0)
      return fail(err, errlen, BFSIM_EINVAL, "run_overloaded: negative steps or warmup");
    if (!(s.backlog >= 0.0)) return fail(err, errlen, BFSIM_EINVAL, "run_overloaded: bad backlog");
    if (single_class_inputs && (*single_class_inputs)[s.input_id])
      return fail(err, errlen, BFSIM_EINVAL,
                  "run_overloaded: single-class prefill never satisfies Def. 1 (reference loops "
                  "forever, SURVEY F12)");
    if (s.warmup + s.steps > INT32_MAX - 2)
      return fail(err, errlen, BFSIM_EINVAL, "run_overloaded: too many steps");
  }
  if (s.horizon > 4096) return fail(err, errlen, BFSIM_EINVAL, "GPU path: horizon > 4096");
  // bounds on the (dyadic-scaled) integer problem
  bfsim_input_t in = inputs[s.input_id];
  in.s_max = static_cast<int32_t>(std::min<int64_t>(static_cast<int64_t>(in.s_max) << dshift, INT32_MAX));
  const double lb = static_cast<double>(s.batch) *
                    (static_cast<double>(in.s_max) + static_cast<double>(d) * (in.max_decode - 1));
  if (lb >= 2147483647.0)
    return fail(err, errlen, BFSIM_EINVAL, "GPU path: per-worker load bound exceeds 2^31");
  if (in.max_decode >= (1 << 30)) return fail(err, errlen, BFSIM_EINVAL, "GPU path: decode too long");
  // noisy draws are carried clamped to +-2^29, exact while decode lengths stay below 2^28
  if (s.lookahead == BFSIM_LOOKAHEAD_NOISY && s.noise_sigma > 0.0 && in.max_decode >= (1 << 28))
    return fail(err, errlen, BFSIM_EINVAL, "GPU path: decode too long for noisy lookahead");
  // per-slot a = s - drift*x is int32 (Poisson runs check this per step: BFSIM_ERANGE)
  if (s.mode == BFSIM_MODE_OVERLOADED &&
      static_cast<double>(d) * static_cast<double>(s.warmup + s.steps) + in.s_max >= 2147483647.0)
    return fail(err, errlen, BFSIM_EINVAL, "GPU path: drift * (warmup + steps) exceeds 2^31");
  return BFSIM_OK;
}

// Noisy lookahead changes decisions only for bfio-greedy with a window
// (H > 0) in the Poisson loop: FCFS/JSQ never read previews, entry h = 0 is
// always exact, and run_overloaded always previews perfectly (oracle.hpp:185-199).
// Elsewhere the draws the reference takes are unobservable.
int noisy_variant(const bfsim_scenario_t& s) {
  return s.lookahead == BFSIM_LOOKAHEAD_NOISY && s.noise_sigma > 0.0 &&
                 s.policy == BFSIM_POLICY_BFIO_GREEDY && s.mode == BFSIM_MODE_POISSON &&
                 s.horizon > 0
             ? 1
             : 0;
}

int bits_for(int64_t x) {  // bits to hold values 0..x (the kernel's bits_for)
  int b = 0;
  while (b < 63 && (x >> b) > 0) ++b;
  return b;
}

// Width of the register-resident lookahead chain (engine_impl.cuh, HR):
// bfio-greedy with 0 < H < 24 on G <= 128 workers whose per-worker loads fit
// 31 bits with the worker index and whose horizon costs fit 31 bits.
int reg_chain_width(const bfsim_scenario_t& s, const bfsim_input_t& in) {
  if (s.policy != BFSIM_POLICY_BFIO_GREEDY || s.horizon <= 0 || s.horizon >= 24 || s.workers > 128)
    return 0;
  const int64_t d = static_cast<int64_t>(s.drift);
  const int64_t lbound = static_cast<int64_t>(s.batch) * (in.s_max + d * (in.max_decode - 1));
  const int gbits = std::max(1, bits_for(s.workers - 1));
  if (bits_for(lbound) + gbits > 31) return 0;
  if ((static_cast<int64_t>(s.horizon) + 1) * lbound >= (int64_t{1} << 31)) return 0;
  return s.horizon < 8 ? 8 : 24;
}

// Placement-chain kind of a scenario: the int32 register-budget chain (8, 24:
// H < chain, G <= 128), the wide CTA (1: bfio-greedy with a window on
// G > 128, not noisy; ceil(G / 128) warps share the chain) or the
// single-warp shared-memory chain (0).
int chain_kind(const bfsim_scenario_t& s, const bfsim_input_t& in, int noisy) {
  const int hr = reg_chain_width(s, in);
  if (hr) return hr;
  if (s.policy == BFSIM_POLICY_BFIO_GREEDY && s.horizon > 0 && !noisy && s.workers > 128) return 1;
  return 0;
}

// int32 chain views (engine_impl.cuh, HP): G worker rows of H + 1 int32
// words rounded up to 4 (128-bit row loads)
int64_t chain_rows_bytes(int H, int G) { return static_cast<int64_t>(G) * ((H + 4) & ~3) * 4; }

int wpl_for(int G) {
  int w = (G + 31) / 32;
  int p = 1;
  while (p < w) p <<= 1;
  return p;
}

struct Group {
  int mode, policy, wpl, small, noisy, hr;
  int64_t hot_bytes = 0;
  std::vector<int32_t> idx;
  Plan plan;
  int wpc = 4, grid = 0;
};

// Lay out every per-warp array; put the hot ones in shared memory until the
// budget is spent, the rest in the warp's global workspace.
void make_plan(Group& g, const bfsim_scenario_t* scen, const bfsim_input_t* inputs, int smem_budget) {
  Plan& p = g.plan;
  std::memset(&p, 0, sizeof(p));
  int G = 1, B = 1, H = 0, S = 1, max_o = 1;
  int64_t max_len = 0;
  for (int32_t i : g.idx) {
    const auto& s = scen[i];
    const auto& in = inputs[s.input_id];
    G = std::max(G, s.workers);
    B = std::max(B, s.batch);
    if (s.policy == BFSIM_POLICY_BFIO_GREEDY) H = std::max(H, s.horizon);
    S = std::max(S, in.s_max);
    max_o = std::max(max_o, in.max_decode);
    max_len = std::max<int64_t>(max_len, in.length);
  }
  int R = 1;
  // admit clocks stay readable until the 32-step TPOT drain; calendar
  // buckets k .. k + max(max_o, H) never alias
  while (R <= max_o + 33 + H) R <<= 1;
  p.G = G;
  p.B = B;
  p.H = H;
  p.S = S;
  p.R = R;
  p.umax = G * B;
  const int wpl = g.wpl;
  const bool greedy = g.policy == BFSIM_POLICY_BFIO_GREEDY;
  const bool ovl = g.mode == BFSIM_MODE_OVERLOADED;
  const int64_t GB = static_cast<int64_t>(G) * B;
  const int rstride = (G & 1) ? G : G + 1;
  const int64_t lvl = static_cast<int64_t>(B) + 2;
  const int64_t bm_words = 64 + (S + 63) / 64 + 1;

  struct Item {
    int64_t* code;
    int64_t bytes;
    bool core;  // always in shared memory: the kernel addresses it with 32-bit shared loads
  };
  // completion calendar: a 64-bucket wheel in shared memory for small G*B,
  // exact finish-step buckets in the workspace once the slots outgrow it
  p.cal = GB > 4096 ? 1 : 2;
  p.noisy = g.noisy;
  p.cbuf = static_cast<int>(std::min<int64_t>(GB + 512, 1 << 24));
  // Hot and small first (first fit: an array that does not fit spills to
  // the warp's global workspace and later, smaller ones may still fit):
  // per-step scalars and per-worker state, class records, argmin keys, the
  // accounting ring, then the per-slot arrays, then per-admission scratch.
  // Core arrays (touched on every step's dependent chain, small) are always
  // in shared memory -- the kernel addresses them with 32-bit shared loads
  // even in its spilled variant (engine_impl.cuh: at<true>) -- then the rest.
  std::vector<Item> items = {
      {&p.o_rdt, 32 * 8, true}, {&p.o_rcs, 32 * 8, true}, {&p.o_rmx, 32 * 4, true}, {&p.o_rac, 32 * 4, true},
      {&p.o_misc, 16, true},    {&p.o_capb, G * 4LL, true}, {&p.o_asum, G * 8LL, true}, {&p.o_cap, G * 4LL, true},
  };
  if (!greedy) {  // level tables of the FIFO policies
    items.push_back({&p.o_lvT, lvl * 4, true});
    items.push_back({&p.o_lvV, lvl * 4, true});
    items.push_back({&p.o_lvK, lvl * 4, true});
    items.push_back({&p.o_lvM, lvl * wpl * 4, true});
  }
  if (greedy || ovl) {
    const bool c = greedy && g.small;  // <= 64 classes (SMALLC)
    items.push_back({&p.o_cls, 5LL * (S + 2) * 4, c});  // int4 records + int32 starts
    items.push_back({&p.o_bm, bm_words * 8, c});
    items.push_back({&p.o_pbm, bm_words * 8, c});
  }
  if (greedy && wpl >= 16) items.push_back({&p.o_key, static_cast<int64_t>(wpl) * 32 * 8, false});
  // M, T, w of the lookahead chain
  // (the int32 chain keeps only its T row there: H + 1 int32 rounded up to 4)
  if (greedy && H > 0)
    items.push_back({&p.o_M, g.hr >= 8 ? ((H + 4) & ~3) * 4LL : std::max<int64_t>(3 * (H + 1) * 8LL, 128), true});
  if (g.noisy) {
    // the draw ring, the draw pass's shared-memory atomics (int32 difference
    // arrays over h) and the int32 chain's [h][g] views
    items.push_back({&p.o_mt, 312 * 8, true});
    items.push_back({&p.o_nring, 2048 * 4, true});  // kRing draws
    items.push_back({&p.o_pre, (G + 1) * 4LL, true});
    items.push_back({&p.o_Wc, static_cast<int64_t>(H) * G * 4, true});
    items.push_back({&p.o_Wa, static_cast<int64_t>(H) * G * 4, true});
    if (g.hr) items.push_back({&p.o_F, chain_rows_bytes(H, G), true});
  }
  // int32 views (register-budget and wide chains)
  if (greedy && H > 0 && !g.noisy && g.hr) {
    if (g.hr == 1) items.push_back({&p.o_F, (H + 1) * 4LL * G, true});  // wide chain: [h][g]
    else items.push_back({&p.o_F, chain_rows_bytes(H, G), true});
  }
  if (greedy && H > 0 && g.hr) items.push_back({&p.o_admc, G * 4LL, true});
  // per-slot state touched every step (retire)
  items.push_back({&p.o_f, ((GB + 3) & ~3LL) * 4});
  items.push_back({&p.o_a, GB * 4});
  items.push_back({&p.o_stk, GB * 2});
  if (greedy && H > 0 && !g.noisy) {
    if (!g.hr) items.push_back({&p.o_F, (H + 1) * 8LL * G});
    items.push_back({&p.o_Wc, static_cast<int64_t>(H) * G * 4});
    items.push_back({&p.o_Wa, static_cast<int64_t>(H) * G * 8});
  }
  if (greedy && H > 0 && g.noisy && !g.hr) items.push_back({&p.o_F, (H + 1) * 8LL * G});
  if (p.cal == 2) {  // the 64-bucket completion wheel lives in shared memory
    items.push_back({&p.o_calh, 64LL * std::min(G, 32) * 4});
    items.push_back({&p.o_calnx, GB * 2});
  }
  const size_t n_hot = items.size();  // the residency planner tries to keep these in shared memory
  items.push_back({&p.o_id, GB * 4});
  items.push_back({&p.o_x, GB * 4});
  items.push_back({&p.o_rl, 32LL * rstride * 4});
  // per-admission scratch (sized for the worst step, touched U times a step)
  items.push_back({&p.o_stage, GB * 8});
  if (g.noisy) items.push_back({&p.o_onz, GB * 4});
  if (greedy) {
    items.push_back({&p.o_res, GB * 4});
    items.push_back({&p.o_pcl, GB * 4});
    items.push_back({&p.o_pt, GB * 4});
    items.push_back({&p.o_oc, GB * 4});
    if (H > 0) {
      items.push_back({&p.o_oo, GB * 4});
      items.push_back({&p.o_oid, GB * 4});
    }
  }
  int64_t hot = 0;
  for (size_t i = 0; i < n_hot; ++i) hot += (items[i].bytes + 15) & ~15LL;
  g.hot_bytes = hot;
  int64_t sm_off = 0, ws_off = 0;
  int spilled = 0;
  for (auto& it : items)
    if (it.core) {
      *it.code = sm_off;
      sm_off += (it.bytes + 15) & ~15LL;
    }
  for (auto& it : items) {
    if (it.core) continue;
    int64_t b = (it.bytes + 15) & ~15LL;
    if (sm_off + b <= smem_budget) {
      *it.code = sm_off;
      sm_off += b;
    } else {
      *it.code = -(ws_off + 1);
      ws_off += b;
      spilled = 1;
    }
  }
  p.all_smem = spilled ? 0 : 1;
  // cold arrays: always in the global workspace (touched once per step or per
  // completion, off the dependent chain): clock ring, TPOT completion buffer,
  // per-class waiting deques (counting-sort layout over the input)
  auto cold = [&](int64_t* code, int64_t bytes) {
    *code = -(ws_off + 1);
    ws_off += (bytes + 15) & ~15LL;
  };
  cold(&p.o_ring, R * 8LL);
  cold(&p.o_cbuf, static_cast<int64_t>(p.cbuf) * 8);
  if (p.cal == 1) {
    cold(&p.o_calh, static_cast<int64_t>(R) * 32 * 4);
    cold(&p.o_calnx, GB * 4);
  }
  if (greedy) cold(&p.o_deq, max_len * 8);
  else p.o_deq = -1;
  if (g.noisy) {
    const int64_t words = (max_len + 63) / 64 + 2;
    cold(&p.o_lst, GB * 8);
    cold(&p.o_eid, GB * 4);
    cold(&p.o_nzb, (GB + max_len) * 4);
    cold(&p.o_abits, words * 8);
    cold(&p.o_zpre, words * 4);
    cold(&p.o_selb, ((max_len + 31) / 32 + 2) * 4);
  }
  p.smem_per_warp = static_cast<int>((sm_off + 15) & ~15LL);
  if (p.smem_per_warp == 0) p.smem_per_warp = 16;
  p.ws_stride = std::max<int64_t>(16, (ws_off + 255) & ~255LL);
}

int64_t est_work(const bfsim_scenario_t& s, const bfsim_input_t& in) {
  if (s.mode == BFSIM_MODE_OVERLOADED) return (s.steps + s.warmup) * s.workers;
  return in.length * 64 + 1;
}

}  // namespace

extern "C" {

int bfsim_ctx_create(int device, bfsim_ctx_t** out, char* err, size_t errlen) {
  *out = nullptr;
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || n == 0)
    return fail(err, errlen, BFSIM_ECUDA, "no CUDA device: the GPU path has no CPU fallback");
  if (device < 0 || device >= n) return fail(err, errlen, BFSIM_EINVAL, "device out of range");
  e = cudaSetDevice(device);
  if (e != cudaSuccess) return cuda_fail(err, errlen, e, "cudaSetDevice");
  cudaDeviceProp prop;
  cudaGetDeviceProperties(&prop, device);
  if (prop.major < 10)
    return fail(err, errlen, BFSIM_ECUDA, "the step engine is built for sm_100a (B200)");
  auto* c = new bfsim_ctx;
  c->device = device;
  c->sm_count = prop.multiProcessorCount;
  c->smem_optin = static_cast<int>(prop.sharedMemPerBlockOptin);
  for (int i = 0; i < kMaxGroups; ++i) {
    cudaStreamCreateWithFlags(&c->side[i], cudaStreamNonBlocking);
    cudaEventCreateWithFlags(&c->join[i], cudaEventDisableTiming);
  }
  cudaEventCreateWithFlags(&c->fork, cudaEventDisableTiming);
  cudaEventCreate(&c->t0);
  cudaEventCreate(&c->t1);
  *out = c;
  return BFSIM_OK;
}

void bfsim_ctx_destroy(bfsim_ctx_t* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  cudaDeviceSynchronize();
  DevBuf* bufs[] = {&c->scen,    &c->inputs, &c->cbase,  &c->traces, &c->streams, &c->results,
                    &c->st_cs,   &c->st_dt,  &c->st_mx,  &c->st_ac,  &c->st_ld,   &c->rq_as,
                    &c->rq_ss,   &c->rq_wk,  &c->rq_ac,  &c->rq_fc,  &c->order,   &c->ws,
                    &c->queue,   &c->a_calls, &c->a_pv,  &c->a_fut,  &c->a_caps,  &c->a_cnt,
                    &c->a_pairs, &c->a_np,   &c->a_cost, &c->a_st,   &c->a_ws,
                    &c->dy_tr,   &c->dy_sm,  &c->dy_cb};
  for (auto* b : bufs) b->release();
  for (int i = 0; i < kMaxGroups; ++i) {
    cudaStreamDestroy(c->side[i]);
    cudaEventDestroy(c->join[i]);
  }
  cudaEventDestroy(c->fork);
  cudaEventDestroy(c->t0);
  cudaEventDestroy(c->t1);
  delete c;
}

int bfsim_ctx_device(const bfsim_ctx_t* c) { return c ? c->device : -1; }

int64_t bfsim_last_launch_count(const bfsim_ctx_t* c) { return c ? c->last_launches : 0; }

double bfsim_last_step_kernel_ms(const bfsim_ctx_t* c) {
  if (!c || !c->timed) return 0.0;
  float ms = 0.f;
  if (cudaEventSynchronize(c->t1) != cudaSuccess) return 0.0;
  if (cudaEventElapsedTime(&ms, c->t0, c->t1) != cudaSuccess) return 0.0;
  return static_cast<double>(ms);
}

}  // extern "C"

namespace {
// reqs_host: device-mapped page-locked mirror of the request sink; each
// trajectory's warp copies its finished slice there (coalesced) as it ends.
int run_batch_device_impl(bfsim_ctx_t* ctx, const bfsim_scenario_t* scen_host, int64_t n_scen,
                          const bfsim_input_t* inputs_host, int32_t n_inputs,
                          const int32_t* class_base_dev, const bfsim_request_t* traces_dev,
                          const bfsim_sample_t* streams_dev, const bfsim_step_sink_t* steps_dev,
                          const bfsim_req_sink_t* reqs_dev, const bfsim_req_sink_t* reqs_host,
                          bfsim_result_t* results_dev, void* stream, char* err, size_t errlen) {
  if (!ctx) return fail(err, errlen, BFSIM_EINVAL, "null context");
  ctx->last_launches = 0;
  ctx->timed = false;
  if (n_scen <= 0) return BFSIM_OK;
  if (n_scen > INT32_MAX) return fail(err, errlen, BFSIM_EINVAL, "too many scenarios");
  cudaSetDevice(ctx->device);
  // scenarios must refer to device-resident scenario rows for the kernel: copy
  cudaStream_t us = static_cast<cudaStream_t>(stream);
  // dyadic drift: such scenarios run on prefill-scaled copies of their inputs
  // (dyadic_drift above); the kernel reads the shift from reserved0
  std::vector<bfsim_scenario_t> scen2(scen_host, scen_host + n_scen);
  std::vector<bfsim_input_t> inputs2(inputs_host, inputs_host + n_inputs);
  struct DyJob {
    int32_t src, dst;
    int e, mode;
  };
  std::vector<DyJob> dy;
  {
    std::map<std::tuple<int32_t, int, int>, int32_t> ids;
    for (auto& s : scen2) {
      s.reserved0 = 0;
      int64_t m = 0;
      int e = 0;
      if (is_int_drift(s.drift) || !dyadic_drift(s.drift, &m, &e) || s.input_id < 0 || s.input_id >= n_inputs)
        continue;  // integer drift, or validate_scenario reports it
      const auto key = std::make_tuple(s.input_id, e, s.mode);
      auto it = ids.find(key);
      if (it == ids.end()) {
        bfsim_input_t in = inputs_host[s.input_id];
        if ((static_cast<int64_t>(in.s_max) << e) > kMaxScaledClasses)
          return fail(err, errlen, BFSIM_EINVAL, "drift: dyadic drift needs s_max * 2^e <= 262143 on the GPU path");
        in.s_max <<= e;
        const int32_t id = static_cast<int32_t>(inputs2.size());
        inputs2.push_back(in);
        dy.push_back({s.input_id, id, e, s.mode});
        it = ids.emplace(key, id).first;
      }
      s.drift = static_cast<double>(m);
      s.per_token = std::ldexp(s.per_token, -e);
      s.reserved0 = e;
      s.input_id = it->second;
    }
  }
  scen_host = scen2.data();
  inputs_host = inputs2.data();
  n_inputs = static_cast<int32_t>(inputs2.size());
  for (int64_t i = 0; i < n_scen; ++i) {
    int rc = validate_scenario(scen_host[i], inputs_host, n_inputs, nullptr, err, errlen);
    if (rc) {
      std::string m = "scenario " + std::to_string(i) + ": " + (err ? std::string(err) : "");
      return fail(err, errlen, rc, m.c_str());
    }
    const auto& in = inputs_host[scen_host[i].input_id];
    if (scen_host[i].mode == BFSIM_MODE_POISSON && !traces_dev && in.length > 0)
      return fail(err, errlen, BFSIM_EINVAL, "poisson scenario without traces");
    if (scen_host[i].mode == BFSIM_MODE_OVERLOADED && !streams_dev)
      return fail(err, errlen, BFSIM_EINVAL, "overloaded scenario without sample streams");
  }
  int64_t dy_launches = 0;
  if (!dy.empty()) {
    int64_t n_tr = 0, n_sm = 0, n_cb = 0;
    for (const auto& j : dy) {
      (j.mode == BFSIM_MODE_POISSON ? n_tr : n_sm) += inputs2[j.src].length;
      n_cb += inputs2[j.dst].s_max + 2;
    }
    cudaError_t e;
    if ((e = ctx->dy_tr.ensure(std::max<int64_t>(n_tr, 1) * sizeof(bfsim_request_t))) != cudaSuccess ||
        (e = ctx->dy_sm.ensure(std::max<int64_t>(n_sm, 1) * sizeof(bfsim_sample_t))) != cudaSuccess ||
        (e = ctx->dy_cb.ensure(n_cb * 4)) != cudaSuccess)
      return cuda_fail(err, errlen, e, "dyadic-drift input alloc");
    // the scaled copies are addressed from the caller's pool bases (offsets
    // across allocations in the flat device address space)
    auto rel = [](const void* p, const void* base, size_t rec, int64_t* off) {
      const intptr_t d = reinterpret_cast<intptr_t>(p) - reinterpret_cast<intptr_t>(base);
      if (d % static_cast<intptr_t>(rec)) return false;
      *off = static_cast<int64_t>(d / static_cast<intptr_t>(rec));
      return true;
    };
    int64_t o_tr = 0, o_sm = 0, o_cb = 0;
    for (const auto& j : dy) {
      const bfsim_input_t& src = inputs2[j.src];
      bfsim_input_t& dst = inputs2[j.dst];
      const int blocks = static_cast<int>(std::min<int64_t>(4 * ctx->sm_count, (src.length + 255) / 256 + 1));
      bool ok;
      if (j.mode == BFSIM_MODE_POISSON) {
        auto* out = static_cast<bfsim_request_t*>(ctx->dy_tr.p) + o_tr;
        ok = rel(out, traces_dev, sizeof(bfsim_request_t), &dst.offset);
        if (ok && src.length > 0) {
          scale_prefill_kernel<<<blocks, 256, 0, us>>>(traces_dev + src.offset, out, src.length, j.e);
          ++dy_launches;
        }
        o_tr += src.length;
      } else {
        auto* out = static_cast<bfsim_sample_t*>(ctx->dy_sm.p) + o_sm;
        ok = rel(out, streams_dev, sizeof(bfsim_sample_t), &dst.offset);
        if (ok && src.length > 0) {
          scale_prefill_kernel<<<blocks, 256, 0, us>>>(streams_dev + src.offset, out, src.length, j.e);
          ++dy_launches;
        }
        o_sm += src.length;
      }
      int32_t* cb = static_cast<int32_t*>(ctx->dy_cb.p) + o_cb;
      ok = ok && rel(cb, class_base_dev, 4, &dst.class_base_offset);
      if (!ok) return fail(err, errlen, BFSIM_ECUDA, "dyadic drift: misaligned input pool");
      scale_class_base_kernel<<<static_cast<int>((dst.s_max + 2 + 255) / 256), 256, 0, us>>>(
          class_base_dev + src.class_base_offset, cb, dst.s_max + 2, j.e);
      ++dy_launches;
      o_cb += dst.s_max + 2;
    }
    if ((e = cudaGetLastError()) != cudaSuccess) return cuda_fail(err, errlen, e, "dyadic-drift input scaling");
  }
  // group by kernel variant; LPT order inside a group
  std::map<std::tuple<int, int, int, int, int, int>, Group> groups;
  for (int64_t i = 0; i < n_scen; ++i) {
    const auto& s = scen_host[i];
    const auto& in = inputs_host[s.input_id];
    int small = in.s_max <= 64 ? 1 : 0;
    int wpl = wpl_for(s.workers);
    int noisy = noisy_variant(s);
    int hr = chain_kind(s, in, noisy);
    auto key = std::make_tuple(s.mode, s.policy, wpl, small, noisy, hr);
    auto& g = groups[key];
    g.mode = s.mode;
    g.policy = s.policy;
    g.wpl = wpl;
    g.small = small;
    g.noisy = noisy;
    g.hr = hr;
    g.idx.push_back(static_cast<int32_t>(i));
  }
  std::vector<int32_t> order;
  std::vector<Group*> gl;
  int64_t ws_total = 0;
  for (auto& kv : groups) {
    Group& g = kv.second;
    std::stable_sort(g.idx.begin(), g.idx.end(), [&](int32_t a, int32_t b) {
      return est_work(scen_host[a], inputs_host[scen_host[a].input_id]) >
             est_work(scen_host[b], inputs_host[scen_host[b].input_id]);
    });
    // shared memory: up to 4 warps per CTA within the opt-in limit
    // shared-memory budget per trajectory: enough trajectories resident per SM
    // to hold every group of the batch at once (the groups run concurrently
    // and the warps are latency-bound); what does not fit spills to the
    // per-warp global workspace (generic-addressing kernel variant)
    // Residency: enough trajectories per SM for the whole batch (measured
    // better on C3 than capping residency to keep the hot arrays in shared
    // memory: more warps in flight beat fewer, faster ones).
    int64_t per_sm = (n_scen + ctx->sm_count - 1) / ctx->sm_count;
    per_sm = std::max<int64_t>(1, std::min<int64_t>(per_sm, 16));
    int budget = static_cast<int>(std::min<int64_t>(ctx->smem_optin - 1024,
                                                    (228 * 1024) / per_sm - 2048));
    budget = std::max(budget, 8 * 1024);
    make_plan(g, scen_host, inputs_host, budget);
    // one warp (trajectory) per CTA: latency-bound warps spread over every SM;
    // noisy: the trajectory's CTA has a second warp producing its draws;
    // wide: ceil(G / 128) warps share the placement chain
    g.wpc = g.noisy ? 2 : (g.hr == 1 ? std::max(1, g.wpl / 4) : 1);
    KParams probe{};
    probe.plan = g.plan;
    int occ = 0;
    int rc = bfsim::launch_step_kernel(g.mode, g.policy, g.wpl, g.small, g.noisy, g.hr, probe, 0, g.wpc,
                                       nullptr, &occ);
    if (rc != 0 || occ <= 0)
      return fail(err, errlen, BFSIM_ECUDA, "step kernel does not fit on the device");
    if (std::getenv("BFSIM_DEBUG_PLAN"))
      std::fprintf(stderr,
                   "bfsim plan: mode %d policy %d wpl %d noisy %d hr %d: %zu trajectories, %d B smem/trajectory "
                   "(all_smem %d), occupancy %d CTAs/SM of %d warps, ws %lld B/trajectory\n",
                   g.mode, g.policy, g.wpl, g.noisy, g.hr, g.idx.size(), g.plan.smem_per_warp, g.plan.all_smem, occ,
                   g.wpc, static_cast<long long>(g.plan.ws_stride));
    const int traj_per_cta = (g.noisy || g.hr == 1) ? 1 : g.wpc;
    int64_t ctas = (static_cast<int64_t>(g.idx.size()) + traj_per_cta - 1) / traj_per_cta;
    g.grid = static_cast<int>(std::min<int64_t>(ctas, static_cast<int64_t>(occ) * ctx->sm_count));
    ws_total += g.plan.ws_stride * g.grid * traj_per_cta;
    gl.push_back(&g);
  }
  for (auto* g : gl) order.insert(order.end(), g->idx.begin(), g->idx.end());
  cudaError_t e;
  if ((e = ctx->order.ensure(order.size() * 4)) != cudaSuccess) return cuda_fail(err, errlen, e, "alloc");
  if ((e = ctx->queue.ensure(std::max<size_t>(gl.size(), 1) * 4)) != cudaSuccess)
    return cuda_fail(err, errlen, e, "alloc");
  if ((e = ctx->ws.ensure(static_cast<size_t>(std::max<int64_t>(ws_total, 256)))) != cudaSuccess)
    return cuda_fail(err, errlen, e, "workspace alloc");
  // device copy of the scenario table (the host table is authoritative)
  if ((e = ctx->scen.ensure(n_scen * sizeof(bfsim_scenario_t))) != cudaSuccess)
    return cuda_fail(err, errlen, e, "alloc");
  if ((e = ctx->inputs.ensure(n_inputs * sizeof(bfsim_input_t))) != cudaSuccess)
    return cuda_fail(err, errlen, e, "alloc");
  cudaMemcpyAsync(ctx->scen.p, scen_host, n_scen * sizeof(bfsim_scenario_t), cudaMemcpyHostToDevice, us);
  cudaMemcpyAsync(ctx->inputs.p, inputs_host, n_inputs * sizeof(bfsim_input_t), cudaMemcpyHostToDevice, us);
  cudaMemcpyAsync(ctx->order.p, order.data(), order.size() * 4, cudaMemcpyHostToDevice, us);
  cudaMemsetAsync(ctx->queue.p, 0, std::max<size_t>(gl.size(), 1) * 4, us);
  int64_t launches = dy_launches;  // kernels only (not copies / memsets)
  cudaEventRecord(ctx->t0, us);
  cudaEventRecord(ctx->fork, us);
  int64_t off = 0, ws_off = 0;
  for (size_t gi = 0; gi < gl.size(); ++gi) {
    Group& g = *gl[gi];
    cudaStream_t s = gl.size() == 1 ? us : ctx->side[gi % kMaxGroups];
    if (gl.size() > 1) cudaStreamWaitEvent(s, ctx->fork, 0);
    KParams kp{};
    kp.scen = static_cast<const bfsim_scenario_t*>(ctx->scen.p);
    kp.order = static_cast<const int32_t*>(ctx->order.p) + off;
    kp.n = static_cast<int32_t>(g.idx.size());
    kp.inputs = static_cast<const bfsim_input_t*>(ctx->inputs.p);
    kp.class_base = class_base_dev;
    kp.traces = traces_dev;
    kp.streams = streams_dev;
    if (steps_dev) kp.steps = *steps_dev;
    if (reqs_dev) kp.reqs = *reqs_dev;
    if (reqs_dev && reqs_host) kp.reqs_host = *reqs_host;
    kp.results = results_dev;
    kp.ws = static_cast<unsigned char*>(ctx->ws.p) + ws_off;
    kp.queue = static_cast<int32_t*>(ctx->queue.p) + gi;
    kp.plan = g.plan;
    int rc = bfsim::launch_step_kernel(g.mode, g.policy, g.wpl, g.small, g.noisy, g.hr, kp, g.grid, g.wpc,
                                       s, nullptr);
    if (rc != 0) return cuda_fail(err, errlen, static_cast<cudaError_t>(rc), "step kernel launch");
    ++launches;
    if (gl.size() > 1) {
      cudaEventRecord(ctx->join[gi % kMaxGroups], s);
      cudaStreamWaitEvent(us, ctx->join[gi % kMaxGroups], 0);
    }
    off += static_cast<int64_t>(g.idx.size());
    ws_off += g.plan.ws_stride * g.grid * ((g.noisy || g.hr == 1) ? 1 : g.wpc);
  }
  cudaEventRecord(ctx->t1, us);
  ctx->timed = true;
  ctx->last_launches = launches;
  return BFSIM_OK;
}
}  // namespace

extern "C" {

int bfsim_run_batch_device(bfsim_ctx_t* ctx, const bfsim_scenario_t* scen_host, int64_t n_scen,
                           const bfsim_input_t* inputs_host, int32_t n_inputs,
                           const int32_t* class_base_dev, const bfsim_request_t* traces_dev,
                           const bfsim_sample_t* streams_dev, const bfsim_step_sink_t* steps_dev,
                           const bfsim_req_sink_t* reqs_dev, bfsim_result_t* results_dev,
                           void* stream, char* err, size_t errlen) {
  return run_batch_device_impl(ctx, scen_host, n_scen, inputs_host, n_inputs, class_base_dev,
                               traces_dev, streams_dev, steps_dev, reqs_dev, nullptr, results_dev,
                               stream, err, errlen);
}

int bfsim_run_batch(bfsim_ctx_t* ctx, const bfsim_scenario_t* scen, int64_t n_scen,
                    const bfsim_input_t* inputs, int32_t n_inputs, const int32_t* class_base,
                    int64_t n_class_base, const bfsim_request_t* traces, int64_t n_trace_records,
                    const bfsim_sample_t* streams, int64_t n_stream_samples,
                    const bfsim_step_sink_t* steps, int64_t n_step_records, int64_t n_load_values,
                    const bfsim_req_sink_t* reqs, int64_t n_req_entries, bfsim_result_t* results,
                    char* err, size_t errlen) {
  if (!ctx) return fail(err, errlen, BFSIM_EINVAL, "null context");
  cudaSetDevice(ctx->device);
  // host-side validation that needs the host inputs (single-class streams, bounds)
  std::vector<int> single(static_cast<size_t>(n_inputs), 0);
  for (int32_t i = 0; i < n_inputs; ++i) {
    const auto& in = inputs[i];
    if (in.offset < 0 || in.length < 0)
      return fail(err, errlen, BFSIM_EINVAL, "input: negative offset/length");
    if (in.class_base_offset < 0 || in.class_base_offset + in.s_max + 2 > n_class_base)
      return fail(err, errlen, BFSIM_EINVAL, "input: class_base slice out of range");
  }
  for (int64_t i = 0; i < n_scen; ++i) {
    const auto& s = scen[i];
    if (s.input_id < 0 || s.input_id >= n_inputs)
      return fail(err, errlen, BFSIM_EINVAL, "scenario: input_id out of range");
    const auto& in = inputs[s.input_id];
    if (s.mode == BFSIM_MODE_OVERLOADED) {
      if (in.offset + in.length > n_stream_samples)
        return fail(err, errlen, BFSIM_EINVAL, "input: stream slice out of range");
      bool one = true;
      for (int64_t j = 1; j < in.length && one; ++j)
        one = streams[in.offset + j].prefill == streams[in.offset].prefill;
      single[s.input_id] = one ? 1 : 0;
    } else if (in.offset + in.length > n_trace_records) {
      return fail(err, errlen, BFSIM_EINVAL, "input: trace slice out of range");
    }
    if (steps && steps->clock_start && s.step_capacity > 0 &&
        (s.step_offset < 0 || s.step_offset + s.step_capacity > n_step_records ||
         s.load_offset < 0 || s.load_offset + s.step_capacity * s.workers > n_load_values))
      return fail(err, errlen, BFSIM_EINVAL, "scenario: step sink slice out of range");
    if (reqs && reqs->start_step &&
        (s.req_offset < 0 || s.req_offset + in.length > n_req_entries))
      return fail(err, errlen, BFSIM_EINVAL, "scenario: request sink slice out of range");
    int rc = validate_scenario(s, inputs, n_inputs, &single, err, errlen);
    if (rc) {
      std::string m = "scenario " + std::to_string(i) + ": " + (err ? std::string(err) : "");
      return fail(err, errlen, rc, m.c_str());
    }
  }
  cudaError_t e;
  cudaStream_t us = nullptr;
  auto up = [&](DevBuf& b, const void* h, size_t bytes) -> cudaError_t {
    cudaError_t x = b.ensure(std::max<size_t>(bytes, 16));
    if (x != cudaSuccess) return x;
    if (bytes) x = cudaMemcpyAsync(b.p, h, bytes, cudaMemcpyHostToDevice, us);
    return x;
  };
  if ((e = up(ctx->cbase, class_base, n_class_base * 4)) != cudaSuccess) return cuda_fail(err, errlen, e, "H2D");
  if (traces && n_trace_records)
    if ((e = up(ctx->traces, traces, n_trace_records * sizeof(bfsim_request_t))) != cudaSuccess)
      return cuda_fail(err, errlen, e, "H2D");
  if (streams && n_stream_samples)
    if ((e = up(ctx->streams, streams, n_stream_samples * sizeof(bfsim_sample_t))) != cudaSuccess)
      return cuda_fail(err, errlen, e, "H2D");
  if ((e = ctx->results.ensure(n_scen * sizeof(bfsim_result_t))) != cudaSuccess)
    return cuda_fail(err, errlen, e, "alloc");
  bfsim_step_sink_t dsteps{};
  bool want_steps = steps && steps->clock_start && n_step_records > 0;
  // Page-locked step sinks (cudaHostAlloc / cudaHostRegister) are written by
  // the kernel directly over the host link: the 32-step record rows stream out
  // while the simulation runs instead of in one copy after it.
  bool zero_copy = false;
  if (want_steps) {
    void* dp[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};
    void* hp[5] = {steps->clock_start, steps->dt, steps->max_load, steps->active_count, steps->loads};
    zero_copy = true;
    for (int i = 0; i < 5 && zero_copy; ++i) {
      cudaPointerAttributes a{};
      zero_copy = hp[i] && cudaPointerGetAttributes(&a, hp[i]) == cudaSuccess &&
                  a.type == cudaMemoryTypeHost && a.devicePointer != nullptr;
      if (zero_copy) dp[i] = a.devicePointer;
    }
    cudaGetLastError();  // clear a failed query on pageable memory
    if (zero_copy) {
      dsteps.clock_start = static_cast<double*>(dp[0]);
      dsteps.dt = static_cast<double*>(dp[1]);
      dsteps.max_load = static_cast<double*>(dp[2]);
      dsteps.active_count = static_cast<int64_t*>(dp[3]);
      dsteps.loads = static_cast<double*>(dp[4]);
    }
  }
  if (want_steps && !zero_copy) {
    if ((e = ctx->st_cs.ensure(n_step_records * 8)) || (e = ctx->st_dt.ensure(n_step_records * 8)) ||
        (e = ctx->st_mx.ensure(n_step_records * 8)) || (e = ctx->st_ac.ensure(n_step_records * 8)) ||
        (e = ctx->st_ld.ensure(std::max<int64_t>(n_load_values, 1) * 8)))
      return cuda_fail(err, errlen, e, "alloc");
    dsteps.clock_start = static_cast<double*>(ctx->st_cs.p);
    dsteps.dt = static_cast<double*>(ctx->st_dt.p);
    dsteps.max_load = static_cast<double*>(ctx->st_mx.p);
    dsteps.active_count = static_cast<int64_t*>(ctx->st_ac.p);
    dsteps.loads = static_cast<double*>(ctx->st_ld.p);
  }
  bfsim_req_sink_t dreqs{}, hreqs{};
  bool want_reqs = reqs && reqs->start_step && n_req_entries > 0;
  // Page-locked request sinks: staged in HBM (the writes are scattered by
  // request id) and copied out per trajectory, coalesced, by its own warp
  // when it finishes -- overlapped with the trajectories still running.
  bool req_mirror = false;
  if (want_reqs) {
    void* hp[5] = {reqs->arrival_step, reqs->start_step, reqs->worker, reqs->admit_clock,
                   reqs->finish_clock};
    void* dp[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};
    req_mirror = true;
    for (int i = 0; i < 5 && req_mirror; ++i) {
      cudaPointerAttributes a{};
      req_mirror = hp[i] && cudaPointerGetAttributes(&a, hp[i]) == cudaSuccess &&
                   a.type == cudaMemoryTypeHost && a.devicePointer != nullptr;
      if (req_mirror) dp[i] = a.devicePointer;
    }
    cudaGetLastError();
    if (req_mirror) {
      hreqs.arrival_step = static_cast<int32_t*>(dp[0]);
      hreqs.start_step = static_cast<int32_t*>(dp[1]);
      hreqs.worker = static_cast<int32_t*>(dp[2]);
      hreqs.admit_clock = static_cast<double*>(dp[3]);
      hreqs.finish_clock = static_cast<double*>(dp[4]);
    }
  }
  if (want_reqs) {
    if ((e = ctx->rq_as.ensure(n_req_entries * 4)) || (e = ctx->rq_ss.ensure(n_req_entries * 4)) ||
        (e = ctx->rq_wk.ensure(n_req_entries * 4)) || (e = ctx->rq_ac.ensure(n_req_entries * 8)) ||
        (e = ctx->rq_fc.ensure(n_req_entries * 8)))
      return cuda_fail(err, errlen, e, "alloc");
    dreqs.arrival_step = static_cast<int32_t*>(ctx->rq_as.p);
    dreqs.start_step = static_cast<int32_t*>(ctx->rq_ss.p);
    dreqs.worker = static_cast<int32_t*>(ctx->rq_wk.p);
    dreqs.admit_clock = static_cast<double*>(ctx->rq_ac.p);
    dreqs.finish_clock = static_cast<double*>(ctx->rq_fc.p);
  }
  int rc = run_batch_device_impl(
      ctx, scen, n_scen, inputs, n_inputs, static_cast<const int32_t*>(ctx->cbase.p),
      traces ? static_cast<const bfsim_request_t*>(ctx->traces.p) : nullptr,
      streams ? static_cast<const bfsim_sample_t*>(ctx->streams.p) : nullptr,
      want_steps ? &dsteps : nullptr, want_reqs ? &dreqs : nullptr, req_mirror ? &hreqs : nullptr,
      static_cast<bfsim_result_t*>(ctx->results.p), us, err, errlen);
  if (rc) return rc;
  auto down = [&](void* h, const DevBuf& b, size_t bytes) {
    if (h && bytes) cudaMemcpyAsync(h, b.p, bytes, cudaMemcpyDeviceToHost, us);
  };
  down(results, ctx->results, n_scen * sizeof(bfsim_result_t));
  if (want_steps && !zero_copy) {
    down(steps->clock_start, ctx->st_cs, n_step_records * 8);
    down(steps->dt, ctx->st_dt, n_step_records * 8);
    down(steps->max_load, ctx->st_mx, n_step_records * 8);
    down(steps->active_count, ctx->st_ac, n_step_records * 8);
    down(steps->loads, ctx->st_ld, n_load_values * 8);
  }
  if (want_reqs && !req_mirror) {
    down(reqs->arrival_step, ctx->rq_as, n_req_entries * 4);
    down(reqs->start_step, ctx->rq_ss, n_req_entries * 4);
    down(reqs->worker, ctx->rq_wk, n_req_entries * 4);
    down(reqs->admit_clock, ctx->rq_ac, n_req_entries * 8);
    down(reqs->finish_clock, ctx->rq_fc, n_req_entries * 8);
  }
  if ((e = cudaStreamSynchronize(us)) != cudaSuccess) return cuda_fail(err, errlen, e, "step kernel");
  int first = BFSIM_OK;
  for (int64_t i = 0; i < n_scen; ++i) {
    int st = results[i].status;
    if (st != BFSIM_OK && st != BFSIM_PARTIAL && first == BFSIM_OK) first = st;
  }
  if (first == BFSIM_ESTREAM)
    return fail(err, errlen, BFSIM_ESTREAM, "overloaded sample stream exhausted");
  if (first == BFSIM_ERANGE)
    return fail(err, errlen, BFSIM_ERANGE, "GPU path: drift * step exceeded the int32 slot range (lower max_steps)");
  return first;
}


int bfsim_assign_batch(bfsim_ctx_t* ctx, const bfsim_assign_call_t* calls, int64_t n_calls,
                       const double* previews, int64_t n_previews, const double* futures,
                       int64_t n_futures, const int32_t* caps, const int32_t* active_counts,
                       int64_t n_workers, int64_t search_limit, int32_t* pairs, int64_t n_pairs_cap,
                       int64_t* n_pairs, double* cost, int32_t* status, char* err, size_t errlen) {
  if (!ctx) return fail(err, errlen, BFSIM_EINVAL, "null context");
  if (n_calls <= 0) return BFSIM_OK;
  if (n_calls > INT32_MAX) return fail(err, errlen, BFSIM_EINVAL, "too many calls");
  if (search_limit < 0) return fail(err, errlen, BFSIM_EINVAL, "search_limit < 0");
  cudaSetDevice(ctx->device);
  int n_max = 1, h_max = 0;
  bool any_exact = false;
  int ex_n = 1, ex_h = 0;  // bfio-exact's per-lane scratch bounds (n <= 64, H <= 16)
  auto int_ok = [](double v) { return v >= 0.0 && v < 2147483648.0 && v == std::floor(v); };
  for (int64_t k = 0; k < n_calls; ++k) {
    const auto& c = calls[k];
    if (c.policy < 0 || c.policy > 3) return fail(err, errlen, BFSIM_EINVAL, "unknown policy");
    if (c.workers < 1 || c.workers > 32)
      return fail(err, errlen, BFSIM_EINVAL, "GPU assign: workers must be 1..32");
    if (c.horizon < 0 || c.horizon > 64 || c.n_waiting < 0 || c.n_waiting > 4096)
      return fail(err, errlen, BFSIM_EINVAL, "GPU assign: horizon 0..64, n_waiting 0..4096");
    if (c.policy == BFSIM_POLICY_BFIO_EXACT && (c.workers > 16 || c.horizon > 16 || c.n_waiting > 64))
      return fail(err, errlen, BFSIM_EINVAL, "GPU bfio-exact: workers <= 16, horizon <= 16, n_waiting <= 64");
    const int64_t H1 = c.horizon + 1;
    if (c.preview_offset < 0 || c.preview_offset + c.n_waiting * H1 > n_previews ||
        c.future_offset < 0 || c.future_offset + c.workers * H1 > n_futures || c.worker_offset < 0 ||
        c.worker_offset + c.workers > n_workers)
      return fail(err, errlen, BFSIM_EINVAL, "assign call: slice out of range");
    int64_t capsum = 0;
    for (int g = 0; g < c.workers; ++g) {
      if (caps[c.worker_offset + g] < 0 || active_counts[c.worker_offset + g] < 0)
        return fail(err, errlen, BFSIM_EINVAL, "assign call: negative cap or active_count");
      // the fcfs / jsq argmax keys pack cap (20 bits) and count (26 bits) with the lane
      if (caps[c.worker_offset + g] >= (1 << 20) || active_counts[c.worker_offset + g] >= (1 << 26))
        return fail(err, errlen, BFSIM_EINVAL, "GPU assign: cap must be < 2^20 and active_count < 2^26");
      capsum += caps[c.worker_offset + g];
    }
    const int64_t U = std::min<int64_t>(c.n_waiting, capsum);
    if (c.pair_offset < 0 || c.pair_offset + 2 * U > n_pairs_cap)
      return fail(err, errlen, BFSIM_EINVAL, "assign call: pair slice out of range");
    for (int64_t j = 0; j < c.n_waiting * H1; ++j)
      if (!int_ok(previews[c.preview_offset + j]))
        return fail(err, errlen, BFSIM_EINVAL, "GPU assign: previews must be integers in [0, 2^31)");
    for (int64_t j = 0; j < c.workers * H1; ++j)
      if (!int_ok(futures[c.future_offset + j]))
        return fail(err, errlen, BFSIM_EINVAL, "GPU assign: futures must be integers in [0, 2^31)");
    n_max = std::max(n_max, c.n_waiting);
    h_max = std::max(h_max, c.horizon);
    if (c.policy == BFSIM_POLICY_BFIO_EXACT) {
      any_exact = true;
      ex_n = std::max(ex_n, c.n_waiting);
      ex_h = std::max(ex_h, c.horizon);
    }
  }
  std::vector<int64_t> pv(static_cast<size_t>(std::max<int64_t>(n_previews, 1)));
  std::vector<int64_t> fu(static_cast<size_t>(std::max<int64_t>(n_futures, 1)));
  for (int64_t j = 0; j < n_previews; ++j) pv[j] = static_cast<int64_t>(previews[j]);
  for (int64_t j = 0; j < n_futures; ++j) fu[j] = static_cast<int64_t>(futures[j]);
  bfsim::AssignParams ap{};
  ap.n_calls = static_cast<int32_t>(n_calls);
  ap.n_max = n_max;
  ap.h_max = h_max;
  ap.ex_n = ex_n;
  auto al = [](int64_t x) { return (x + 15) & ~int64_t{15}; };
  ap.i64_offset = al(3LL * n_max * 4);
  ap.lane_offset = al(ap.i64_offset + (33LL * (h_max + 1)) * 8);
  // per-lane exact-search scratch only when a bfio-exact call is present
  ap.lane_i64_offset = any_exact ? al((3LL * ex_n + 33) * 4) : 0;
  ap.lane_stride = any_exact ? al(ap.lane_i64_offset + (ex_h + 1) * 32LL * 8) : 0;
  ap.ws_stride = al(ap.lane_offset + 32 * ap.lane_stride);
  ap.limit = search_limit;
  cudaStream_t us = nullptr;
  cudaError_t e;
  auto up = [&](DevBuf& b, const void* h, size_t bytes) -> cudaError_t {
    cudaError_t x = b.ensure(std::max<size_t>(bytes, 16));
    if (x == cudaSuccess && bytes) x = cudaMemcpyAsync(b.p, h, bytes, cudaMemcpyHostToDevice, us);
    return x;
  };
  if ((e = up(ctx->a_calls, calls, n_calls * sizeof(bfsim_assign_call_t))) ||
      (e = up(ctx->a_pv, pv.data(), pv.size() * 8)) || (e = up(ctx->a_fut, fu.data(), fu.size() * 8)) ||
      (e = up(ctx->a_caps, caps, n_workers * 4)) || (e = up(ctx->a_cnt, active_counts, n_workers * 4)) ||
      (e = up(ctx->a_pairs, pairs, n_pairs_cap > 0 ? n_pairs_cap * 4 : 0)) ||
      (e = ctx->a_np.ensure(n_calls * 8)) || (e = ctx->a_cost.ensure(n_calls * 8)) ||
      (e = ctx->a_st.ensure(n_calls * 4)) || (e = ctx->a_ws.ensure(ap.ws_stride * n_calls)))
    return cuda_fail(err, errlen, e, "assign buffers");
  ap.calls = static_cast<const bfsim_assign_call_t*>(ctx->a_calls.p);
  ap.previews = static_cast<const int64_t*>(ctx->a_pv.p);
  ap.futures = static_cast<const int64_t*>(ctx->a_fut.p);
  ap.caps = static_cast<const int32_t*>(ctx->a_caps.p);
  ap.counts = static_cast<const int32_t*>(ctx->a_cnt.p);
  ap.pairs = static_cast<int32_t*>(ctx->a_pairs.p);
  ap.n_pairs = static_cast<int64_t*>(ctx->a_np.p);
  ap.cost = static_cast<double*>(ctx->a_cost.p);
  ap.status = static_cast<int32_t*>(ctx->a_st.p);
  ap.ws = static_cast<unsigned char*>(ctx->a_ws.p);
  int rc = bfsim::launch_assign(ap, us);
  if (rc) return cuda_fail(err, errlen, static_cast<cudaError_t>(rc), "assign kernel launch");
  ctx->last_launches = 1;
  if (n_pairs_cap > 0) cudaMemcpyAsync(pairs, ctx->a_pairs.p, n_pairs_cap * 4, cudaMemcpyDeviceToHost, us);
  cudaMemcpyAsync(n_pairs, ctx->a_np.p, n_calls * 8, cudaMemcpyDeviceToHost, us);
  cudaMemcpyAsync(cost, ctx->a_cost.p, n_calls * 8, cudaMemcpyDeviceToHost, us);
  cudaMemcpyAsync(status, ctx->a_st.p, n_calls * 4, cudaMemcpyDeviceToHost, us);
  if ((e = cudaStreamSynchronize(us)) != cudaSuccess) return cuda_fail(err, errlen, e, "assign kernel");
  for (int64_t k = 0; k < n_calls; ++k)
    if (status[k] == BFSIM_ELIMIT) return fail(err, errlen, BFSIM_ELIMIT, "bfio-exact: feasible allocations exceed search limit; use bfio-greedy");
  return BFSIM_OK;
}

}  // extern "C"
