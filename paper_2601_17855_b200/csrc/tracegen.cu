// Device-side synthetic input generation: the reference's
// sample_instance traces (workload.hpp:241-266) and run_overloaded's top-up
// sample streams (oracle.hpp:177-183), generated in HBM, byte-identical to the
// host batcher (host_batcher.cpp) and therefore to the reference.
//
// One warp per trace / stream. The trace is one mt19937_64(seed) stream read
// in the reference's order: the first gap, then per arrival prefill, decode and
// the next gap (workload.hpp:255-263). Almost every record consumes the same
// number of engine words (k = [uniform/empirical prefill] + [geometric/
// empirical decode] + [gap]), so lane j of a 32-record chunk reads its words
// at cursor + j*k and computes its record independently:
//   * uniform_int_distribution (libstdc++ uniform_int_dist.h:257-281, Lemire's
//     nearly-divisionless method on the 128-bit product for a 64-bit engine),
//   * geometric_distribution (random.tcc:1052-1073: floor(log(1-U)/log(1-p)),
//     redrawn while >= LONG_MAX + 1/2),
//   * exponential_distribution (random.h:4904: -log(1-U)/rate),
// with U = generate_canonical<double, 53> and glibc's own `log`
// (libm_log.cuh). A record whose draw would take an extra word (a Lemire
// rejection or a geometric redraw) ends the regular prefix of the chunk; the
// warp replays that record through the sequential rules and continues from
// the shifted cursor. The arrival times t_{i+1} = t_i + gap are accumulated
// left to right exactly as the reference does (a 32-deep dependent add per
// chunk, the only serial part). The engine's tempered output words live in a
// shared-memory ring refilled a block of 312 at a time by the warp-parallel
// twist.
//
// Per input the kernel also produces what bfsim_prepare_trace computes on the
// host: length, largest prefill and decode present, and the class_base
// counting-sort table (#records with prefill < c).
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "bfsim_gpu.h"
#include "common.h"
#include "libm_log.cuh"

namespace {

using bfsim::fail;

constexpr int kN = 312, kM = 156;
constexpr int kWarps = 4;         // warps (traces) per CTA
constexpr int kRingWords = 1024;  // tempered engine words per warp
constexpr uint64_t kA = 0xB5026F5AA96619E9ull;
constexpr uint64_t kUpper = 0xFFFFFFFF80000000ull, kLower = 0x000000007FFFFFFFull;

// Per-input generation spec (device copy). kind: 0 uniform / geometric,
// 1 fixed, 2 empirical.
struct GenSpec {
  int32_t pkind, dkind;
  int64_t pfixed;      // uniform s_max or fixed prefill
  int64_t dfixed;      // fixed decode length
  double p;            // geometric p
  double log_1_p;      // log(1 - p), geometric_distribution::param_type (random.h)
  int64_t pval_off, pval_n, dval_off, dval_n;  // empirical lists in the value pool
  double rate, duration;
  uint64_t seed;
  int64_t n_fixed;     // stream mode: samples to draw
  int64_t rec_off, rec_cap;  // output slice
  int64_t cb_off;      // class_base slice (cb_len entries)
  int32_t cb_len;
  uint32_t force_slow;  // test hook: lanes whose record takes the sequential path anyway
};

struct GenOut {
  int64_t n;  // records (trace: may exceed rec_cap -> ERANGE)
  int32_t s_max, max_decode;
  int32_t status, pad;
};

__device__ __forceinline__ uint64_t temper(uint64_t y) {
  y ^= (y >> 29) & 0x5555555555555555ull;
  y ^= (y << 17) & 0x71D67FFFEDA60000ull;
  y ^= (y << 37) & 0xFFF7EEE000000000ull;
  y ^= y >> 43;
  return y;
}
__device__ __forceinline__ uint64_t mix(uint64_t lo_word, uint64_t next, uint64_t far) {
  const uint64_t x = (lo_word & kUpper) | (next & kLower);
  return far ^ (x >> 1) ^ ((x & 1ull) ? kA : 0ull);
}

// Warp-private engine: state + a ring of tempered outputs, position-addressed.
struct Engine {
  uint64_t* mt;    // kN words
  uint64_t* ring;  // kRingWords words
  uint64_t produced;

  __device__ void seed(uint64_t s) {
    if ((threadIdx.x & 31) == 0) {
      uint64_t x = s;
      mt[0] = x;
      for (int i = 1; i < kN; ++i) {
        x = 6364136223846793005ull * (x ^ (x >> 62)) + static_cast<uint64_t>(i);
        mt[i] = x;
      }
    }
    produced = 0;
    __syncwarp();
  }
  // _M_gen_rand in two parallel halves (see engine_impl.cuh mt_twist), then the
  // 312 tempered outputs appended to the ring.
  __device__ void refill() {
    const int lane = threadIdx.x & 31;
    uint64_t v[5];
#pragma unroll
    for (int t = 0; t < 5; ++t) {
      const int i = lane + 32 * t;
      v[t] = i < kM ? mix(mt[i], mt[i + 1], mt[i + kM]) : 0ull;
    }
    __syncwarp();
#pragma unroll
    for (int t = 0; t < 5; ++t)
      if (lane + 32 * t < kM) mt[lane + 32 * t] = v[t];
    __syncwarp();
#pragma unroll
    for (int t = 0; t < 5; ++t) {
      const int i = kM + lane + 32 * t;
      v[t] = i < kN ? mix(mt[i], mt[i + 1 < kN ? i + 1 : 0], mt[i - kM]) : 0ull;
    }
    __syncwarp();
#pragma unroll
    for (int t = 0; t < 5; ++t)
      if (kM + lane + 32 * t < kN) mt[kM + lane + 32 * t] = v[t];
    __syncwarp();
    for (int i = lane; i < kN; i += 32) ring[(produced + i) & (kRingWords - 1)] = temper(mt[i]);
    produced += kN;
    __syncwarp();
  }
  // make words [.., pos] available (warp-uniform call)
  __device__ void ensure(uint64_t pos) {
    while (produced <= pos) refill();
  }
  __device__ uint64_t at(uint64_t pos) const { return ring[pos & (kRingWords - 1)]; }
};

// generate_canonical<double, 53> over a 64-bit engine (random.tcc): one word.
__device__ __forceinline__ double canonical(uint64_t u) {
  const double r = __dmul_rn(__ull2double_rn(u), 0x1p-64);
  return r >= 1.0 ? 0x1.fffffffffffffp-1 : r;
}

// Lemire step for range `er` (= urange + 1): returns true and the value when
// the first word decides it (low >= er, or low >= threshold).
__device__ __forceinline__ bool lemire_first(uint64_t w, uint64_t er, uint64_t* out) {
  const uint64_t low = w * er;
  *out = __umul64hi(w, er);
  if (low >= er) return true;
  const uint64_t thr = (0ull - er) % er;
  return low >= thr;
}

constexpr double kNaf = 0x1.fffffffffffffp-2;  // (1 - eps) / 2
constexpr double kThr = 0x1p63;                // LONG_MAX + naf as a double

// One geometric candidate: floor(log(1 - U) / log(1 - p)).
__device__ __forceinline__ double geo_cand(uint64_t w, double log_1_p, const bfsim::libm::LogEntry* tab) {
  const double u = canonical(w);
  return floor(__ddiv_rn(bfsim::libm::log(__dsub_rn(1.0, u), tab), log_1_p));
}
__device__ __forceinline__ double exp_gap(uint64_t w, double rate, const bfsim::libm::LogEntry* tab) {
  const double u = canonical(w);
  return __ddiv_rn(-bfsim::libm::log(__dsub_rn(1.0, u), tab), rate);
}

// The sequential rules for one (prefill, decode) pair from word `pos` on
// (any number of rejections); warp-uniform. Returns the next position.
__device__ uint64_t draw_pair_seq(Engine& eng, uint64_t pos, const GenSpec& sp, const int64_t* vals,
                                  const bfsim::libm::LogEntry* tab, int64_t* s_out, int64_t* o_out) {
  int64_t s = sp.pfixed;
  if (sp.pkind != 1) {
    const uint64_t er = sp.pkind == 2 ? static_cast<uint64_t>(sp.pval_n) : static_cast<uint64_t>(sp.pfixed);
    eng.ensure(pos);
    uint64_t w = eng.at(pos++);
    uint64_t low = w * er, hi = __umul64hi(w, er);
    if (low < er) {
      const uint64_t thr = (0ull - er) % er;
      while (low < thr) {
        eng.ensure(pos);
        w = eng.at(pos++);
        low = w * er;
        hi = __umul64hi(w, er);
      }
    }
    s = sp.pkind == 2 ? vals[sp.pval_off + static_cast<int64_t>(hi)] : static_cast<int64_t>(hi) + 1;
  }
  int64_t o = sp.dfixed;
  if (sp.dkind == 0) {
    double c;
    do {
      eng.ensure(pos);
      c = geo_cand(eng.at(pos++), sp.log_1_p, tab);
    } while (c >= kThr);
    o = 1 + static_cast<int64_t>(__dadd_rn(c, kNaf));
  } else if (sp.dkind == 2) {
    const uint64_t er = static_cast<uint64_t>(sp.dval_n);
    eng.ensure(pos);
    uint64_t w = eng.at(pos++);
    uint64_t low = w * er, hi = __umul64hi(w, er);
    if (low < er) {
      const uint64_t thr = (0ull - er) % er;
      while (low < thr) {
        eng.ensure(pos);
        w = eng.at(pos++);
        low = w * er;
        hi = __umul64hi(w, er);
      }
    }
    o = vals[sp.dval_off + static_cast<int64_t>(hi)];
  }
  *s_out = s;
  *o_out = o;
  return pos;
}

__constant__ double c_logtab[256] = {BFSIM_LOG_TAB};

// 16-byte record stores (the pool slices are 16-byte aligned)
__device__ __forceinline__ void put_record(bfsim_request_t* base, int64_t i, double a, int64_t s, int64_t o) {
  const long long ab = __double_as_longlong(a);
  reinterpret_cast<int4*>(base)[i] = make_int4(static_cast<int>(ab & 0xffffffffll), static_cast<int>(ab >> 32),
                                               static_cast<int>(s), static_cast<int>(o));
}

// MODE 0: sample_instance trace; MODE 1: overloaded stream of n_fixed samples.
template <int MODE>
__global__ void __launch_bounds__(32 * kWarps) gen_kernel(const GenSpec* __restrict__ specs, int32_t n_specs,
                                                          const int64_t* __restrict__ vals,
                                                          bfsim_request_t* __restrict__ traces,
                                                          bfsim_sample_t* __restrict__ streams,
                                                          int32_t* __restrict__ class_base,
                                                          GenOut* __restrict__ outs) {
  __shared__ bfsim::libm::LogEntry tab[128];
  __shared__ uint64_t mt_s[kWarps][kN];
  __shared__ uint64_t ring_s[kWarps][kRingWords];
  for (int i = threadIdx.x; i < 128; i += blockDim.x) tab[i] = {c_logtab[2 * i], c_logtab[2 * i + 1]};
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const unsigned full = 0xffffffffu;
  Engine eng{mt_s[warp], ring_s[warp], 0};
  for (int id = blockIdx.x * kWarps + warp; id < n_specs; id += gridDim.x * kWarps) {
    const GenSpec sp = specs[id];
    eng.seed(sp.seed);
    int32_t* cb = class_base + sp.cb_off;
    const int kp = sp.pkind != 1 ? 1 : 0, kd = sp.dkind != 1 ? 1 : 0;
    const int k = kp + kd + (MODE == 0 ? 1 : 0);
    uint64_t pos = 0;
    double t = 0.0;
    if (MODE == 0) {
      eng.ensure(0);
      t = exp_gap(eng.at(0), sp.rate, tab);
      pos = 1;
    }
    int64_t n = 0;
    int32_t smax = 1, omax = 1, status = BFSIM_OK;  // as bfsim_prepare_trace
    const int64_t limit = MODE == 0 ? INT64_MAX : sp.n_fixed;
    while (n < limit && (MODE != 0 || t < sp.duration)) {
      eng.ensure(pos + 32 * k + 1);
      // --- regular chunk: lane j's words at pos + j*k
      const uint64_t p0 = pos + static_cast<uint64_t>(lane) * k;
      bool regular = true;
      int64_t s = sp.pfixed, o = sp.dfixed;
      double gap = 0.0;
      int q = 0;
      if (kp) {
        const uint64_t er = sp.pkind == 2 ? static_cast<uint64_t>(sp.pval_n) : static_cast<uint64_t>(sp.pfixed);
        uint64_t v;
        regular = lemire_first(eng.at(p0 + q++), er, &v);
        s = sp.pkind == 2 ? vals[sp.pval_off + static_cast<int64_t>(v)] : static_cast<int64_t>(v) + 1;
      }
      if (kd) {
        if (sp.dkind == 0) {
          const double c = geo_cand(eng.at(p0 + q++), sp.log_1_p, tab);
          regular = regular && c < kThr;
          o = 1 + static_cast<int64_t>(__dadd_rn(c, kNaf));
        } else {
          uint64_t v;
          regular = lemire_first(eng.at(p0 + q++), static_cast<uint64_t>(sp.dval_n), &v) && regular;
          o = vals[sp.dval_off + static_cast<int64_t>(v)];
        }
      }
      if (MODE == 0) gap = exp_gap(eng.at(p0 + q), sp.rate, tab);
      regular = regular && !((sp.force_slow >> lane) & 1u);
      const unsigned irr = __ballot_sync(full, !regular);
      int f = irr ? __ffs(irr) - 1 : 32;  // regular prefix length
      if (MODE == 1 && n + f > limit) f = static_cast<int>(limit - n);
      // arrivals: a_j = t + gap_0 + ... + gap_{j-1}, left to right
      double a = t, next_t = t;
      int stop = f;
      if (MODE == 0) {
        double acc = t;
        for (int j = 0; j < f; ++j) {
          if (j == lane) a = acc;
          acc = __dadd_rn(acc, __shfl_sync(full, gap, j));
        }
        next_t = acc;
        const unsigned past = __ballot_sync(full, lane < f && !(a < sp.duration));
        if (past) stop = __ffs(past) - 1;
      }
      const bool keep = lane < stop;
      if (keep && o > INT32_MAX) status = BFSIM_EINVAL;
      if (keep) {
        const int64_t r = n + lane;
        smax = max(smax, static_cast<int32_t>(s));
        omax = max(omax, static_cast<int32_t>(o < INT32_MAX ? o : INT32_MAX));
        if (MODE == 0) {
          if (r < sp.rec_cap) {
            put_record(traces, sp.rec_off + r, a, s, o);
            atomicAdd(cb + s + 1, 1);
          }
        } else {
          streams[sp.rec_off + r] = bfsim_sample_t{static_cast<int32_t>(s), static_cast<int32_t>(o)};
          atomicAdd(cb + s + 1, 1);
        }
      }
      n += stop;
      pos += static_cast<uint64_t>(stop) * k;
      if (MODE == 0) {
        if (stop < f) break;  // an arrival reached the duration
        t = next_t;
      }
      if (f == 32 || (MODE == 1 && n >= limit)) continue;
      // --- the irregular record at lane f: the sequential rules
      if (MODE == 0 && !(t < sp.duration)) break;
      int64_t s2, o2;
      pos = draw_pair_seq(eng, pos, sp, vals, tab, &s2, &o2);
      if (lane == 0) {
        if (o2 > INT32_MAX) status = BFSIM_EINVAL;
        smax = max(smax, static_cast<int32_t>(s2));
        omax = max(omax, static_cast<int32_t>(o2 < INT32_MAX ? o2 : INT32_MAX));
        if (MODE == 0) {
          if (n < sp.rec_cap) {
            put_record(traces, sp.rec_off + n, t, s2, o2);
            atomicAdd(cb + s2 + 1, 1);
          }
        } else {
          streams[sp.rec_off + n] = bfsim_sample_t{static_cast<int32_t>(s2), static_cast<int32_t>(o2)};
          atomicAdd(cb + s2 + 1, 1);
        }
      }
      ++n;
      if (MODE == 0) {
        eng.ensure(pos);
        t = __dadd_rn(t, exp_gap(eng.at(pos), sp.rate, tab));
        ++pos;
      }
    }
    // warp reductions of the statistics
#pragma unroll
    for (int d = 16; d; d >>= 1) {
      smax = max(smax, __shfl_xor_sync(full, smax, d));
      omax = max(omax, __shfl_xor_sync(full, omax, d));
      status = max(status, __shfl_xor_sync(full, status, d));
    }
    if (lane == 0) outs[id] = GenOut{n, smax, omax, status, 0};
    __syncwarp();
  }
}

// class_base: inclusive scan of the per-class counts (count of prefill v at
// index v + 1), one warp per input.
__global__ void __launch_bounds__(128) class_scan_kernel(const GenSpec* __restrict__ specs, int32_t n_specs,
                                                         int32_t* __restrict__ class_base) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= n_specs) return;
  const GenSpec sp = specs[warp];
  int32_t* cb = class_base + sp.cb_off;
  int32_t carry = 0;
  for (int base = 0; base < sp.cb_len; base += 32) {
    const int i = base + lane;
    int32_t v = i < sp.cb_len ? cb[i] : 0;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const int32_t u = __shfl_up_sync(0xffffffffu, v, d);
      if (lane >= d) v += u;
    }
    v += carry;
    if (i < sp.cb_len) cb[i] = v;
    carry = __shfl_sync(0xffffffffu, v, 31);
  }
}

int cuda_fail(char* err, size_t errlen, cudaError_t e, const char* what) {
  std::string m = std::string(what) + ": " + cudaGetErrorString(e);
  return fail(err, errlen, BFSIM_ECUDA, m.c_str());
}

// Validation as the host batcher's (host_batcher.cpp make_dists, mirroring the
// reference's distribution factories), plus the pool bounds.
int prefill_bound(const bfsim_dist_t& d, int64_t* smax, char* err, size_t errlen) {
  if (d.kind == 2) {
    if (!d.values || d.n_values < 1) return fail(err, errlen, BFSIM_EINVAL, "prefill: empty empirical list");
    int64_t mx = 0;
    for (int64_t i = 0; i < d.n_values; ++i) {
      if (d.values[i] < 1) return fail(err, errlen, BFSIM_EINVAL, "prefill: empirical value < 1");
      if (d.values[i] > BFSIM_MAX_CLASSES)
        return fail(err, errlen, BFSIM_EINVAL, "prefill: empirical value exceeds the GPU class limit");
      mx = std::max(mx, d.values[i]);
    }
    *smax = mx;
    return BFSIM_OK;
  }
  if (d.kind != 0 && d.kind != 1) return fail(err, errlen, BFSIM_EINVAL, "prefill: unknown distribution kind");
  if (d.fixed < 1)
    return fail(err, errlen, BFSIM_EINVAL, d.kind ? "prefill: fixed value must be >= 1" : "prefill: s_max must be >= 1");
  if (d.fixed > BFSIM_MAX_CLASSES)
    return fail(err, errlen, BFSIM_EINVAL, "prefill: value exceeds the GPU class limit");
  *smax = d.fixed;
  return BFSIM_OK;
}
int decode_check(const bfsim_dist_t& d, char* err, size_t errlen) {
  if (d.kind == 2) {
    if (!d.values || d.n_values < 1) return fail(err, errlen, BFSIM_EINVAL, "decode: empty empirical list");
    for (int64_t i = 0; i < d.n_values; ++i) {
      if (d.values[i] < 1) return fail(err, errlen, BFSIM_EINVAL, "decode: empirical value < 1");
      if (d.values[i] > INT32_MAX) return fail(err, errlen, BFSIM_EINVAL, "decode: empirical value exceeds int32");
    }
    return BFSIM_OK;
  }
  if (d.kind == 0 && !(d.p > 0.0 && d.p < 1.0)) return fail(err, errlen, BFSIM_EINVAL, "decode: p must be in (0,1)");
  if (d.kind == 1 && d.fixed < 1) return fail(err, errlen, BFSIM_EINVAL, "decode: fixed length must be >= 1");
  if (d.kind != 0 && d.kind != 1) return fail(err, errlen, BFSIM_EINVAL, "decode: unknown distribution kind");
  return BFSIM_OK;
}

// Records reserved for a Poisson(rate * duration) count: mean + 12 sd + 64
// (exceeded with probability < 1e-30; the kernel reports ERANGE if it is).
int64_t trace_bound(double rate, double duration) {
  const double mu = rate * duration;
  return static_cast<int64_t>(std::ceil(mu + 12.0 * std::sqrt(mu) + 64.0));
}

int plan(const bfsim_gen_spec_t* specs, int32_t n, bool stream_mode, int64_t n_samples,
         std::vector<GenSpec>* out, std::vector<int64_t>* vals, int64_t* rec_total, int64_t* cb_total, char* err,
         size_t errlen) {
  if (n < 0 || (n > 0 && !specs)) return fail(err, errlen, BFSIM_EINVAL, "generate: bad spec list");
  if (stream_mode && n_samples < 0) return fail(err, errlen, BFSIM_EINVAL, "generate: negative stream length");
  out->resize(n);
  vals->clear();
  // test hook (tests/test_gpu_tracegen.py): a lane mask whose records replay
  // through the sequential rules, exercising the rejection path's cursor logic
  const char* fs = std::getenv("BFSIM_GEN_FORCE_SLOW");
  const uint32_t force = fs ? static_cast<uint32_t>(std::strtoul(fs, nullptr, 0)) : 0u;
  int64_t rec = 0, cbo = 0;
  for (int32_t i = 0; i < n; ++i) {
    const bfsim_gen_spec_t& s = specs[i];
    int64_t smax = 0;
    int rc = prefill_bound(s.prefill, &smax, err, errlen);
    if (rc) return rc;
    if ((rc = decode_check(s.decode, err, errlen))) return rc;
    if (!stream_mode) {
      if (s.rate <= 0.0) return fail(err, errlen, BFSIM_EINVAL, "sample_instance: rate must be > 0");
      if (s.duration <= 0.0) return fail(err, errlen, BFSIM_EINVAL, "sample_instance: duration must be > 0");
      if (!(s.rate * s.duration < 4e9)) return fail(err, errlen, BFSIM_EINVAL, "generate: trace too long");
    }
    GenSpec g{};
    g.pkind = s.prefill.kind;
    g.dkind = s.decode.kind;
    g.pfixed = s.prefill.kind == 2 ? 0 : s.prefill.fixed;
    g.dfixed = s.decode.kind == 1 ? s.decode.fixed : 0;
    g.p = s.decode.p;
    g.log_1_p = 0.0;
    if (s.decode.kind == 0) g.log_1_p = std::log(1.0 - s.decode.p);  // glibc, as param_type does
    if (s.prefill.kind == 2) {
      g.pval_off = static_cast<int64_t>(vals->size());
      g.pval_n = s.prefill.n_values;
      vals->insert(vals->end(), s.prefill.values, s.prefill.values + s.prefill.n_values);
    }
    if (s.decode.kind == 2) {
      g.dval_off = static_cast<int64_t>(vals->size());
      g.dval_n = s.decode.n_values;
      vals->insert(vals->end(), s.decode.values, s.decode.values + s.decode.n_values);
    }
    g.rate = s.rate;
    g.duration = s.duration;
    g.seed = s.seed;
    g.n_fixed = n_samples;
    g.rec_off = rec;
    g.rec_cap = stream_mode ? n_samples : trace_bound(s.rate, s.duration);
    g.cb_off = cbo;
    g.cb_len = static_cast<int32_t>(smax + 2);
    g.force_slow = force;
    rec += g.rec_cap;
    cbo += g.cb_len;
    (*out)[i] = g;
  }
  *rec_total = rec;
  *cb_total = cbo;
  return BFSIM_OK;
}

int generate(bfsim_ctx_t* ctx, const bfsim_gen_spec_t* specs, int32_t n, bool stream_mode, int64_t n_samples,
             void* records_dev, int64_t records_cap, int32_t* class_base_dev, int64_t class_base_cap,
             bfsim_input_t* inputs_out, void* stream_v, char* err, size_t errlen) {
  if (!ctx) return fail(err, errlen, BFSIM_EINVAL, "null context");
  std::vector<GenSpec> gs;
  std::vector<int64_t> vals;
  int64_t rec_total = 0, cb_total = 0;
  int rc = plan(specs, n, stream_mode, n_samples, &gs, &vals, &rec_total, &cb_total, err, errlen);
  if (rc) return rc;
  if (rec_total > records_cap || cb_total > class_base_cap)
    return fail(err, errlen, BFSIM_EINVAL, "generate: pool smaller than bfsim_generate_bounds");
  if (n == 0) return BFSIM_OK;
  if (!records_dev || !class_base_dev || !inputs_out) return fail(err, errlen, BFSIM_EINVAL, "generate: null buffer");
  cudaError_t e = cudaSetDevice(bfsim_ctx_device(ctx));
  if (e != cudaSuccess) return cuda_fail(err, errlen, e, "cudaSetDevice");
  cudaStream_t st = static_cast<cudaStream_t>(stream_v);
  const size_t spec_b = gs.size() * sizeof(GenSpec), val_b = std::max<size_t>(8, vals.size() * 8),
               out_b = gs.size() * sizeof(GenOut);
  char* scratch = nullptr;
  if ((e = cudaMallocAsync(reinterpret_cast<void**>(&scratch), spec_b + val_b + out_b + 64, st)) != cudaSuccess)
    return cuda_fail(err, errlen, e, "generate: scratch");
  GenSpec* d_specs = reinterpret_cast<GenSpec*>(scratch);
  int64_t* d_vals = reinterpret_cast<int64_t*>(scratch + spec_b);
  GenOut* d_out = reinterpret_cast<GenOut*>(scratch + spec_b + val_b);
  std::vector<GenOut> ho(gs.size());
  e = cudaMemcpyAsync(d_specs, gs.data(), spec_b, cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess && !vals.empty())
    e = cudaMemcpyAsync(d_vals, vals.data(), vals.size() * 8, cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess) e = cudaMemsetAsync(class_base_dev, 0, cb_total * sizeof(int32_t), st);
  if (e == cudaSuccess) {
    const int blocks = static_cast<int>((n + kWarps - 1) / kWarps);
    if (stream_mode)
      gen_kernel<1><<<blocks, 32 * kWarps, 0, st>>>(d_specs, n, d_vals, nullptr,
                                                     static_cast<bfsim_sample_t*>(records_dev), class_base_dev, d_out);
    else
      gen_kernel<0><<<blocks, 32 * kWarps, 0, st>>>(d_specs, n, d_vals, static_cast<bfsim_request_t*>(records_dev),
                                                     nullptr, class_base_dev, d_out);
    e = cudaGetLastError();
  }
  if (e == cudaSuccess) {
    class_scan_kernel<<<(n + 3) / 4, 128, 0, st>>>(d_specs, n, class_base_dev);
    e = cudaGetLastError();
  }
  if (e == cudaSuccess) e = cudaMemcpyAsync(ho.data(), d_out, out_b, cudaMemcpyDeviceToHost, st);
  cudaFreeAsync(scratch, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return cuda_fail(err, errlen, e, "generate");
  for (int32_t i = 0; i < n; ++i) {
    if (ho[i].status == BFSIM_EINVAL)
      return fail(err, errlen, BFSIM_EINVAL, "sample_instance: decode exceeds int32");
    if (ho[i].n > gs[i].rec_cap) return fail(err, errlen, BFSIM_ERANGE, "generate: trace longer than its bound");
    bfsim_input_t& in = inputs_out[i];
    in.offset = gs[i].rec_off;
    in.length = ho[i].n;
    in.class_base_offset = gs[i].cb_off;
    in.s_max = ho[i].s_max;
    in.max_decode = ho[i].max_decode;
  }
  return BFSIM_OK;
}

}  // namespace

extern "C" {

int bfsim_generate_bounds(const bfsim_gen_spec_t* specs, int32_t n, int64_t stream_samples, int64_t* n_records,
                          int64_t* n_class_base, char* err, size_t errlen) {
  std::vector<GenSpec> gs;
  std::vector<int64_t> vals;
  int64_t rec = 0, cb = 0;
  int rc = plan(specs, n, stream_samples >= 0, stream_samples, &gs, &vals, &rec, &cb, err, errlen);
  if (rc) return rc;
  if (n_records) *n_records = rec;
  if (n_class_base) *n_class_base = cb;
  return BFSIM_OK;
}

int bfsim_generate_traces(bfsim_ctx_t* ctx, const bfsim_gen_spec_t* specs, int32_t n, bfsim_request_t* traces_dev,
                          int64_t n_records, int32_t* class_base_dev, int64_t n_class_base,
                          bfsim_input_t* inputs_out, void* stream, char* err, size_t errlen) {
  return generate(ctx, specs, n, false, 0, traces_dev, n_records, class_base_dev, n_class_base, inputs_out, stream,
                  err, errlen);
}

int bfsim_generate_streams(bfsim_ctx_t* ctx, const bfsim_gen_spec_t* specs, int32_t n, int64_t samples,
                           bfsim_sample_t* streams_dev, int64_t n_samples_cap, int32_t* class_base_dev,
                           int64_t n_class_base, bfsim_input_t* inputs_out, void* stream, char* err,
                           size_t errlen) {
  return generate(ctx, specs, n, true, samples, streams_dev, n_samples_cap, class_base_dev, n_class_base, inputs_out,
                  stream, err, errlen);
}

// The host twin of the device log (libm_log.cuh), for the tests that pin it to
// glibc.
void bfsim_libm_log_host(const double* x, double* y, int64_t n) {
  static const bfsim::libm::LogEntry tab[128] = {BFSIM_LOG_TAB};
  for (int64_t i = 0; i < n; ++i) y[i] = bfsim::libm::log(x[i], tab);
}

}  // extern "C"
