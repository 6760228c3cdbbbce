// glibc's natural log, bit for bit, on the device and the host.
//
// The reference's synthetic traces come from libstdc++ distributions that call
// glibc's `log`: exponential_distribution (-log(1 - U) / rate, the Poisson
// gaps of sample_instance, workload.hpp:252-263) and geometric_distribution
// (floor(log(1 - U) / log(1 - p)), DecodeDistribution::sample
// workload.hpp:198). CUDA's `log` is within 1 ulp of glibc's but not
// identical, so a device generator built on it would drift from the
// reference's traces. This is glibc 2.39's x86-64 `__log_fma` -- the variant
// its ifunc selects on FMA+AVX2 hosts, i.e. what the reference's `log` runs on
// this image and on the GPU boxes -- restated instruction for instruction from
// its disassembly: every fused multiply-add the compiler formed there is an
// explicit fma here, every other operation is a separately rounded add / sub /
// mul (no contraction). The constants are glibc's `__log_data`
// (libm_log_table.h, extracted by tools/gen_libm_log.py). Pinned against the
// host's glibc on random and structured inputs by tests/test_libm_log.py.
#pragma once

#include <cstdint>
#include <cstring>

#include "libm_log_table.h"

#ifdef __CUDACC__
#define BFSIM_HD __host__ __device__ __forceinline__
#else
#define BFSIM_HD inline
#include <cmath>
#endif

namespace bfsim {
namespace libm {

struct LogEntry {
  double invc, logc;
};

#ifdef __CUDA_ARCH__
#define LM_ADD(a, b) __dadd_rn(a, b)
#define LM_SUB(a, b) __dsub_rn(a, b)
#define LM_MUL(a, b) __dmul_rn(a, b)
#define LM_FMA(a, b, c) __fma_rn(a, b, c)
#define LM_BITS(x) static_cast<uint64_t>(__double_as_longlong(x))
#define LM_DBL(u) __longlong_as_double(static_cast<long long>(u))
#else
#define LM_ADD(a, b) ((a) + (b))
#define LM_SUB(a, b) ((a) - (b))
#define LM_MUL(a, b) ((a) * (b))
#define LM_FMA(a, b, c) std::fma(a, b, c)
BFSIM_HD uint64_t lm_bits_host(double x) {
  uint64_t u;
  std::memcpy(&u, &x, 8);
  return u;
}
BFSIM_HD double lm_dbl_host(uint64_t u) {
  double x;
  std::memcpy(&x, &u, 8);
  return x;
}
#define LM_BITS(x) lm_bits_host(x)
#define LM_DBL(u) lm_dbl_host(u)
#endif

// `tab` = the 128 {invc, logc} entries (BFSIM_LOG_TAB), wherever the caller
// staged them (shared memory in the kernels).
BFSIM_HD double log(double x, const LogEntry* tab) {
  uint64_t ix = LM_BITS(x);
  // |x - 1| < ~0.0625: the log1p-style polynomial (glibc's LO/HI window)
  if (ix - 0x3fee000000000000ull < 0x3090000000000ull) {
    if (ix == 0x3ff0000000000000ull) return 0.0;
    const double r = LM_SUB(x, 1.0);
    const double r2 = LM_MUL(r, r);
    const double r3 = LM_MUL(r, r2);
    double p1 = LM_FMA(r, BFSIM_LOG_B2, BFSIM_LOG_B1);
    double p2 = LM_FMA(r, BFSIM_LOG_B5, BFSIM_LOG_B4);
    double q = LM_FMA(r, BFSIM_LOG_B8, BFSIM_LOG_B7);
    p1 = LM_FMA(r2, BFSIM_LOG_B3, p1);
    p2 = LM_FMA(r2, BFSIM_LOG_B6, p2);
    q = LM_FMA(r2, BFSIM_LOG_B9, q);
    q = LM_FMA(r3, BFSIM_LOG_B10, q);
    q = LM_FMA(q, r3, p2);
    q = LM_FMA(q, r3, p1);
    // rhi = r + w - w with w = r * 2^27 (both steps fused)
    const double t = LM_FMA(r, 0x1p27, r);
    const double rhi = LM_FMA(-r, 0x1p27, t);
    const double rhi2 = LM_MUL(rhi, rhi);
    const double rlo = LM_SUB(r, rhi);
    const double hi = LM_FMA(rhi2, BFSIM_LOG_B0, r);
    double lo = LM_FMA(rhi2, BFSIM_LOG_B0, LM_SUB(r, hi));
    lo = LM_FMA(LM_MUL(BFSIM_LOG_B0, rlo), LM_ADD(r, rhi), lo);
    return LM_ADD(hi, LM_FMA(q, r3, lo));
  }
  const uint32_t top = static_cast<uint32_t>(ix >> 48);
  if (top - 0x0010u > 0x7fdfu) {  // subnormal, zero, negative, inf, nan
    if ((ix << 1) == 0) return -__builtin_inf();
    if (ix == 0x7ff0000000000000ull) return x;
    if ((top & 0x8000u) || (top & 0x7ff0u) == 0x7ff0u) return __builtin_nan("");
    ix = LM_BITS(LM_MUL(x, 0x1p52)) - (52ull << 52);  // normalize a subnormal
  }
  const uint64_t tmp = ix - 0x3fe6000000000000ull;
  const int i = static_cast<int>((tmp >> 45) & 127u);
  const int k = static_cast<int>(static_cast<int64_t>(tmp) >> 52);
  const uint64_t iz = ix - (tmp & 0xfff0000000000000ull);
  const double invc = tab[i].invc, logc = tab[i].logc;
  const double z = LM_DBL(iz);
  const double kd = static_cast<double>(k);
  const double w = LM_FMA(kd, BFSIM_LOG_LN2HI, logc);
  const double r = LM_FMA(z, invc, -1.0);
  const double p21 = LM_FMA(r, BFSIM_LOG_A2, BFSIM_LOG_A1);
  const double hi = LM_ADD(r, w);
  const double r2 = LM_MUL(r, r);
  double lo = LM_ADD(LM_SUB(w, hi), r);
  lo = LM_FMA(kd, BFSIM_LOG_LN2LO, lo);
  const double r3 = LM_MUL(r, r2);
  const double p43 = LM_FMA(r, BFSIM_LOG_A4, BFSIM_LOG_A3);
  lo = LM_FMA(r2, BFSIM_LOG_A0, lo);
  const double p = LM_FMA(p43, r2, p21);
  return LM_ADD(LM_FMA(r3, p, lo), hi);
}

}  // namespace libm
}  // namespace bfsim
