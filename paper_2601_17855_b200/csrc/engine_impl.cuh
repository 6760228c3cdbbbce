#pragma once
// B200 (sm_100a) batched step engine for the BF-IO hot path.
//
// One warp simulates one trajectory (scenario) end to end; persistent CTAs of
// one warp pull scenarios from an atomic queue. Worker g is owned by lane
// g % 32 (slot j = g / 32 of WPL register-resident workers per lane), so
// per-worker state (active count, load aggregate) lives in registers and every
// per-worker update is lane-local. Per-slot, per-class and lookahead-window
// state lives in the warp's shared-memory arena (SM = true: 32-bit LDS/STS);
// the per-prefill-class waiting deques live in a per-warp global workspace
// (L2-resident) and the records an admission needs are prefetched into shared
// memory with cp.async while the sequential placement chain runs.
//
// Reference semantics (paths under /root/reference/proj/include/bfsim/):
//   step order            engine.hpp:112-160 (Poisson), oracle.hpp:163-242 (overloaded)
//   reveal                engine.hpp:123-128
//   fcfs / jsq            policies.hpp:100-138   -> closed-form level filling
//   bfio-greedy           policies.hpp:269-370   -> class-deque water filling (F4)
//                                                   + warp-argmin placement (F3)
//   loads / dt / clock    engine.hpp:136-146 (dt = C (+) t (x) max, no FMA: F6)
//   completion            engine.hpp:149-157, 118-120; oracle.hpp:225-240
//   accounting            metrics.hpp:17-126, metrics_power.hpp:24-27
#include <cuda_runtime.h>

#include <climits>
#include <cstdint>
#include <type_traits>

#include "engine.cuh"

// Template implementation of the step kernel; instantiated per (mode, policy)
// in engine_<mode>_<policy>.cu so the variants compile in parallel.

namespace bfsim {
namespace detail {

#define FULLMASK 0xffffffffu
// Loops over a lane's WPL workers: unrolled into registers up to 8 workers per
// lane; above that (G > 256) the per-lane arrays live in L1-cached local memory.
#define BFSIM_UNROLL_W _Pragma("unroll (WPL > 8 ? 1 : WPL)")

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

__device__ __forceinline__ uint64_t wmin_u64(uint64_t v) {
  uint32_t hi = __reduce_min_sync(FULLMASK, static_cast<uint32_t>(v >> 32));
  uint32_t lo = __reduce_min_sync(
      FULLMASK, static_cast<uint32_t>(v >> 32) == hi ? static_cast<uint32_t>(v) : 0xFFFFFFFFu);
  return (static_cast<uint64_t>(hi) << 32) | lo;
}

// warp argmin of packed (value << gbits | g) keys; K32: every key fits 31 bits
template <bool K32>
__device__ __forceinline__ uint64_t argmin_key(uint64_t key) {
  if constexpr (K32) {
    return static_cast<uint64_t>(__reduce_min_sync(FULLMASK, static_cast<uint32_t>(key)));
  } else {
    return wmin_u64(key);
  }
}

__device__ __forceinline__ long long wsum_i64(long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULLMASK, v, o);
  return v;
}

__device__ __forceinline__ double wsum_f64(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = __dadd_rn(v, __shfl_xor_sync(FULLMASK, v, o));
  return v;
}

__device__ __forceinline__ int bits_for(long long x) {  // bits to hold values 0..x
  return x <= 0 ? 0 : 64 - __clzll(static_cast<unsigned long long>(x));
}

__device__ __forceinline__ void cp_async8(void* smem_dst, const void* gsrc) {
  unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem_dst));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.wait_all;\n" ::: "memory");
}

// ---------------------------------------------------------------------------
// libstdc++ std::mt19937_64 (bits/random.h parameters) and the draws
// make_preview takes from it in Noisy mode (policies.hpp:74-76):
// normal_distribution<double>(0, sigma) -- polar method, a fresh object per
// call (random.tcc:1809-1844) -- over generate_canonical<double, 53>, which is
// one engine call for a 64-bit engine (random.tcc:3349-3381). Every rounding
// step is spelled out with _rn intrinsics so nothing is FMA-contracted
// (the reference build: -ffp-contract=off).
constexpr int kMtN = 312, kMtM = 156;
constexpr uint64_t kMtA = 0xB5026F5AA96619E9ull;
constexpr uint64_t kMtUpper = 0xFFFFFFFF80000000ull, kMtLower = 0x000000007FFFFFFFull;

__device__ __forceinline__ uint64_t mt_temper(uint64_t y) {
  y ^= (y >> 29) & 0x5555555555555555ull;
  y ^= (y << 17) & 0x71D67FFFEDA60000ull;
  y ^= (y << 37) & 0xFFF7EEE000000000ull;
  y ^= y >> 43;
  return y;
}

__device__ __forceinline__ uint64_t mt_mix(uint64_t lo_word, uint64_t next, uint64_t far) {
  const uint64_t x = (lo_word & kMtUpper) | (next & kMtLower);
  return far ^ (x >> 1) ^ ((x & 1ull) ? kMtA : 0ull);
}

// mersenne_twister_engine::seed: a 311-step sequential recurrence (lane 0).
__device__ __forceinline__ void mt_seed(uint64_t* mt, uint64_t seed) {
  if ((threadIdx.x & 31) == 0) {
    uint64_t x = seed;
    mt[0] = x;
    for (int i = 1; i < kMtN; ++i) {
      x = 6364136223846793005ull * (x ^ (x >> 62)) + static_cast<uint64_t>(i);
      mt[i] = x;
    }
  }
  __syncwarp();
}

// _M_gen_rand, warp-parallel. The sequential loop reads, for i < 156, only
// words not yet rewritten (i+1, i+156); for 156 <= i < 311 the rewritten word
// i-156 and the old word i+1; i = 311 reads the rewritten words 155 and 0.
// So two parallel halves reproduce it exactly (reads of a 32-wide chunk are
// fenced from its writes by __syncwarp).
__device__ __forceinline__ void mt_twist(uint64_t* mt) {
  const int lane = threadIdx.x & 31;
  uint64_t v[5];
#pragma unroll
  for (int t = 0; t < 5; ++t) {  // i < 156: all reads before any write
    const int i = lane + 32 * t;
    v[t] = i < kMtM ? mt_mix(mt[i], mt[i + 1], mt[i + kMtM]) : 0ull;
  }
  __syncwarp();
#pragma unroll
  for (int t = 0; t < 5; ++t)
    if (lane + 32 * t < kMtM) mt[lane + 32 * t] = v[t];
  __syncwarp();
#pragma unroll
  for (int t = 0; t < 5; ++t) {  // 156 <= i < 312
    const int i = kMtM + lane + 32 * t;
    v[t] = i < kMtN ? mt_mix(mt[i], mt[i + 1 < kMtN ? i + 1 : 0], mt[i - kMtM]) : 0ull;
  }
  __syncwarp();
#pragma unroll
  for (int t = 0; t < 5; ++t)
    if (kMtM + lane + 32 * t < kMtN) mt[kMtM + lane + 32 * t] = v[t];
  __syncwarp();
}

// generate_canonical<double, 53>: (double)u / 2^64, clamped below 1.
__device__ __forceinline__ double mt_canonical(uint64_t u) {
  const double r = __dmul_rn(__ull2double_rn(u), 0x1p-64);
  return r >= 1.0 ? 0x1.fffffffffffffp-1 : r;
}

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.cta.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(unsigned* p, unsigned v) {
  asm volatile("st.release.cta.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// L2 residency hints for the noisy per-worker lists (read and rewritten every
// step, ~32 KB per trajectory in the global workspace): evict_last keeps them
// in L2 ahead of the streaming data (deques, traces, draw scratch)
__device__ __forceinline__ uint64_t l2_keep_policy() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ int2 ld_keep(const int2* ptr, uint64_t pol) {
  int2 v;
  asm volatile("ld.global.L2::cache_hint.v2.s32 {%0, %1}, [%2], %3;" : "=r"(v.x), "=r"(v.y) : "l"(ptr), "l"(pol));
  return v;
}
__device__ __forceinline__ void st_keep(int2* ptr, int2 v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.v2.s32 [%0], {%1, %2}, %3;" ::"l"(ptr), "r"(v.x), "r"(v.y), "l"(pol)
               : "memory");
}

// Noisy lookahead draw stream (make_preview, policies.hpp:74-76). Every step
// the reference draws normal_distribution(0, sigma) values from the
// simulation's mt19937_64 -- one per active request, then one per waiting
// request (engine.hpp:131, 204-231) -- with a fresh distribution object per
// call, so draw i of the trajectory is the i-th accepted polar pair of the
// engine stream (random.tcc:1809-1844), independent of how draws are split
// into steps. A producer warp generates that stream ahead of the simulation
// warp: lround(N(0, sigma)) of every accepted pair, clamped to +-2^29 (exact
// for the previews: decode lengths are < 2^28), stored as 2 v + (near-tie
// flag) in a shared-memory ring of kRing entries. ctr[0] = draws produced,
// ctr[1] = draws the consumer has released, ctr[2] = trajectory finished.
constexpr int kRing = 2048;

// lround(y * sqrt(-2 ln r2 / r2) * sigma) for an accepted pair, and whether it
// lies next to a half-integer (CUDA log is within 1 ulp of glibc's). A float
// estimate decides it unless the value lies within 1e-5 (relative) of a
// half-integer: its error is below 1e-6 relative (-ln r2 as -log1pf(r2 - 1),
// r2 - 1 exact in double, or -logf(r2), each within 1 ulp and ~2.2 ulp after
// the input rounding, then IEEE division, sqrt and products, no fast-math:
// ~10 ulp of 2^-24 in all). Those rare draws take the reference's
// double-precision formula, every step spelled with _rn (no FMA).
__device__ __forceinline__ int normal_code(double y, double r2, double sigma, float sf) {
  const float r2f = static_cast<float>(r2);
  const float L = r2 < 0.25 ? -logf(r2f) : -log1pf(static_cast<float>(r2 - 1.0));
  const float nf = static_cast<float>(y) * sqrtf(2.0f * L / r2f) * sf;
  const float af = fabsf(nf);
  long long l;
  int tie = 0;
  if (af < 1048576.0f && fabsf((af - floorf(af)) - 0.5f) > 1e-5f * fmaxf(1.0f, af)) {
    l = static_cast<long long>(lroundf(nf));
  } else {
    const double mult = __dsqrt_rn(__ddiv_rn(__dmul_rn(-2.0, log(r2)), r2));
    const double nv = __dadd_rn(__dmul_rn(__dmul_rn(y, mult), sigma), 0.0);
    l = llround(nv);
    const double av = fabs(nv);
    tie = fabs(__dsub_rn(av, floor(av)) - 0.5) <= 1e-12 * fmax(1.0, av) ? 1 : 0;
  }
  l = l > (1ll << 29) ? (1ll << 29) : (l < -(1ll << 29) ? -(1ll << 29) : l);
  return static_cast<int>(2 * l + tie);
}

static __device__ void noisy_producer(uint64_t* mt, int* ring, unsigned* ctr, uint64_t seed, double sigma) {
  const int lane = threadIdx.x & 31;
  const float sf = static_cast<float>(sigma);
  mt_seed(mt, seed);  // Simulation::rng_(config.seed), engine.hpp:97-98
  int mt_i = kMtN;
  unsigned prod = 0;
  for (;;) {
    // room for one slice (<= 32 draws) behind the consumer's release
    for (;;) {
      const unsigned rel = ld_acquire(&ctr[1]);
      if (static_cast<int>(prod - rel) <= kRing - 32) break;
      if (ld_acquire(&ctr[2])) return;
      __nanosleep(256);  // the consumer is behind: stay off the issue slots
    }
    if (ld_acquire(&ctr[2])) return;
    if (mt_i >= kMtN) {
      mt_twist(mt);
      mt_i = 0;
    }
    const int np = (kMtN - mt_i) >> 1;  // pairs left in the block
    const bool valid = lane < np;
    const int pi = mt_i + 2 * (valid ? lane : 0);
    const double u1 = mt_canonical(mt_temper(mt[pi]));
    const double u2 = mt_canonical(mt_temper(mt[pi + 1]));
    const double x = __dsub_rn(__dmul_rn(2.0, u1), 1.0);
    const double y = __dsub_rn(__dmul_rn(2.0, u2), 1.0);
    const double r2 = __dadd_rn(__dmul_rn(x, x), __dmul_rn(y, y));
    const bool acc = valid && !(r2 > 1.0 || r2 == 0.0);
    const unsigned am = __ballot_sync(FULLMASK, acc);
    if (acc) ring[(prod + __popc(am & lanemask_lt())) & (kRing - 1)] = normal_code(y, r2, sigma, sf);
    __threadfence_block();
    __syncwarp();
    prod += __popc(am);
    mt_i += 2 * (np < 32 ? np : 32);
    if (lane == 0) st_release(&ctr[0], prod);
  }
}

// Array placement from the planner. SM: every code is a shared-memory offset,
// so the compiler emits 32-bit shared loads/stores. Otherwise a code < 0 is
// byte (-code - 1) of the warp's global workspace.
template <bool SM, class T>
__device__ __forceinline__ T* at(unsigned char* sm, unsigned char* ws, int64_t code) {
  if constexpr (SM) {
    return reinterpret_cast<T*>(sm + code);
  } else {
    return code >= 0 ? reinterpret_cast<T*>(sm + code) : reinterpret_cast<T*>(ws + (-code - 1));
  }
}

// Cold arrays always live in the global workspace (code < 0).
template <class T>
__device__ __forceinline__ T* gat(unsigned char* ws, int64_t code) {
  return reinterpret_cast<T*>(ws + (-code - 1));
}

// ---------------------------------------------------------------------------
// Set of non-empty prefill classes c = 1..S (bit c-1). SMALL: S <= 64 in one
// uniform register word. Otherwise a 3-level 64-ary bitmap (top word in a
// register, mid/leaf words in memory). Every operation is executed uniformly
// by all lanes; stores write the same value from every lane, so a lane's later
// load sees its own store without a warp barrier.
template <bool SMALL>
struct ClassSet;

template <>
struct ClassSet<true> {
  uint64_t bits;
  __device__ void init(uint64_t*, uint64_t*, int) { bits = 0; }
  __device__ bool empty() const { return bits == 0; }
  __device__ int highest() const { return bits ? 64 - __clzll(bits) : 0; }
  __device__ int lowest() const { return bits ? __ffsll(static_cast<long long>(bits)) : 0; }
  __device__ int highest_le(long long d) const {
    // classes 1..d are bits 0..d-1: shift them to the top, the rest falls off
    if (d >= 64) return highest();
    const uint64_t m = d < 1 ? 0ull : bits << (64 - static_cast<int>(d));
    return m ? static_cast<int>(d) - __clzll(m) : 0;
  }
  __device__ void clear(int c) { bits &= ~(1ull << (c - 1)); }
  __device__ void add_from_lanes(bool has, int c) {
    uint64_t m = has ? (1ull << (c - 1)) : 0ull;
    uint32_t lo = __reduce_or_sync(FULLMASK, static_cast<uint32_t>(m));
    uint32_t hi = __reduce_or_sync(FULLMASK, static_cast<uint32_t>(m >> 32));
    bits |= (static_cast<uint64_t>(hi) << 32) | lo;
  }
  __device__ void add_uniform(int c) { bits |= 1ull << (c - 1); }
  __device__ void clear_all() { bits = 0; }
};

template <>
struct ClassSet<false> {
  uint64_t top;    // bit m: mid word m non-empty
  uint64_t* mid;   // 64 words; bit w: leaf word w non-empty
  uint64_t* leaf;  // ceil(S/64) words; bit b: class b+1 present
  int nbits;       // S
  __device__ void init(uint64_t* mid_, uint64_t* leaf_, int S) {
    mid = mid_;
    leaf = leaf_;
    nbits = S;
    top = 0;
    const int lane = threadIdx.x & 31;
    int nl = (S + 63) >> 6;
    for (int i = lane; i < nl; i += 32) leaf[i] = 0;
    for (int i = lane; i < 64; i += 32) mid[i] = 0;
    __syncwarp();
  }
  __device__ bool empty() const { return top == 0; }
  __device__ static uint64_t mask_le(int b) {  // bits 0..b
    return b >= 63 ? ~0ull : ((1ull << (b + 1)) - 1ull);
  }
  __device__ int from_top(uint64_t m2) const {  // highest class under top mask m2
    int mw = 63 - __clzll(m2);
    int lw = (mw << 6) + 63 - __clzll(mid[mw]);
    return (lw << 6) + 63 - __clzll(leaf[lw]) + 1;
  }
  __device__ int highest() const { return top ? from_top(top) : 0; }
  __device__ int lowest() const {
    if (!top) return 0;
    int mw = __ffsll(static_cast<long long>(top)) - 1;
    int lw = (mw << 6) + __ffsll(static_cast<long long>(mid[mw])) - 1;
    return (lw << 6) + __ffsll(static_cast<long long>(leaf[lw]));
  }
  // largest class c <= d, 0 if none
  __device__ int highest_le(long long d) const {
    if (d < 1 || !top) return 0;
    long long q = d - 1;
    if (q > nbits - 1) q = nbits - 1;
    const int w0 = static_cast<int>(q >> 6);
    const int mw0 = w0 >> 6;
    if ((top >> mw0) & 1ull) {
      uint64_t lm = leaf[w0] & mask_le(static_cast<int>(q & 63));
      if (lm) return (w0 << 6) + 63 - __clzll(lm) + 1;
      if (w0 & 63) {
        uint64_t mm = mid[mw0] & mask_le((w0 & 63) - 1);
        if (mm) {
          int lw = (mw0 << 6) + 63 - __clzll(mm);
          return (lw << 6) + 63 - __clzll(leaf[lw]) + 1;
        }
      }
    }
    if (mw0 == 0) return 0;
    uint64_t tm = top & mask_le(mw0 - 1);
    return tm ? from_top(tm) : 0;
  }
  __device__ void clear(int c) {
    int b = c - 1, w = b >> 6;
    uint64_t lw = leaf[w] & ~(1ull << (b & 63));
    leaf[w] = lw;
    if (lw == 0) {
      uint64_t m2 = mid[w >> 6] & ~(1ull << (w & 63));
      mid[w >> 6] = m2;
      if (m2 == 0) top &= ~(1ull << (w >> 6));
    }
  }
  __device__ void add_from_lanes(bool has, int c) {
    uint64_t tb = 0;
    __syncwarp();
    if (has) {
      int b = c - 1, w = b >> 6;
      atomicOr(reinterpret_cast<unsigned long long*>(&leaf[w]), 1ull << (b & 63));
      atomicOr(reinterpret_cast<unsigned long long*>(&mid[w >> 6]), 1ull << (w & 63));
      tb = 1ull << (w >> 6);
    }
    uint32_t lo = __reduce_or_sync(FULLMASK, static_cast<uint32_t>(tb));
    uint32_t hi = __reduce_or_sync(FULLMASK, static_cast<uint32_t>(tb >> 32));
    top |= (static_cast<uint64_t>(hi) << 32) | lo;
    __syncwarp();
  }
  __device__ void add_uniform(int c) {
    int b = c - 1, w = b >> 6;
    leaf[w] |= 1ull << (b & 63);
    mid[w >> 6] |= 1ull << (w & 63);
    top |= 1ull << (w >> 6);
  }
};

// ---------------------------------------------------------------------------


// ---------------------------------------------------------------------------
// Wide trajectories (bfio-greedy with a lookahead window on G > 128 workers,
// BASELINE C4's G = 256..1024; SURVEY hard part 3): the trajectory's CTA has
// W = ceil(G / 128) warps. Warp 0 runs the step loop; for the placement chain
// (phase 2, policies.hpp:339-367) it hands the items to all W warps, which
// split the workers (thread t: workers t, t + 32 W, ...; at most 4 each).
// The views F_h[g] and maxima M_h are int32 rows in shared memory (every load
// is below 2^31: validate_scenario); costs are summed in 64 bits.
struct WideChain {
  int cmd;  // 1: run the chain below, 0: the trajectory is done
  int U, H, G, gbits, Hm, trunc;
  long long k, d, ak;
  // byte offsets of core arrays in the CTA's dynamic shared memory (the
  // trajectory's arena starts at 0): views F [h][g] (int32), maxima M and
  // per-item T_h = M_h - w_h (int32), free slots, admissions, admitted workload
  int F, M, cap, admc, asum;
  const int32_t* o_c;
  const int32_t* o_o;
  uint32_t* res;
  int32_t* Wc;
  long long* Wa;
};

extern __shared__ __align__(16) unsigned char bfsim_dsmem[];

// Named barrier 1 over the CTA's nthreads (warp-converged first: bar.sync is
// the .aligned form).
__device__ __forceinline__ void cta_bar(int nthreads) {
  __syncwarp();
  asm volatile("barrier.sync 1, %0;" ::"r"(nthreads) : "memory");
}

// Per item: the fast-path candidate g* = argmin (F_0[g], g) over free
// workers (per-warp minima exchanged in shared memory); when no horizon of
// g* would rise above the current maximum it wins outright (its cost is the
// minimum sum_h M_h and its tie-break key the smallest). Otherwise every
// thread scores its workers, cost = sum_h max(M_h - w_h, F_h[g]) (the
// reference's sum_h max(M_h, F_h[g] + w_h) less sum_h w_h, which does not
// depend on g: same argmin and ties over (cost, F_0, g)), and the per-warp
// best (cost, F_0, g) are exchanged again. Threads over h then add w_h to the
// chosen row and raise M_h; the owner books the admission.
static __device__ __forceinline__ void wide_chain(const WideChain& wsh, unsigned long long (*red)[2], int nthreads) {
  // a private copy: once the chain's last barrier is passed, warp 0 may
  // already be writing the next chain's parameters
  const WideChain w = wsh;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5, nw = nthreads >> 5;
  const int G = w.G, H = w.H, gbits = w.gbits;
  const long long d = w.d;
  // core arrays addressed in the shared window (32-bit shared loads)
  int32_t* F = reinterpret_cast<int32_t*>(bfsim_dsmem + w.F);
  int32_t* M = reinterpret_cast<int32_t*>(bfsim_dsmem + w.M);
  int32_t* Tsh = M + (H + 1);
  int32_t* cap = reinterpret_cast<int32_t*>(bfsim_dsmem + w.cap);
  int32_t* admc = reinterpret_cast<int32_t*>(bfsim_dsmem + w.admc);
  unsigned long long* asum = reinterpret_cast<unsigned long long*>(bfsim_dsmem + w.asum);
  const uint64_t gmask = (1ull << gbits) - 1ull;
  for (int h = warp; h <= H; h += nw) {  // M_h = max over every worker
    int32_t m = 0;
    for (int g = lane; g < G; g += 32) m = F[h * G + g] > m ? F[h * G + g] : m;
    m = static_cast<int32_t>(__reduce_max_sync(FULLMASK, static_cast<uint32_t>(m)));
    if (lane == 0) M[h] = m;
  }
  cta_bar(nthreads);
  for (int q = 0; q < w.U; ++q) {
    const int c = w.o_c[q], o = w.o_o[q];
    const long long lim = (w.trunc && o < H + 1) ? H + 1 : o;
    const int limH = static_cast<int>(lim < H + 1 ? lim : H + 1);
    const long long sat = d * (o - 1);
    uint64_t fk = ~0ull;
    for (int g = t; g < G; g += nthreads)
      if (cap[g] > 0) {
        const uint64_t kk = (static_cast<uint64_t>(static_cast<uint32_t>(F[g])) << gbits) | static_cast<uint64_t>(g);
        fk = kk < fk ? kk : fk;
      }
    fk = wmin_u64(fk);
    if (lane == 0) red[warp][0] = fk;
    cta_bar(nthreads);
    uint64_t best = ~0ull;
    for (int i = 0; i < nw; ++i) best = red[i][0] < best ? red[i][0] : best;
    int gs = static_cast<int>(best & gmask);
    // thread t checks (and below updates) horizons t, t + nthreads, ...: no
    // thread reads a row entry another thread writes in this item
    bool over = false;
    for (int h = t; h <= H; h += nthreads) {
      const long long wh = h < limH ? c + (d * h < sat ? d * h : sat) : 0;
      over = over || F[h * G + gs] + wh > M[h];
      Tsh[h] = static_cast<int32_t>(M[h] - wh);  // for the full scan
    }
    const unsigned ow = __ballot_sync(FULLMASK, over);
    if (lane == 0) red[warp][1] = ow;
    cta_bar(nthreads);
    unsigned long long anyo = 0;
    for (int i = 0; i < nw; ++i) anyo |= red[i][1];
    if (anyo) {  // the same outcome in every warp
      long long cost[4] = {0, 0, 0, 0};
      const int32_t* col = F + t;
      for (int h = 0; h <= H; ++h, col += G) {
        const int32_t T = Tsh[h];
#pragma unroll
        for (int j = 0; j < 4; ++j)
          if (t + j * nthreads < G) {
            const int32_t f = col[j * nthreads];
            cost[j] += T > f ? T : f;
          }
      }
      uint64_t bc = ~0ull, bk = ~0ull;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int g = t + j * nthreads;
        if (g < G && cap[g] > 0) {
          const uint64_t c64 = static_cast<uint64_t>(cost[j]);
          const uint64_t k2 = (static_cast<uint64_t>(static_cast<uint32_t>(F[g])) << gbits) | static_cast<uint64_t>(g);
          if (c64 < bc || (c64 == bc && k2 < bk)) {
            bc = c64;
            bk = k2;
          }
        }
      }
      const uint64_t cmin = wmin_u64(bc);
      const uint64_t kmin = wmin_u64(bc == cmin ? bk : ~0ull);
      cta_bar(nthreads);  // every thread has read red[][] above
      if (lane == 0) {
        red[warp][0] = cmin;
        red[warp][1] = kmin;
      }
      cta_bar(nthreads);
      uint64_t c2 = ~0ull, k2 = ~0ull;
      for (int i = 0; i < nw; ++i)
        if (red[i][0] < c2 || (red[i][0] == c2 && red[i][1] < k2)) {
          c2 = red[i][0];
          k2 = red[i][1];
        }
      gs = static_cast<int>(k2 & gmask);
    }
    for (int h = t; h <= H; h += nthreads) {
      const long long wh = h < limH ? c + (d * h < sat ? d * h : sat) : 0;
      const int32_t v = static_cast<int32_t>(F[h * G + gs] + wh);
      F[h * G + gs] = v;
      if (v > M[h]) M[h] = v;
    }
    if (t == gs % nthreads) {
      const int rank = admc[gs];
      admc[gs] = rank + 1;
      cap[gs] -= 1;
      asum[gs] += static_cast<unsigned long long>(c + w.ak);
      w.res[q] = static_cast<uint32_t>(gs) | (static_cast<uint32_t>(rank) << 16);
      if (o <= H) {  // finishes inside the window [k, k+H-1]
        const int r = static_cast<int>((w.k + o - 1) % w.Hm);
        w.Wc[r * G + gs] += 1;
        w.Wa[r * G + gs] += c + w.ak;
      }
    }
    cta_bar(nthreads);
  }
}

// ---------------------------------------------------------------------------
template <int MODE, int POL, int WPL, bool SMALLC, bool SM, bool NOISY, int HR, bool WIDE = false>
__device__ void run_traj(const KParams& P, int si, unsigned char* sm, unsigned char* ws, WideChain* wctl = nullptr,
                         unsigned long long (*wred)[2] = nullptr) {
  constexpr bool OVL = MODE == BFSIM_MODE_OVERLOADED;
  constexpr bool GREEDY = POL == BFSIM_POLICY_BFIO_GREEDY;
  static_assert(!NOISY || (GREEDY && !OVL), "noisy lookahead: Poisson bfio-greedy only");
  static_assert(HR == 0 || (GREEDY && WPL <= 4), "register lookahead chain: bfio-greedy, G <= 128");
  constexpr bool JSQ = POL == BFSIM_POLICY_JSQ;
  const Plan& pl = P.plan;
  const int lane = threadIdx.x & 31;
  const bfsim_scenario_t sc = P.scen[si];
  const bfsim_input_t in = P.inputs[sc.input_id];
  const int G = sc.workers, B = sc.batch;
  const int H = GREEDY ? sc.horizon : 0;
  const int Hm = H > 0 ? H : 1;  // modulus for the window ring (unused when H == 0)
  // run_overloaded always previews perfectly (oracle.hpp:185-199)
  const bool trunc = !OVL && sc.lookahead == BFSIM_LOOKAHEAD_TRUNCATED;
  const long long d = static_cast<long long>(sc.drift);
  const int S = in.s_max;
  const long long N = in.length;
  const bfsim_request_t* tr = P.traces ? P.traces + in.offset : nullptr;
  const bfsim_sample_t* st = P.streams ? P.streams + in.offset : nullptr;
  const int32_t* cbase_g = P.class_base + in.class_base_offset;
  const double C0 = sc.overhead, TL = sc.per_token;
  // dyadic drift m / 2^e: the host scaled every workload by 2^e (and t_ell by
  // 2^-e, capi.cu scale_dyadic); loads leave the kernel scaled back, exactly
  const double lsc = sc.reserved0 > 0 ? ldexp(1.0, -sc.reserved0) : 1.0;
  const double p_idle = sc.p_idle, p_diff = sc.p_max - sc.p_idle, gam = sc.gamma;
  const long long warmup = OVL ? sc.warmup : 0;
  const long long total_steps =
      OVL ? sc.warmup + sc.steps : (sc.max_steps < INT_MAX - 2 ? sc.max_steps : INT_MAX - 2);
  const bool emit_steps = P.steps.clock_start != nullptr;
  const bool emit_reqs = P.reqs.start_step != nullptr;
  const long long so = sc.step_offset, scap = sc.step_capacity, lo = sc.load_offset;
  const long long ro = sc.req_offset;
  const int rstride = (G & 1) ? G : G + 1;  // padded accounting-ring row (bank conflicts)
  const int umax = pl.umax;
  const float invB = 1.0f / static_cast<float>(B);
  const int cbuf_cap = pl.cbuf;

  // --- arenas --------------------------------------------------------------
  uint32_t* s_f = at<SM, uint32_t>(sm, ws, pl.o_f);
  int32_t* s_a = at<SM, int32_t>(sm, ws, pl.o_a);
  int32_t* s_x = at<SM, int32_t>(sm, ws, pl.o_x);
  int32_t* s_id = at<SM, int32_t>(sm, ws, pl.o_id);
  uint16_t* s_stk = at<SM, uint16_t>(sm, ws, pl.o_stk);
  int32_t* s_capb = at<true, int32_t>(sm, ws, pl.o_capb);  // core arrays: always shared memory
  unsigned long long* s_asum = at<true, unsigned long long>(sm, ws, pl.o_asum);
  int32_t* s_admc = at<true, int32_t>(sm, ws, pl.o_admc);  // admissions per worker (int32 chain)
  int32_t* s_cap = at<true, int32_t>(sm, ws, pl.o_cap);
  uint32_t* r_l = at<SM, uint32_t>(sm, ws, pl.o_rl);
  double* r_dt = at<true, double>(sm, ws, pl.o_rdt);
  double* r_cs = at<true, double>(sm, ws, pl.o_rcs);
  uint32_t* r_mx = at<true, uint32_t>(sm, ws, pl.o_rmx);
  int32_t* r_ac = at<true, int32_t>(sm, ws, pl.o_rac);
  double* ring = gat<double>(ws, pl.o_ring);  // cold: global workspace (L1/L2)
  const int Rm = pl.R - 1;
  // per-class record {front, back, picks this step, deque base} + chain start
  int4* c_rec = at<SM || (GREEDY && SMALLC), int4>(sm, ws, pl.o_cls);
  int32_t* c_cs = reinterpret_cast<int32_t*>(c_rec + (pl.S + 2));
  int2* deq = gat<int2>(ws, pl.o_deq);
  int2* stage = at<SM, int2>(sm, ws, pl.o_stage);  // prefetched (id|s, o) records
  int32_t* p_cl = at<SM, int32_t>(sm, ws, pl.o_pcl);
  int32_t* p_t = at<SM, int32_t>(sm, ws, pl.o_pt);
  uint32_t* s_res = at<SM, uint32_t>(sm, ws, pl.o_res);
  int32_t* lvT = at<SM || !GREEDY, int32_t>(sm, ws, pl.o_lvT);
  int32_t* lvV = at<SM || !GREEDY, int32_t>(sm, ws, pl.o_lvV);
  int32_t* lvK = at<SM || !GREEDY, int32_t>(sm, ws, pl.o_lvK);
  uint32_t* lvM = at<SM || !GREEDY, uint32_t>(sm, ws, pl.o_lvM);
  long long* s_F = at<SM || (HR > 0) || WIDE, long long>(sm, ws, pl.o_F);
  // int32 chain (HR > 0): views F_h[g] worker-major, row g = F_0..F_{HP-1}
  // (zero past H), HP = the group's H + 1 rounded up to 4 words, so a lane
  // reads 4 horizons of its worker per 128-bit load (capi.cu
  // chain_rows_bytes). The wide chain keeps [h][g].
  const int HP = (pl.H + 4) & ~3;
  constexpr int HP4MAX = HR > 8 ? 6 : 2;  // H < HR
  long long* s_M = at<SM || GREEDY, long long>(sm, ws, pl.o_M);
  int32_t* s_Wc = at<SM || NOISY, int32_t>(sm, ws, pl.o_Wc);
  long long* s_Wa = at<SM || NOISY, long long>(sm, ws, pl.o_Wa);
  int32_t* o_c = at<SM, int32_t>(sm, ws, pl.o_oc);
  int2* cbuf = gat<int2>(ws, pl.o_cbuf);  // cold: completions (x, finish step) for TPOT
  int32_t* s_misc = at<true, int32_t>(sm, ws, pl.o_misc);  // [0] completion-buffer fill
  int32_t* o_o = at<SM, int32_t>(sm, ws, pl.o_oo);
  int32_t* o_id = at<SM, int32_t>(sm, ws, pl.o_oid);
  uint64_t* s_key = (GREEDY && WPL >= 16) ? at<SM, uint64_t>(sm, ws, pl.o_key) : nullptr;
  // Completion calendar (large G*B): bucket f mod R holds, per owner lane
  // (g mod 32), a linked list of the slots finishing at step f.
  // cal 1 (G*B > 4096): bucket f mod R exactly, in the global workspace.
  // cal 2 (small G*B): a 64-bucket wheel in shared memory, bucket f mod 64;
  // an entry is retired when its bucket comes round at its finish step.
  const int cal = pl.cal;
  constexpr int kWheel = 64;
  const int LS = G < 32 ? G : 32;  // lanes that own workers (wheel row stride)
  int32_t* calh = cal == 1 ? gat<int32_t>(ws, pl.o_calh) : (cal == 2 ? at<SM, int32_t>(sm, ws, pl.o_calh) : nullptr);
  int32_t* calnx = cal == 1 ? gat<int32_t>(ws, pl.o_calnx) : nullptr;
  uint16_t* wnx = cal == 2 ? at<SM, uint16_t>(sm, ws, pl.o_calnx) : nullptr;
  // Noisy lookahead (NOISY): engine state; per-worker active lists in
  // insertion order, worker-major ([g * B + pos]), whose entries carry the
  // request's {finish step, a} so the draw pass reads them coalesced in draw
  // order, plus the ids of a step's appended entries (sort key); the
  // exclusive prefix of the active counts over workers (draw r -> worker);
  // difference arrays over h in int32 (shared-memory atomics); per-item
  // draws; the admitted waiting draws and the admitted-id bitmap that gives
  // waiting ranks.
  int* s_ring = NOISY ? at<true, int>(sm, ws, pl.o_nring) : nullptr;  // the producer warp's draws
  unsigned* s_ctr = NOISY ? at<true, unsigned>(sm, ws, pl.o_misc) + 1 : nullptr;
  int2* s_E = NOISY ? gat<int2>(ws, pl.o_lst) : nullptr;
  const uint64_t lkeep = NOISY ? l2_keep_policy() : 0;
  int32_t* s_Eid = NOISY ? gat<int32_t>(ws, pl.o_eid) : nullptr;
  int32_t* s_len = NOISY ? at<true, int32_t>(sm, ws, pl.o_pre) : nullptr;  // noisy: per-worker list lengths
  int32_t* n_Wa = NOISY ? reinterpret_cast<int32_t*>(s_Wa) : nullptr;
  int32_t* o_nz = NOISY ? at<SM, int32_t>(sm, ws, pl.o_onz) : nullptr;
  int32_t* nzb = NOISY ? gat<int32_t>(ws, pl.o_nzb) : nullptr;
  unsigned long long* abits = NOISY ? gat<unsigned long long>(ws, pl.o_abits) : nullptr;
  int32_t* zpre = NOISY ? gat<int32_t>(ws, pl.o_zpre) : nullptr;
  unsigned* selb = NOISY ? gat<unsigned>(ws, pl.o_selb) : nullptr;  // waiting ranks admitted this step
  const double sigma = sc.noise_sigma;

  // --- init ----------------------------------------------------------------
  for (int i = lane; i < ((G * B + 3) & ~3); i += 32) {
    s_f[i] = kEmpty;
    if (i < G * B) s_stk[i] = static_cast<uint16_t>(i % B);
  }
  for (int i = lane; i < G; i += 32) {
    s_cap[i] = B;
    s_asum[i] = 0;
    if constexpr (NOISY) s_len[i] = 0;
  }
  if (lane == 0) s_misc[0] = 0;
  constexpr bool kClasses = GREEDY || OVL;
  if (kClasses)
    for (int c = lane; c <= S + 1; c += 32) c_rec[c] = make_int4(0, 0, 0, GREEDY ? cbase_g[c] : 0);
  if (GREEDY && H > 0)
    for (int i = lane; i < H * G; i += 32) {
      s_Wc[i] = 0;
      if constexpr (NOISY) n_Wa[i] = 0;
      else s_Wa[i] = 0;
    }
  ClassSet<SMALLC> wset, pset;  // waiting classes; classes picked in phase 1
  {
    uint64_t* bm = at<SM || (GREEDY && SMALLC), uint64_t>(sm, ws, pl.o_bm);
    uint64_t* pbm = at<SM || (GREEDY && SMALLC), uint64_t>(sm, ws, pl.o_pbm);
    wset.init(bm, bm + 64, S);
    pset.init(pbm, pbm + 64, S);
  }
  if (cal == 1)
    for (int i = lane; i < pl.R * 32; i += 32) calh[i] = -1;
  if (cal == 2)
    for (int i = lane; i < kWheel * LS; i += 32) calh[i] = -1;
  unsigned cons = 0;     // noisy: draws of the stream consumed so far
  long long aw0 = 0;     // first bitmap word holding a waiting (revealed, unadmitted) id
  bool ntie = false;     // a draw landed next to an lround tie (BFSIM_FLAG_NOISE_NEAR_TIE)
  if constexpr (NOISY) {
    for (long long w = lane; w < (N + 63) / 64 + 1; w += 32) abits[w] = 0ull;
    for (long long w = lane; w < (N + 31) / 32 + 1; w += 32) selb[w] = 0u;
  }
  __syncwarp();

  int n[WPL];
  long long A[WPL];
BFSIM_UNROLL_W
  for (int j = 0; j < WPL; ++j) {
    n[j] = 0;
    A[j] = 0;
  }
  const int gbits = bits_for(G - 1) > 0 ? bits_for(G - 1) : 1;
  const uint64_t gmask = (1ull << gbits) - 1ull;
  // largest per-worker load: B requests at their largest workload
  const long long lbound =
      static_cast<long long>(B) * (static_cast<long long>(S) + d * (in.max_decode - 1));
  const bool k32 = bits_for(lbound) + gbits <= 31;

  // a = s - d*x is kept in int32 per slot: steps beyond k_safe would wrap it
  const long long k_safe = d > 0 ? (static_cast<long long>(INT_MAX) - S) / d : LLONG_MAX;
  long long k = 0;
  double clock = 0.0;
  long long nxt = 0, head = 0, n_wait = 0, act = 0, done = 0, tail = 0, adm_total = 0;
  long long maxcount = 0;
  const long long min_pool =
      OVL ? static_cast<long long>(sc.backlog * static_cast<double>(G) * static_cast<double>(B)) : 0;
  long long imb = 0, work = 0, tok = 0, records = 0;
  double energy = 0.0, elapsed = 0.0, tpot_sum = 0.0;
  int status = BFSIM_OK;
  uint32_t flags = 0;

  // Reveal windows: lane j holds trace records nxt + j (A, unpacked) and
  // nxt + 32 + j (B, raw 16-byte record still in flight from the trace).
  double a_arr = 0.0;
  int a_s = 0, a_o = 0;
  int4 b4 = make_int4(0, 0, 0, 0);
  auto load_raw = [&](long long idx) -> int4 {
    return idx < N ? __ldg(reinterpret_cast<const int4*>(tr) + idx) : make_int4(0, 0, 0, 0);
  };
  if (!OVL) {
    const int4 v = load_raw(lane);
    a_arr = __hiloint2double(v.y, v.x);
    a_s = v.z;
    a_o = v.w;
    b4 = load_raw(32 + lane);
  }

  // ---- TPOT terms of buffered completions (metrics.hpp:43-53): request
  // admitted at x, finished at step f: (clock_start[f+1] - clock_start[x]) / o,
  // both read from the clock ring (callers guarantee ring[f+1] is written).
  auto drain_tpot = [&]() {
    __syncwarp();
    const int nb = s_misc[0];
    // four completions per lane in flight (independent loads and partial
    // sums; the sum order is free within the 1e-9 TPOT bar)
    double tp0 = 0.0, tp1 = 0.0, tp2 = 0.0, tp3 = 0.0;
    int e = lane;
    for (; e + 96 < nb; e += 128) {
      const int2 v0 = cbuf[e], v1 = cbuf[e + 32], v2 = cbuf[e + 64], v3 = cbuf[e + 96];
      const double f0 = ring[(v0.y + 1) & Rm], a0 = ring[v0.x & Rm];
      const double f1 = ring[(v1.y + 1) & Rm], a1 = ring[v1.x & Rm];
      const double f2 = ring[(v2.y + 1) & Rm], a2 = ring[v2.x & Rm];
      const double f3 = ring[(v3.y + 1) & Rm], a3 = ring[v3.x & Rm];
      tp0 = __dadd_rn(tp0, __ddiv_rn(__dsub_rn(f0, a0), static_cast<double>(v0.y - v0.x + 1)));
      tp1 = __dadd_rn(tp1, __ddiv_rn(__dsub_rn(f1, a1), static_cast<double>(v1.y - v1.x + 1)));
      tp2 = __dadd_rn(tp2, __ddiv_rn(__dsub_rn(f2, a2), static_cast<double>(v2.y - v2.x + 1)));
      tp3 = __dadd_rn(tp3, __ddiv_rn(__dsub_rn(f3, a3), static_cast<double>(v3.y - v3.x + 1)));
    }
    for (; e < nb; e += 32) {
      const int2 v = cbuf[e];
      const double fin = ring[(v.y + 1) & Rm], adm = ring[v.x & Rm];
      tp0 = __dadd_rn(tp0, __ddiv_rn(__dsub_rn(fin, adm), static_cast<double>(v.y - v.x + 1)));
    }
    const double tp = __dadd_rn(__dadd_rn(tp0, tp1), __dadd_rn(tp2, tp3));
    tpot_sum = __dadd_rn(tpot_sum, wsum_f64(tp));
    __syncwarp();
    if (lane == 0) s_misc[0] = 0;
    __syncwarp();
  };

  // ---- per-step accounting flush: steps k0 .. k0+cnt-1 in ring rows 0..cnt-1
  auto flush = [&](long long k0, int cnt) {
    drain_tpot();
    double dp = 0.0, dtl = 0.0;
    long long imb_l = 0, sum_l = 0, ac_l = 0;
    bool counted = false;
    if (lane < cnt) {
      long long kk = k0 + lane;
      counted = kk >= warmup;
      uint32_t mx = r_mx[lane];
      double dt = r_dt[lane];
      const uint32_t* row = r_l + lane * rstride;
      double mxd = static_cast<double>(mx);
      double p = 0.0;
      unsigned long long smv = 0;
      const double lmx = mx ? log2(mxd) : 0.0;
      for (int g = 0; g < G; ++g) {
        uint32_t L = row[g];
        smv += L;
        // utilization u = L / max (metrics.hpp:56-62), power (metrics_power.hpp:24-27):
        // u^gamma as 2^(gamma (log2 L - log2 max)) -- a few ulp from
        // glibc's pow(L / max, gamma), far inside the 1e-9 energy bar; the
        // idle (u = 0) and straggler (u = 1) workers are exact
        const double pu = L == 0 ? 0.0 : (L == mx ? 1.0 : exp2(gam * (log2(static_cast<double>(L)) - lmx)));
        p = __dadd_rn(p, __dadd_rn(p_idle, __dmul_rn(p_diff, pu)));
      }
      if (counted) {
        imb_l = static_cast<long long>(G) * mx - static_cast<long long>(smv);
        sum_l = static_cast<long long>(smv);
        ac_l = r_ac[lane];
        dp = __dmul_rn(dt, p);
        dtl = dt;
      }
      if (emit_steps && kk < scap) {
        P.steps.clock_start[so + kk] = r_cs[lane];
        P.steps.dt[so + kk] = dt;
        P.steps.max_load[so + kk] = mxd * lsc;
        P.steps.active_count[so + kk] = r_ac[lane];
      }
    }
    imb += wsum_i64(imb_l);
    work += wsum_i64(sum_l);
    tok += wsum_i64(ac_l);
    unsigned cm = __ballot_sync(FULLMASK, counted);
    records += __popc(cm);
    // energy and elapsed summed in step order, as metrics.hpp:32-40,67-76
    for (int i = 0; i < cnt; ++i) {
      double e = __shfl_sync(FULLMASK, dp, i);
      double t = __shfl_sync(FULLMASK, dtl, i);
      if ((cm >> i) & 1u) {
        energy = __dadd_rn(energy, e);
        elapsed = __dadd_rn(elapsed, t);
      }
    }
    if (emit_steps && k0 < scap) {
      long long rows = scap - k0 < cnt ? scap - k0 : cnt;
      for (long long r = 0; r < rows; ++r)
        for (int g = lane; g < G; g += 32)
          P.steps.loads[lo + (k0 + r) * G + g] = static_cast<double>(r_l[r * rstride + g]) * lsc;
    }
    __syncwarp();
  };

  // ---- Poisson reveal (engine.hpp:123-128) ----
  auto reveal = [&]() {
    for (;;) {
      bool ok = (nxt + lane < N) && (a_arr <= clock);
      unsigned m = __ballot_sync(FULLMASK, ok);
      int cnt = __popc(m);  // arrivals sorted: m is a prefix of the lanes
      if (cnt == 0) break;
      long long id = nxt + lane;
      if (ok && emit_reqs) {
        P.reqs.arrival_step[ro + id] = static_cast<int32_t>(k);
        P.reqs.start_step[ro + id] = -1;
        P.reqs.worker[ro + id] = -1;
        P.reqs.admit_clock[ro + id] = 0.0;
        P.reqs.finish_clock[ro + id] = 0.0;
      }
      if constexpr (GREEDY) {
        // push to the back of the per-class deque, arrival order within class
        int pos = 0, npeer = 0;
        bool leader = false;
        int cbase = 0;
        if (ok) {
          unsigned peers = __match_any_sync(m, a_s);
          const int4 cr = c_rec[a_s];
          pos = cr.y + __popc(peers & lanemask_lt());
          cbase = cr.w;
          npeer = __popc(peers);
          leader = (__ffs(peers) - 1) == lane;
        }
        __syncwarp();
        if (ok) {
          deq[cbase + pos] = make_int2(static_cast<int>(id), a_o);
          if (leader) c_rec[a_s].y = pos + npeer;
        }
        wset.add_from_lanes(ok, ok ? a_s : 1);
        __syncwarp();
      } else {
        // stash (s, o) for the FIFO admission: slot = position in the queue
        long long t = id - head;
        if (ok && t < umax) stage[t] = make_int2(a_s, a_o);
      }
      n_wait += cnt;
      nxt += cnt;
      // shift both windows by cnt; refill the tail of B from the trace
      const int src = (lane + cnt) & 31;
      const bool fromA = lane + cnt < 32;
      const double xa = __shfl_sync(FULLMASK, a_arr, src);
      const int sa = __shfl_sync(FULLMASK, a_s, src), oa = __shfl_sync(FULLMASK, a_o, src);
      int4 vb;
      vb.x = __shfl_sync(FULLMASK, b4.x, src);
      vb.y = __shfl_sync(FULLMASK, b4.y, src);
      vb.z = __shfl_sync(FULLMASK, b4.z, src);
      vb.w = __shfl_sync(FULLMASK, b4.w, src);
      if (fromA) {
        a_arr = xa;
        a_s = sa;
        a_o = oa;
        b4 = vb;
      } else {
        a_arr = __hiloint2double(vb.y, vb.x);
        a_s = vb.z;
        a_o = vb.w;
        b4 = load_raw(nxt + 32 + lane);
      }
      if (cnt < 32) break;
    }
  };

  // ---- overloaded top-up until Def. 1 and the backlog hold (oracle.hpp:167-183)
  auto topup = [&]() -> bool {
    const long long freeslots = static_cast<long long>(G) * B - act;
    while (!(n_wait >= min_pool && n_wait - maxcount >= freeslots)) {
      long long idx = tail + lane;
      bool valid = idx < N;
      if (!__any_sync(FULLMASK, valid)) return false;
      int s = 0, o = 0;
      if (valid) {
        int2 v = __ldg(reinterpret_cast<const int2*>(st) + idx);
        s = v.x;
        o = v.y;
      }
      unsigned peers = __match_any_sync(FULLMASK, valid ? s : -1 - lane);
      int4 cr = valid ? c_rec[s] : make_int4(0, 0, 0, 0);
      long long base = static_cast<long long>(cr.y - cr.x);
      unsigned le = lanemask_lt() | (1u << lane);
      long long ncount = valid ? base + __popc(peers & le) : 0;
      long long pm = ncount;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        long long v = __shfl_up_sync(FULLMASK, pm, off);
        if (lane >= off && v > pm) pm = v;
      }
      long long mc = pm > maxcount ? pm : maxcount;
      long long pool_j = n_wait + lane + 1;
      bool cond = valid && pool_j >= min_pool && pool_j - mc >= freeslots;
      unsigned cmask = __ballot_sync(FULLMASK, cond);
      int take = cmask ? __ffs(cmask) : __popc(__ballot_sync(FULLMASK, valid));
      unsigned tm = take >= 32 ? FULLMASK : ((1u << take) - 1u);
      bool tk = lane < take;
      int pos = 0, npeer = 0;
      bool leader = false;
      if (tk) {
        unsigned p2 = peers & tm;
        pos = cr.y + __popc(p2 & lanemask_lt());
        npeer = __popc(p2);
        leader = (__ffs(p2) - 1) == lane;
      }
      __syncwarp();
      if (tk) {
        if (GREEDY) {
          deq[cr.w + pos] = make_int2(static_cast<int>(idx), o);
        } else {
          long long t = idx - head;
          if (t < umax) stage[t] = make_int2(s, o);
        }
        if (leader) c_rec[s].y = pos + npeer;
        if (emit_reqs) {
          P.reqs.arrival_step[ro + idx] = -1;
          P.reqs.start_step[ro + idx] = -1;
          P.reqs.worker[ro + idx] = -1;
          P.reqs.admit_clock[ro + idx] = 0.0;
          P.reqs.finish_clock[ro + idx] = 0.0;
        }
      }
      if (GREEDY) wset.add_from_lanes(tk, tk ? s : 1);
      maxcount = __shfl_sync(FULLMASK, mc, take - 1);
      n_wait += take;
      tail += take;
      __syncwarp();
    }
    return true;
  };

  // Recompute the largest pool class after admissions (is_overloaded_at).
  auto refresh_maxcount = [&]() {
    long long m = 0;
    for (int c = 1 + lane; c <= S; c += 32) {
      const int4 cr = c_rec[c];
      long long v = cr.y - cr.x;
      m = v > m ? v : m;
    }
    maxcount = static_cast<long long>(__reduce_max_sync(FULLMASK, static_cast<uint32_t>(m)));
  };

  // place item (slot write + outputs); called by the item's lane
  auto place = [&](int g, int rank, long long id, int s, int o) {
    int slot = g * B + s_stk[g * B + s_capb[g] - 1 - rank];
    s_f[slot] = static_cast<uint32_t>(k + o - 1);
    s_a[slot] = static_cast<int32_t>(s - d * k);
    if constexpr (NOISY) {  // appended after the worker's active entries (sorted by id below)
      const int pos = g * B + (B - s_capb[g]) + rank;
      st_keep(s_E + pos, make_int2(static_cast<int>(k + o - 1), static_cast<int>(s - d * k)), lkeep);
      s_Eid[pos] = static_cast<int32_t>(id);
    }
    s_x[slot] = static_cast<int32_t>(k);
    s_id[slot] = static_cast<int32_t>(id);
    if (cal == 1) {
      const int b = static_cast<int>((k + o - 1) & Rm);
      calnx[slot] = atomicExch(&calh[b * 32 + (g & 31)], slot);
    } else if (cal == 2) {
      const int b = static_cast<int>((k + o - 1) & (kWheel - 1));
      const int old = atomicExch(&calh[b * LS + (g & 31)], slot);
      wnx[slot] = static_cast<uint16_t>(old < 0 ? 0xFFFF : old);
    }
    if (emit_reqs) {
      P.reqs.start_step[ro + id] = static_cast<int32_t>(k);
      P.reqs.worker[ro + id] = g;
      P.reqs.admit_clock[ro + id] = clock;
    }
  };

  // ---- Noisy lookahead (NOISY) ------------------------------------------
  // The D = active + waiting normal draws of one step, in the reference's
  // order (engine.hpp:131 with GCC's right-to-left argument evaluation:
  // worker_views -- g ascending, insertion order, engine.hpp:204-220 -- then
  // waiting_views in waiting order, :222-231), taken from the producer
  // warp's ring (draws cons .. cons + D - 1 of the trajectory's stream).
  // With `values`, the active draws go straight into the lookahead views:
  // the warp walks each worker's insertion-ordered list {finish step, a}
  // (32 entries per chunk, coalesced, the next chunk in flight). Retirement
  // leaves finished entries in place (finish < k); the walk skips them,
  // numbers the live ones by ballot (draw = running count + rank), and
  // compacts the list as it goes -- one pass over the lists per step instead
  // of a compaction pass at retirement and a draw pass here. s_len[g] is the
  // list length (live entries + not yet dropped finished ones). Each live
  // request's preview (make_preview, policies.hpp:67-90) is added to the
  // worker's difference arrays over h with shared-memory atomics:
  // w_i + d*h while h < min(c_i, rem_i), its last workload a + d*f while
  // rem_i <= h < c_i, with c_i = min(max(1, rem_i + lround(n_i)), H + 1) and
  // rem_i = f - k + 1. A waiting draw's value is kept (nzb[r]) only when its
  // request is admitted this step.
  auto gen_normals = [&](long long D, bool values) {
    if (values) {
      // loop-local copies (the kernel-wide ones live in spilled registers) and
      // 32-bit arithmetic: every quantity below is a step count, a clamped
      // draw or a per-request workload, all < 2^31 (capi.cu bounds)
      const unsigned cn = cons;
      const int32_t kk32 = static_cast<int32_t>(k), d32 = static_cast<int32_t>(d), H1 = H + 1;
      const int32_t dk32 = static_cast<int32_t>(d * k);
      unsigned tie = 0;
      // wait until the producer has published draws [.., cn + hi)
      // (returns the producer count it saw, warp-uniform)
      auto wait_draws = [&](unsigned hi) {
        unsigned seen;
        for (int spin = 0; static_cast<int>((seen = ld_acquire(&s_ctr[0])) - hi) < 0; ++spin) {
          if (spin > (1 << 26)) __trap();  // the producer never stalls this long: fail, do not hang
          __nanosleep(32);
        }
        return __shfl_sync(FULLMASK, seen, 0);
      };
      // the active walk re-reads the producer count only when the draws it
      // saw run out, and releases consumed draws every 256 (a release store
      // orders all of lane 0's earlier memory operations: not per chunk)
      unsigned avail = cn, relp = 0;
      // ---- active draws: worker lists in g order, 32 entries per chunk,
      // the next two chunks' loads in flight (the lists live in L2 / HBM)
      auto next_chunk = [&](int g, int p0, int len, int& g2, int& p2, int& len2) {
        g2 = g;
        p2 = p0 + 32;
        len2 = len;
        if (p2 >= len) {
          p2 = 0;
          len2 = 0;
          while (len2 == 0 && ++g2 < G) len2 = s_len[g2];
        }
      };
      auto load_chunk = [&](int g, int p0, int len) {
        return g < G && p0 + lane < len ? ld_keep(s_E + g * B + p0 + lane, lkeep) : make_int2(0, 0);
      };
      constexpr int PF = 3;  // chunks in flight (the one being processed + PF - 1 ahead)
      int cg[PF], cp[PF], cl[PF];
      int2 ce[PF];
      cg[0] = -1;
      cl[0] = 0;
      cp[0] = 0;
      while (cl[0] == 0 && ++cg[0] < G) cl[0] = s_len[cg[0]];
#pragma unroll
      for (int i = 1; i < PF; ++i) next_chunk(cg[i - 1], cp[i - 1], cl[i - 1], cg[i], cp[i], cl[i]);
#pragma unroll
      for (int i = 0; i < PF; ++i) ce[i] = load_chunk(cg[i], cp[i], cl[i]);
      int wpos = 0;
      unsigned rb = 0;  // active draws taken so far
      while (cg[0] < G) {
        // the next chunk in line, loaded before this chunk's stores (an entry
        // only moves down within its worker's row)
        int gN, pN, lN;
        next_chunk(cg[PF - 1], cp[PF - 1], cl[PF - 1], gN, pN, lN);
        const int2 eN = load_chunk(gN, pN, lN);
        const int g = cg[0], p0 = cp[0], len = cl[0];
        const int2 ecur = ce[0];
        const int p = p0 + lane;
        const bool live = p < len && ecur.x >= kk32;
        const unsigned lm = __ballot_sync(FULLMASK, live);
        const int nl = __popc(lm);
        if (nl) {
          const int rk = __popc(lm & lanemask_lt());
          const unsigned need = cn + rb + static_cast<unsigned>(nl);
          if (static_cast<int>(avail - need) < 0) {
            if (lane == 0) st_release(&s_ctr[1], cn + rb);  // the producer may be waiting for room
            relp = rb;
            avail = wait_draws(need);
          } else if (rb - relp >= 256u) {
            if (lane == 0) st_release(&s_ctr[1], cn + rb);
            relp = rb;
          }
          if (live) {
            const int code = s_ring[(cn + rb + static_cast<unsigned>(rk)) & (kRing - 1)];
            const int32_t lr = code >> 1;
            tie |= static_cast<unsigned>(code) & 1u;
            const int32_t f = ecur.x;
            const int32_t a = ecur.y;
            const int32_t rem = f - kk32 + 1;
            int32_t pred = rem + lr;
            pred = pred > 1 ? pred : 1;
            const int32_t c = pred < H1 ? pred : H1;
            const int32_t m = c < rem ? c : rem;
            if (m <= H) {
              atomicAdd(&n_Wa[(m - 1) * G + g], -(a + dk32));
              atomicAdd(&s_Wc[(m - 1) * G + g], -1);
            }
            if (c > rem) {
              // the last workload a + d*f < 2^31; the product alone may not be
              const int32_t wl = static_cast<int32_t>(static_cast<uint32_t>(a) +
                                                      static_cast<uint32_t>(d32) * static_cast<uint32_t>(f));
              atomicAdd(&n_Wa[(rem - 1) * G + g], wl);
              if (c <= H) atomicAdd(&n_Wa[(c - 1) * G + g], -wl);
            }
            // compaction in place (an entry only moves down; the next chunk
            // is already loaded)
            if (wpos + rk != p) st_keep(s_E + g * B + wpos + rk, ecur, lkeep);
          }
          rb += static_cast<unsigned>(nl);
          wpos += nl;
        }
        if (cg[1] != g) {
          if (lane == 0) s_len[g] = wpos;
          wpos = 0;
        }
#pragma unroll
        for (int i = 0; i + 1 < PF; ++i) {
          cg[i] = cg[i + 1];
          cp[i] = cp[i + 1];
          cl[i] = cl[i + 1];
          ce[i] = ce[i + 1];
        }
        cg[PF - 1] = gN;
        cp[PF - 1] = pN;
        cl[PF - 1] = lN;
        ce[PF - 1] = eN;
      }
      __syncwarp();
      // ---- waiting draws (r >= act): only the admitted ranks' values matter
      for (long long r0 = act; r0 < D; r0 += 32) {
        const long long r = r0 + lane;
        bool need = r < D;
        if (need) {
          const long long q = r - act;
          need = (__ldcg(selb + (q >> 5)) >> (q & 31)) & 1u;
        }
        if (__any_sync(FULLMASK, need)) {
          if (lane == 0) st_release(&s_ctr[1], cn + static_cast<unsigned>(r0));
          const unsigned hi = cn + static_cast<unsigned>(r0 + 32 < D ? r0 + 32 : D);
          wait_draws(hi);
          if (need) {
            const int code = s_ring[(cn + static_cast<unsigned>(r)) & (kRing - 1)];
            tie |= static_cast<unsigned>(code) & 1u;
            nzb[r] = code >> 1;
          }
          __syncwarp();
          if (lane == 0) st_release(&s_ctr[1], hi);
        }
      }
      if (tie) ntie = true;
    }
    cons += static_cast<unsigned>(D);
    __syncwarp();
    if (lane == 0) st_release(&s_ctr[1], cons);
  };

  // Rank of each admitted request in the waiting order (arrival order of the
  // revealed, unadmitted ids): zeros of the admitted-id bitmap below its id.
  auto waiting_ranks = [&](int U, const int32_t* ids, int32_t* out) {
    const long long wl = (nxt - 1) >> 6;
    long long run = 0;
    for (long long b = aw0; b <= wl; b += 32) {
      const long long w = b + lane;
      const int z = w <= wl ? 64 - __popcll(__ldcg(abits + w)) : 0;
      int incl = z;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const int v = __shfl_up_sync(FULLMASK, incl, off);
        if (lane >= off) incl += v;
      }
      if (w <= wl) zpre[w - aw0] = static_cast<int32_t>(run + incl - z);
      run += __shfl_sync(FULLMASK, incl, 31);
    }
    __syncwarp();
    for (int q = lane; q < U; q += 32) {
      const long long id = ids[q];
      const unsigned long long below = (1ull << (id & 63)) - 1ull;
      const int rank = zpre[(id >> 6) - aw0] + __popcll(~__ldcg(abits + (id >> 6)) & below);
      out[q] = rank;
      atomicOr(selb + (rank >> 5), 1u << (rank & 31));
    }
    __syncwarp();
  };

  // Lookahead views F_h[g] (worker_views, engine.hpp:204-220) of the shared
  // chain: prefix of the difference arrays the draw pass filled (zeroed for
  // the next step), F_h[g] = A_g + d k n_g + sum_{h'<=h} Wa + d h (n_g + sum Wc).
  auto noisy_views = [&]() {
BFSIM_UNROLL_W
    for (int j = 0; j < WPL; ++j) {
      const int g = lane + 32 * j;
      if (g >= G) continue;
      long long SW = A[j] + d * k * n[j];
      long long CN = n[j];
      s_F[g] = SW;
      for (int h = 1; h <= H; ++h) {
        SW += n_Wa[(h - 1) * G + g];
        CN += s_Wc[(h - 1) * G + g];
        n_Wa[(h - 1) * G + g] = 0;
        s_Wc[(h - 1) * G + g] = 0;
        s_F[h * G + g] = SW + d * h * CN;
      }
    }
    __syncwarp();
  };

  // FIFO policies: prefetch the (s, o) of the next step's oldest waiting
  // requests (already revealed) into the stage while the tail of this step runs.
  auto prefetch_fifo = [&]() {
    if constexpr (!GREEDY && SM) {
      long long freeslots = static_cast<long long>(G) * B - act;
      long long np = n_wait < freeslots ? n_wait : freeslots;
      np = np < umax ? np : umax;
      for (long long t = lane; t < np; t += 32) {
        const void* src = OVL ? static_cast<const void*>(st + head + t)
                              : static_cast<const void*>(&tr[head + t].prefill);
        cp_async8(&stage[t], src);
      }
    }
  };

  // ---- FCFS / JSQ: closed-form level filling (policies.hpp:100-138) ----
  auto admit_fifo = [&](int U) {
    int cap0[WPL];
    int vext = JSQ ? INT_MAX : 0;
BFSIM_UNROLL_W
    for (int j = 0; j < WPL; ++j) {
      int g = lane + 32 * j;
      cap0[j] = g < G ? B - n[j] : 0;
      if (g < G) s_capb[g] = cap0[j];
      if (!JSQ) vext = cap0[j] > vext ? cap0[j] : vext;
      else if (g < G && cap0[j] > 0 && n[j] < vext) vext = n[j];
    }
    int nl = 0, T = 0;
    // fully served levels end at vfull (-1: none); at most the last level,
    // vpart, is served partially (its first takep workers in index order)
    int vfull = -1, vpart = -1, takep = 0;
    if (!JSQ) {
      // Alg. 3: argmax cap, lowest index first. Level v (cap value, descending)
      // serves every worker with cap0 >= v in index order.
      int v = static_cast<int>(__reduce_max_sync(FULLMASK, static_cast<uint32_t>(vext)));
      for (; v >= 1 && T < U; --v, ++nl) {
        int cnt = 0;
BFSIM_UNROLL_W
        for (int j = 0; j < WPL; ++j) {
          unsigned mk = __ballot_sync(FULLMASK, cap0[j] >= v);
          cnt += __popc(mk);
          if (lane == 0) lvM[nl * WPL + j] = mk;
        }
        int take = cnt < U - T ? cnt : U - T;
        if (lane == 0) {
          lvT[nl] = T;
          lvV[nl] = v;
          lvK[nl] = take;
        }
        if (take == cnt) vfull = v;
        else {
          vpart = v;
          takep = take;
        }
        T += take;
      }
    } else {
      // JSQ: argmin active count over cap > 0, lowest index first. Level v
      // (count value, ascending) serves every worker with count0 <= v < B.
      int v = static_cast<int>(__reduce_min_sync(FULLMASK, static_cast<uint32_t>(vext)));
      for (; v <= B - 1 && T < U; ++v, ++nl) {
        int cnt = 0;
BFSIM_UNROLL_W
        for (int j = 0; j < WPL; ++j) {
          int g = lane + 32 * j;
          unsigned mk = __ballot_sync(FULLMASK, g < G && n[j] <= v);
          cnt += __popc(mk);
          if (lane == 0) lvM[nl * WPL + j] = mk;
        }
        int take = cnt < U - T ? cnt : U - T;
        if (lane == 0) {
          lvT[nl] = T;
          lvV[nl] = v;
          lvK[nl] = take;
        }
        if (take == cnt) vfull = v;
        else {
          vpart = v;
          takep = take;
        }
        T += take;
      }
    }
    if (SM) cp_async_wait_all();
    __syncwarp();
    // placement: admission t takes waiting request head + t and goes to the
    // worker it is the t-th of, levels in order, index order within a level
    auto fifo_place = [&](int t, int g, int vl) {
      const int rank = JSQ ? vl - (B - s_capb[g]) : s_capb[g] - vl;
      const long long id = head + t;
      int s, o;
      if (SM && t < umax) {
        int2 v = stage[t];
        s = v.x;
        o = v.y;
      } else if (OVL) {
        int2 v = __ldg(reinterpret_cast<const int2*>(st) + id);
        s = v.x;
        o = v.y;
      } else {
        int4 v = __ldg(reinterpret_cast<const int4*>(tr) + id);
        s = v.z;
        o = v.w;
      }
      if (OVL) atomicAdd(&c_rec[s].x, 1);  // leaves the pool (class count for Def. 1)
      place(g, rank, id, s, o);
      atomicAdd(&s_asum[g], static_cast<unsigned long long>(static_cast<long long>(s) - d * k));
    };
    if constexpr (WPL <= 2) {
      // item-parallel: few worker blocks, so each lane finds its level and
      // worker directly
      for (int t = lane; t < U; t += 32) {
        int l = 0;
        while (l + 1 < nl && lvT[l + 1] <= t) ++l;
        int pos = t - lvT[l];
        int g = 0;
#pragma unroll
        for (int j = 0; j < WPL; ++j) {
          const uint32_t mk = lvM[l * WPL + j];
          const int c = __popc(mk);
          if (pos >= 0 && pos < c) {
            g = static_cast<int>(__fns(mk, 0, pos + 1)) + 32 * j;
            pos = -1;
          } else if (pos >= 0) {
            pos -= c;
          }
        }
        fifo_place(t, g, lvV[l]);
      }
    } else {
      // segment by segment: level l, worker block j holds the next
      // min(popc, left) admissions
      int t0 = 0;
      for (int l = 0; l < nl; ++l) {
        int left = lvK[l];
        const int vl = lvV[l];
        for (int j = 0; j < WPL && left > 0; ++j) {
          const uint32_t mk = lvM[l * WPL + j];
          int c = __popc(mk);
          c = c < left ? c : left;
          for (int i = lane; i < c; i += 32)
            fifo_place(t0 + i, static_cast<int>(__fns(mk, 0, i + 1)) + 32 * j, vl);
          t0 += c;
          left -= c;
        }
      }
    }
    __syncwarp();
    // admissions per worker in closed form: every fully served level the
    // worker is eligible for, plus its rank in the partial level
    {
      int before = 0;
BFSIM_UNROLL_W
      for (int j = 0; j < WPL; ++j) {
        const int g = lane + 32 * j;
        int adm = 0;
        if (g < G) {
          if (!JSQ) adm = vfull >= 1 && cap0[j] >= vfull ? cap0[j] - vfull + 1 : 0;
          else adm = vfull >= 0 && cap0[j] > 0 && n[j] <= vfull ? vfull - n[j] + 1 : 0;
        }
        const bool elig = vpart >= 0 && g < G && (JSQ ? n[j] <= vpart : cap0[j] >= vpart);
        const unsigned mk = __ballot_sync(FULLMASK, elig);
        if (elig && before + __popc(mk & lanemask_lt()) < takep) ++adm;
        before += __popc(mk);
        if (g < G) {
          n[j] += adm;
          A[j] += static_cast<long long>(s_asum[g]);
          s_asum[g] = 0;
        }
      }
    }
    head += U;
    __syncwarp();
  };

  // ---- bfio-greedy (policies.hpp:269-370) ----
  // Keys are (load << gbits | g), 32-bit when every load fits (K32).
  auto admit_greedy = [&](int U, long long free_total, auto k32c) {
    constexpr bool K32 = decltype(k32c)::value;
    using key_t = typename std::conditional<K32, uint32_t, uint64_t>::type;
    constexpr key_t KMAX = static_cast<key_t>(~0ull);
    const bool phase1 = n_wait > free_total;
    int cp[WPL];
    long long F0[WPL];
BFSIM_UNROLL_W
    for (int j = 0; j < WPL; ++j) {
      int g = lane + 32 * j;
      cp[j] = g < G ? B - n[j] : 0;
      F0[j] = g < G ? A[j] + d * k * n[j] : 0;
      if (g < G) s_capb[g] = cp[j];
    }
    auto lane_key = [&](const long long* ld, const int* fr) -> key_t {
      key_t best = KMAX;
BFSIM_UNROLL_W
      for (int j = 0; j < WPL; ++j) {
        const int g = lane + 32 * j;
        const key_t kk = (static_cast<key_t>(ld[j]) << gbits) | static_cast<key_t>(g);
        best = (fr[j] > 0 && kk < best) ? kk : best;  // fr == 0 for g >= G
      }
      return best;
    };
    auto wmin = [&](key_t key) -> key_t {
      if constexpr (K32) return __reduce_min_sync(FULLMASK, key);
      else return wmin_u64(key);
    };
    // WPL >= 16 (G > 256): the lane arrays live in local memory, so a lane
    // does not rescan its workers after a pick. Worker keys sit in s_key and
    // the owner lane's best is re-reduced by the whole warp (one load each).
    constexpr bool kCoop = WPL >= 16;
    auto coop_init = [&](const long long* ld, const int* fr) {
      if constexpr (kCoop) {
BFSIM_UNROLL_W
        for (int j = 0; j < WPL; ++j) {
          const int g = lane + 32 * j;
          s_key[g] = fr[j] > 0 ? (static_cast<uint64_t>(ld[j]) << gbits) | static_cast<uint64_t>(g)
                               : ~0ull;
        }
        __syncwarp();
      }
    };
    // after worker gs changed: its owner lane's new best, reduced cooperatively
    auto coop_best = [&](int gs, key_t lk) -> key_t {
      if constexpr (kCoop) {
        __syncwarp();
        const int own = gs & 31;
        const key_t v = lane < WPL ? static_cast<key_t>(s_key[own + 32 * lane]) : KMAX;
        const key_t m = wmin(v);
        return lane == own ? m : lk;
      } else {
        return lk;
      }
    };
    // prefetch one deque entry into the stage (async; waited before resolution)
    auto fetch = [&](int slot, int base, int idx) {
      if constexpr (SM) cp_async8(&stage[slot], &deq[base + idx]);
      else stage[slot] = deq[base + idx];
    };

    if (phase1) {
      // water filling (policies.hpp:274-323) restated over class deques (F4):
      // the lowest-loaded worker with a free slot takes the latest request of
      // the largest class <= deficit, else the earliest of the smallest class.
      long long ld[WPL];
      int fr[WPL];
      long long tmax = 0;
BFSIM_UNROLL_W
      for (int j = 0; j < WPL; ++j) {
        ld[j] = F0[j];
        fr[j] = cp[j];
        tmax = ld[j] > tmax ? ld[j] : tmax;
      }
      long long target = static_cast<long long>(
          __reduce_max_sync(FULLMASK, static_cast<uint32_t>(tmax)));
      key_t lk = lane_key(ld, fr);
      coop_init(ld, fr);
      for (int q = 0; q < U; ++q) {
        const key_t km = wmin(lk);
        const long long lmin = static_cast<long long>(km >> gbits);
        const int gs = static_cast<int>(km) & static_cast<int>(gmask);
        int c = wset.highest_le(target - lmin);
        const bool back = c != 0;
        if (!back) c = wset.lowest();
        // one 128-bit record load; every lane stores the same updated record
        int4 cr = c_rec[c];
        const int idx = back ? cr.y - 1 : cr.x;
        const int t = cr.z;
        if (cr.y - cr.x == 1) wset.clear(c);
        if (back) cr.y -= 1;
        else cr.x += 1;
        cr.z = t + 1;
        c_rec[c] = cr;
        if (lane == 0) {
          p_cl[q] = c;
          p_t[q] = t;
          fetch(q, cr.w, idx);
        }
        if constexpr (!SMALLC) pset.add_uniform(c);
        if constexpr (kCoop) {
          if (lane == (gs & 31)) {
            const int jj = gs >> 5;
            ld[jj] += c;
            fr[jj] -= 1;
            s_key[gs] = fr[jj] > 0 ? (static_cast<uint64_t>(ld[jj]) << gbits) | static_cast<uint64_t>(gs)
                                   : ~0ull;
          }
          lk = coop_best(gs, lk);
        } else {
BFSIM_UNROLL_W
          for (int j = 0; j < WPL; ++j)
            if (lane + 32 * j == gs) {
              ld[j] += c;
              fr[j] -= 1;
            }
          lk = lane_key(ld, fr);
        }
        const long long nl = lmin + c;
        target = nl > target ? nl : target;
      }
    }

    int adm[WPL];
BFSIM_UNROLL_W
    for (int j = 0; j < WPL; ++j) adm[j] = 0;
    const long long ak = -d * k;  // a = s - d*x with x = k

    // Order the U admitted items as the reference's stable sort by w0
    // descending (policies.hpp:324-326): class descending; within a class pick
    // order (phase 1) or waiting order. o_c[j] = class of the j-th item;
    // c_cs[c] = first position of class c. Without phase 1 every waiting
    // request is admitted: the deques are drained and their entries prefetched
    // into stage[j].
    if constexpr (SMALLC) {
      int run = 0;
      for (int base = S; base >= 1; base -= 32) {  // S <= 64: at most two rounds
        const int c = base - lane;
        int nc = 0;
        int4 cr = make_int4(0, 0, 0, 0);
        if (c >= 1) {
          cr = c_rec[c];
          nc = phase1 ? cr.z : cr.y - cr.x;
        }
        int incl = nc;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
          const int v = __shfl_up_sync(FULLMASK, incl, off);
          if (lane >= off) incl += v;
        }
        const int start = run + incl - nc;
        run += __shfl_sync(FULLMASK, incl, 31);
        if (nc > 0) {
          c_cs[c] = start;
          if (phase1) {
            cr.z = 0;
          } else {
            for (int t = 0; t < nc; ++t) {
              o_c[start + t] = c;
              fetch(start + t, cr.w, cr.x + t);
            }
            cr.x = cr.y;
          }
          c_rec[c] = cr;
        }
      }
      if (!phase1) wset.clear_all();
    } else {
      int jpos = 0;
      ClassSet<SMALLC>& set = phase1 ? pset : wset;
      while (!set.empty()) {
        const int c = set.highest();
        int4 cr = c_rec[c];
        int nc;
        if (phase1) {
          nc = cr.z;
          cr.z = 0;
        } else {
          nc = cr.y - cr.x;
          for (int t = lane; t < nc; t += 32) {
            o_c[jpos + t] = c;
            fetch(jpos + t, cr.w, cr.x + t);
          }
          cr.x = cr.y;
        }
        c_rec[c] = cr;
        c_cs[c] = jpos;
        set.clear(c);
        jpos += nc;
      }
    }
    __syncwarp();
    if (phase1)
      for (int q = lane; q < U; q += 32) {
        const int c = p_cl[q];
        o_c[c_cs[c] + p_t[q]] = c;
      }
    __syncwarp();

    if (H == 0) {
      // placement (policies.hpp:339-367) at H = 0: argmin (load, index) over
      // workers with a free slot (F3), one warp reduction per item
      key_t lk = lane_key(F0, cp);
      coop_init(F0, cp);
      int cnext = o_c[0], cnext2 = U > 1 ? o_c[1] : 0;  // item classes, two ahead
      for (int j = 0; j < U; ++j) {
        const int c = cnext;
        cnext = cnext2;
        if (j + 2 < U) cnext2 = o_c[j + 2];
        const key_t km = wmin(lk);
        const int gs = static_cast<int>(km) & static_cast<int>(gmask);
        if constexpr (kCoop) {
          if (lane == (gs & 31)) {
            const int jj = gs >> 5;
            F0[jj] += c;
            cp[jj] -= 1;
            A[jj] += c + ak;
            s_res[j] = static_cast<uint32_t>(gs) | (static_cast<uint32_t>(adm[jj]) << 16);
            adm[jj] += 1;
            s_key[gs] = cp[jj] > 0 ? (static_cast<uint64_t>(F0[jj]) << gbits) | static_cast<uint64_t>(gs)
                                   : ~0ull;
          }
          lk = coop_best(gs, lk);
        } else {
BFSIM_UNROLL_W
          for (int jj = 0; jj < WPL; ++jj)
            if (lane + 32 * jj == gs) {
              F0[jj] += c;
              cp[jj] -= 1;
              A[jj] += c + ak;
              s_res[j] = static_cast<uint32_t>(gs) | (static_cast<uint32_t>(adm[jj]) << 16);
              adm[jj] += 1;
            }
          lk = lane_key(F0, cp);
        }
      }
      if (SM) cp_async_wait_all();
      __syncwarp();
      for (int q = lane; q < U; q += 32) {
        const int c = phase1 ? p_cl[q] : o_c[q];
        const uint32_t r = s_res[phase1 ? c_cs[c] + p_t[q] : q];
        const int2 e = stage[q];
        place(static_cast<int>(r & 0xFFFFu), static_cast<int>(r >> 16), e.x, c, e.y);
      }
    } else {
      // general H: lookahead views F_h[g] from the finish window
      // (HR > 0: int32 views F_h[g] in shared memory, row-major [h][g], for
      // the chain below)
      int32_t* s_F32 = reinterpret_cast<int32_t*>(s_F);
      if constexpr (!NOISY && (HR > 0 || WIDE)) {
BFSIM_UNROLL_W
        for (int j = 0; j < WPL; ++j) {
          const int g = lane + 32 * j;
          if (g >= G) continue;
          long long PA = 0, PC = 0, Q = 0;
          int r = static_cast<int>(k % Hm);  // ring row of step k + h - 1
          for (int h = 0; h <= H; ++h) {
            if (h > 0) {
              PA += s_Wa[r * G + g];
              PC += s_Wc[r * G + g];
              Q += PC;
              r = r + 1 == Hm ? 0 : r + 1;
            }
            const long long kh = k + h;
            const long long F = trunc ? A[j] + d * kh * n[j] - d * Q : (A[j] + d * kh * n[j]) - (PA + d * kh * PC);
            if constexpr (HR > 0) s_F32[g * HP + h] = static_cast<int32_t>(F);
            else s_F32[h * G + g] = static_cast<int32_t>(F);
          }
          if constexpr (HR > 0)
            for (int h = H + 1; h < HP; ++h) s_F32[g * HP + h] = 0;
        }
      }
      if constexpr (!NOISY && HR == 0 && !WIDE) {
BFSIM_UNROLL_W
        for (int j = 0; j < WPL; ++j) {
          int g = lane + 32 * j;
          if (g >= G) continue;
          long long PA = 0, PC = 0, Q = 0;
          for (int h = 0; h <= H; ++h) {
            if (h > 0) {
              int r = static_cast<int>((k + h - 1) % Hm);
              PA += s_Wa[r * G + g];
              PC += s_Wc[r * G + g];
              Q += PC;
            }
            long long kh = k + h;
            long long F = trunc ? A[j] + d * kh * n[j] - d * Q
                                : (A[j] + d * kh * n[j]) - (PA + d * kh * PC);
            s_F[h * G + g] = F;
          }
        }
      }
      if (SM) cp_async_wait_all();
      __syncwarp();
      for (int q = lane; q < U; q += 32) {
        const int jp = phase1 ? c_cs[p_cl[q]] + p_t[q] : q;
        const int2 e = stage[q];
        o_o[jp] = e.y;
        o_id[jp] = e.x;
      }
      __syncwarp();
      if constexpr (NOISY) {
        // this step's draws (all of them, as the reference takes them): the
        // active draws build the views' difference arrays, each admitted
        // request keeps its own waiting draw
        waiting_ranks(U, o_id, o_nz);
        gen_normals(act + n_wait, true);
        if constexpr (HR == 0) noisy_views();
        for (int q = lane; q < U; q += 32) {
          const int rank = o_nz[q];
          o_nz[q] = nzb[act + rank];
          selb[rank >> 5] = 0u;
        }
      }
      // Per-item class, decode length and predicted completion, lane-held 32
      // items at a time with the next 32 in flight: coalesced loads off the
      // placement chain instead of dependent scalar loads per item.
      int ic = 0, io = 1, iz = 0, nc2 = 0, no2 = 1, nz2 = 0;
      auto item_load = [&](int q0) {
        const int qi = q0 + lane;
        nc2 = qi < U ? o_c[qi] : 0;
        no2 = qi < U ? o_o[qi] : 1;
        if constexpr (NOISY) nz2 = qi < U ? o_nz[qi] : 0;
      };
      // preview (make_preview, policies.hpp:67-90): w_h = c + d*min(h, o-1)
      // for h < lim, else 0; lim = predicted completion (perfect: o;
      // truncated: max(o, H+1); noisy: max(1, o + lround(n)))
      auto item_at = [&](int q, int& c, int& o, long long& lim) {
        if ((q & 31) == 0) {
          ic = nc2;
          io = no2;
          iz = nz2;
          item_load(q + 32);
        }
        c = __shfl_sync(FULLMASK, ic, q & 31);
        o = __shfl_sync(FULLMASK, io, q & 31);
        lim = o;
        if constexpr (NOISY) {
          lim = static_cast<long long>(o) + __shfl_sync(FULLMASK, iz, q & 31);
          lim = lim > 1 ? lim : 1;
        } else {
          if (trunc && lim < H + 1) lim = H + 1;
        }
      };
      item_load(0);
      if constexpr (HR > 0) {
        // int32 chain (H < HR <= 24, G <= 128, every cost < 2^31; the planner
        // checks the bounds). F_h[g] lives in shared memory ([h][g]); lane h
        // holds M_h = max_g F_h[g] and, per item, w_h and T_h = M_h - w_h;
        // lane g holds F_0 of its workers. The placement cost of worker g is
        // sum_h max(M_h, F_h[g] + w_h) = sum_h w_h + sum_h max(T_h, F_h[g]);
        // the first sum does not depend on g, so the argmin and its ties over
        // (cost, F_0[g], g) are unchanged (policies.hpp:339-367).
        if constexpr (NOISY) {
          // views: prefix of the difference arrays the draw pass filled
          // (zeroed for the next step)
BFSIM_UNROLL_W
          for (int j = 0; j < WPL; ++j) {
            const int g = lane + 32 * j;
            if (g >= G) continue;
            long long SW = A[j] + d * k * n[j];
            long long CN = n[j];
            int4* row = reinterpret_cast<int4*>(s_F32 + g * HP);
            int32_t v[4];
            v[0] = static_cast<int32_t>(SW);
#pragma unroll
            for (int h = 1; h < 4 * HP4MAX; ++h) {
              if (h >= HP) break;
              if (h <= H) {
                SW += n_Wa[(h - 1) * G + g];
                CN += s_Wc[(h - 1) * G + g];
                n_Wa[(h - 1) * G + g] = 0;
                s_Wc[(h - 1) * G + g] = 0;
                v[h & 3] = static_cast<int32_t>(SW + d * h * CN);
              } else {
                v[h & 3] = 0;
              }
              if ((h & 3) == 3) row[h >> 2] = make_int4(v[0], v[1], v[2], v[3]);
            }
          }
        }
        __syncwarp();
        const bool hl = lane <= H;  // this lane holds horizon h = lane
        int32_t Ml = 0;              // M_lane
        if (hl)
          for (int g = 0; g < G; ++g) {
            const int32_t v = s_F32[g * HP + lane];
            Ml = v > Ml ? v : Ml;
          }
        // The chain's per-worker state is in shared memory too (lane-owned
        // registers would be spilled at this kernel's register budget): the
        // free slots left (s_cap, already the pre-admission cap), the
        // admissions so far (s_admc, rank of the next one) and the workload
        // admitted (s_asum), folded into the registers after the chain.
BFSIM_UNROLL_W
        for (int j = 0; j < WPL; ++j)
          if (lane + 32 * j < G) s_admc[lane + 32 * j] = 0;
        __syncwarp();
        const int32_t d32 = static_cast<int32_t>(d);
        const int32_t dl = d32 * lane;
        // F_0 and the free slots of the lane's workers stay in registers
        // across the items (only the chosen worker's change: F_0 += w_0 = c,
        // one slot less), so the per-item fast-path key needs no shared loads
        int32_t F0r[WPL], capr[WPL];
BFSIM_UNROLL_W
        for (int j = 0; j < WPL; ++j) {
          const int g = lane + 32 * j;
          F0r[j] = g < G ? s_F32[g * HP] : 0;
          capr[j] = g < G ? s_cap[g] : 0;
        }
        for (int q = 0; q < U; ++q) {
          int c, o;
          long long lim;
          item_at(q, c, o, lim);
          const int limH = static_cast<int>(lim < H + 1 ? lim : H + 1);
          const int32_t sat = d32 * (o - 1);
          const int32_t wl = lane < limH ? c + (dl < sat ? dl : sat) : 0;
          // Fast path: g* = argmin (F_0[g], g) over workers with a free slot.
          // Every cost is >= sum_h M_h, and g*'s cost equals it iff
          // F_h[g*] + w_h <= M_h for every h; then g* has the minimum cost
          // and the smallest (F_0, g) tie-break key, so it wins outright.
          // Otherwise the full scan over every worker.
          key_t fk = KMAX;
          int32_t F0v[WPL];
          bool fre[WPL];
BFSIM_UNROLL_W
          for (int j = 0; j < WPL; ++j) {
            const int g = lane + 32 * j;
            F0v[j] = F0r[j];
            fre[j] = capr[j] > 0;
            const key_t kk = (static_cast<key_t>(static_cast<uint32_t>(F0v[j])) << gbits) | static_cast<key_t>(g);
            if (fre[j] && kk < fk) fk = kk;
          }
          int gs = static_cast<int>(wmin(fk) & static_cast<key_t>(gmask));
          int32_t Fg = hl ? s_F32[gs * HP + lane] : 0;
          if (__any_sync(FULLMASK, hl && Fg + wl > Ml)) {
            // T_h = M_h - w_h from lane h (zero past H, like the rows); every
            // lane scans its workers' rows 4 horizons per 128-bit load
            const int32_t Tl = Ml - wl;
            uint32_t cost[WPL];
BFSIM_UNROLL_W
            for (int j = 0; j < WPL; ++j) cost[j] = 0;
            const int nh4 = (H + 4) >> 2;
#pragma unroll
            for (int h4 = 0; h4 < HP4MAX; ++h4) {
              if (h4 < nh4) {
                int4 T;
                T.x = __shfl_sync(FULLMASK, Tl, 4 * h4);
                T.y = __shfl_sync(FULLMASK, Tl, 4 * h4 + 1);
                T.z = __shfl_sync(FULLMASK, Tl, 4 * h4 + 2);
                T.w = __shfl_sync(FULLMASK, Tl, 4 * h4 + 3);
BFSIM_UNROLL_W
                for (int j = 0; j < WPL; ++j) {
                  const int g = lane + 32 * j;
                  const int4 f = reinterpret_cast<const int4*>(s_F32 + (g < G ? g : 0) * HP)[h4];
                  cost[j] += static_cast<uint32_t>(T.x > f.x ? T.x : f.x) + static_cast<uint32_t>(T.y > f.y ? T.y : f.y) +
                             static_cast<uint32_t>(T.z > f.z ? T.z : f.z) + static_cast<uint32_t>(T.w > f.w ? T.w : f.w);
                }
              }
            }
            uint64_t best = ~0ull;
BFSIM_UNROLL_W
            for (int j = 0; j < WPL; ++j) {
              const int g = lane + 32 * j;
              const uint64_t key = (static_cast<uint64_t>(cost[j]) << 32) |
                                   (static_cast<uint64_t>(static_cast<uint32_t>(F0v[j])) << gbits) |
                                   static_cast<uint64_t>(g);
              if (fre[j] && key < best) best = key;
            }
            gs = static_cast<int>(wmin_u64(best) & gmask);
            Fg = hl ? s_F32[gs * HP + lane] : 0;
          }
          // lane h adds w_h to the chosen row (row 0: its F_0) and raises
          // M_h; the owner lane books the admission
          if (hl) {
            const int32_t v = Fg + wl;
            s_F32[gs * HP + lane] = v;
            Ml = v > Ml ? v : Ml;
          }
BFSIM_UNROLL_W
          for (int j = 0; j < WPL; ++j)
            if (lane + 32 * j == gs) {
              F0r[j] += c;
              capr[j] -= 1;
            }
          if (lane == (gs & 31)) {
            const int rank = s_admc[gs];
            s_admc[gs] = rank + 1;
            s_cap[gs] -= 1;
            s_asum[gs] += static_cast<unsigned long long>(static_cast<long long>(c) + ak);
            s_res[q] = static_cast<uint32_t>(gs) | (static_cast<uint32_t>(rank) << 16);
            if (!NOISY && o <= H) {  // finishes inside the window [k, k+H-1]
              int r = static_cast<int>((k + o - 1) % Hm);
              s_Wc[r * G + gs] += 1;
              s_Wa[r * G + gs] += c + ak;
            }
          }
          __syncwarp();
        }
BFSIM_UNROLL_W
        for (int j = 0; j < WPL; ++j) {
          const int g = lane + 32 * j;
          if (g >= G) continue;
          adm[j] = s_admc[g];
          cp[j] = s_cap[g];
          A[j] += static_cast<long long>(s_asum[g]);
          s_asum[g] = 0;
        }
        __syncwarp();
      } else if constexpr (WIDE) {
        // the CTA's W warps place the items together (wide_chain); the
        // per-worker chain state goes through shared memory and is folded
        // into warp 0's registers afterwards
BFSIM_UNROLL_W
        for (int j = 0; j < WPL; ++j)
          if (lane + 32 * j < G) s_admc[lane + 32 * j] = 0;
        if (lane == 0) {
          WideChain& w = *wctl;
          w.cmd = 1;
          w.U = U;
          w.H = H;
          w.G = G;
          w.gbits = gbits;
          w.Hm = Hm;
          w.trunc = trunc ? 1 : 0;
          w.k = k;
          w.d = d;
          w.ak = ak;
          w.o_c = o_c;
          w.o_o = o_o;
          w.F = static_cast<int>(pl.o_F);  // core arrays: offsets in the arena (at the start of
          w.M = static_cast<int>(pl.o_M);  // the CTA's dynamic shared memory)
          w.cap = static_cast<int>(pl.o_cap);
          w.admc = static_cast<int>(pl.o_admc);
          w.asum = static_cast<int>(pl.o_asum);
          w.res = s_res;
          w.Wc = s_Wc;
          w.Wa = s_Wa;
        }
        __threadfence_block();
        const int nthreads = static_cast<int>(blockDim.x);
        cta_bar(nthreads);  // the helper warps start
        wide_chain(*wctl, wred, nthreads);
BFSIM_UNROLL_W
        for (int j = 0; j < WPL; ++j) {
          const int g = lane + 32 * j;
          if (g >= G) continue;
          adm[j] = s_admc[g];
          cp[j] = s_cap[g];
          A[j] += static_cast<long long>(s_asum[g]);
          s_asum[g] = 0;
        }
        __syncwarp();
      } else {
        // Shared-memory chain (any G and H): the same cost split as the
        // register chain -- sum_h max(T_h, F_h[g]) with T_h = M_h - w_h per
        // item in shared memory -- and the chosen row / maxima updated by all
        // lanes in parallel over h.
        long long* s_T = s_M + (H + 1);
        long long* s_w = s_M + 2 * (H + 1);
        for (int h = 0; h <= H; ++h) {
          long long m = 0;
          for (int g = lane; g < G; g += 32) m = s_F[h * G + g] > m ? s_F[h * G + g] : m;
#pragma unroll
          for (int off = 16; off > 0; off >>= 1) {
            const long long t = __shfl_xor_sync(FULLMASK, m, off);
            m = t > m ? t : m;
          }
          if (lane == 0) s_M[h] = m;
        }
        __syncwarp();
        for (int q = 0; q < U; ++q) {
          int c, o;
          long long lim;
          item_at(q, c, o, lim);
          for (int h = lane; h <= H; h += 32) {
            const long long w = h < lim ? c + d * (h < o ? h : o - 1) : 0;
            s_w[h] = w;
            s_T[h] = s_M[h] - w;
          }
          __syncwarp();
          // Fast path: g* = argmin (F_0[g], g) over workers with a free slot.
          // Its excess sum_h max(0, F_h[g*] - T_h) is 0 iff no horizon rises
          // above the current maximum; every cost is >= sum_h T_h, so then g*
          // wins outright (cost and tie-break). Otherwise the full scan.
          uint64_t fk = ~0ull;
  BFSIM_UNROLL_W
          for (int j = 0; j < WPL; ++j) {
            const int g = lane + 32 * j;
            const uint64_t key = (static_cast<uint64_t>(s_F[g]) << gbits) | static_cast<uint64_t>(g);
            if (g < G && cp[j] > 0 && key < fk) fk = key;
          }
          const int gstar = static_cast<int>(wmin_u64(fk) & gmask);
          bool over = false;
          for (int h = lane; h <= H; h += 32) over = over || s_F[h * G + gstar] > s_T[h];
          int gs = gstar;
          if (__any_sync(FULLMASK, over)) {
            // lane-best (cost, F0, g) over owned workers with a free slot
            uint64_t bc = ~0ull, bk = ~0ull;
    BFSIM_UNROLL_W
            for (int j = 0; j < WPL; ++j) {
              const int g = lane + 32 * j;
              if (g >= G || cp[j] <= 0) continue;
              long long a0 = 0, a1 = 0, a2 = 0, a3 = 0;
              int h = 0;
              for (; h + 3 <= H; h += 4) {
                const long long f0 = s_F[h * G + g], f1 = s_F[(h + 1) * G + g];
                const long long f2 = s_F[(h + 2) * G + g], f3 = s_F[(h + 3) * G + g];
                const long long t0 = s_T[h], t1 = s_T[h + 1], t2 = s_T[h + 2], t3 = s_T[h + 3];
                a0 += t0 > f0 ? t0 : f0;
                a1 += t1 > f1 ? t1 : f1;
                a2 += t2 > f2 ? t2 : f2;
                a3 += t3 > f3 ? t3 : f3;
              }
              for (; h <= H; ++h) {
                const long long f0 = s_F[h * G + g], t0 = s_T[h];
                a0 += t0 > f0 ? t0 : f0;
              }
              const uint64_t cost = static_cast<uint64_t>(a0 + a1 + a2 + a3);
              const uint64_t k2 = (static_cast<uint64_t>(s_F[g]) << gbits) | static_cast<uint64_t>(g);
              if (cost < bc || (cost == bc && k2 < bk)) {
                bc = cost;
                bk = k2;
              }
            }
            const uint64_t cmin = wmin_u64(bc);
            const uint64_t kmin = wmin_u64(bc == cmin ? bk : ~0ull);
            gs = static_cast<int>(kmin & gmask);
          }
          for (int h = lane; h <= H; h += 32) {
            const long long v = s_F[h * G + gs] + s_w[h];
            s_F[h * G + gs] = v;
            if (v > s_M[h]) s_M[h] = v;
          }
          if (lane == (gs & 31)) {
            const int jj = gs >> 5;
            if constexpr (WPL > 8) {
              cp[jj] -= 1;
              A[jj] += c + ak;
              s_res[q] = static_cast<uint32_t>(gs) | (static_cast<uint32_t>(adm[jj]) << 16);
              adm[jj] += 1;
            } else {
#pragma unroll
              for (int j = 0; j < WPL; ++j)
                if (j == jj) {
                  cp[j] -= 1;
                  A[j] += c + ak;
                  s_res[q] = static_cast<uint32_t>(gs) | (static_cast<uint32_t>(adm[j]) << 16);
                  adm[j] += 1;
                }
            }
            if (!NOISY && o <= H) {  // finishes inside the window [k, k+H-1]
              const int r = static_cast<int>((k + o - 1) % Hm);
              s_Wc[r * G + gs] += 1;
              s_Wa[r * G + gs] += c + ak;
            }
          }
          __syncwarp();
        }
      }
      for (int q = lane; q < U; q += 32) {
        uint32_t r = s_res[q];
        place(static_cast<int>(r & 0xFFFFu), static_cast<int>(r >> 16), o_id[q], o_c[q], o_o[q]);
        if constexpr (NOISY) {
          const long long id = o_id[q];
          atomicOr(abits + (id >> 6), 1ull << (id & 63));
        }
      }
      if constexpr (NOISY) {
        // this step's admissions were appended to each worker's list in
        // placement order: sort them into waiting order (Simulation::apply
        // pushes in assignment order, sorted by waiting index:
        // engine.hpp:233-248, policies.hpp:368)
        __syncwarp();
BFSIM_UNROLL_W
        for (int j = 0; j < WPL; ++j) {
          const int g = lane + 32 * j;
          if (g >= G) continue;
          const int base = g * B + n[j];
          s_len[g] = n[j] + adm[j];  // the draw pass compacted the list to n[j] live entries
          for (int t = 1; t < adm[j]; ++t) {
            const int key = s_Eid[base + t];
            const int2 ev = s_E[base + t];
            int pos = t;
            while (pos > 0 && s_Eid[base + pos - 1] > key) {
              s_Eid[base + pos] = s_Eid[base + pos - 1];
              s_E[base + pos] = s_E[base + pos - 1];
              --pos;
            }
            s_Eid[base + pos] = key;
            s_E[base + pos] = ev;
          }
        }
        // advance the first bitmap word that still holds a waiting id
        const long long nw = (N + 63) / 64;
        for (;;) {
          const long long w = aw0 + lane;
          const bool full = w < nw && __ldcg(abits + w) == ~0ull;
          const unsigned m = __ballot_sync(FULLMASK, !full);
          if (m) {
            aw0 += __ffs(m) - 1;
            break;
          }
          aw0 += 32;
        }
      }
    }
BFSIM_UNROLL_W
    for (int j = 0; j < WPL; ++j) n[j] += adm[j];
    __syncwarp();
  };

  // ---- retire requests finishing at step k (+ window entry at k + H) ----
  // A completion calendar (a 64-bucket wheel in shared memory, or exact
  // buckets in the workspace for large G*B) holds, per owner lane, the slots
  // finishing in each bucket: a step touches only its completions (and, on
  // the wheel, entries a lap away), not every slot. Owner lanes retire in
  // registers; TPOT terms are buffered (x, k) and evaluated off the chain.
  auto retire = [&]() {
    const uint32_t kf = static_cast<uint32_t>(k);
    constexpr bool kWinPolicy = GREEDY && !NOISY;  // perfect/truncated finish window
    const bool win = kWinPolicy && H > 0;
    const uint32_t kh = win ? static_cast<uint32_t>(k + H) : kf;
    const int rk = win ? static_cast<int>(k % Hm) : 0;
    if (win) {
BFSIM_UNROLL_W
      for (int j = 0; j < WPL; ++j) {
        int g = lane + 32 * j;
        if (g < G) {
          s_Wc[rk * G + g] = 0;
          s_Wa[rk * G + g] = 0;
        }
      }
      __syncwarp();
    }
    auto slot_worker = [&](int slot) -> int {
      int g = static_cast<int>(static_cast<float>(slot) * invB);
      g -= (g * B > slot) ? 1 : 0;
      g += ((g + 1) * B <= slot) ? 1 : 0;
      return g;
    };
    {
      // Calendar: each lane walks its own lists (it owns every worker on
      // them, so worker state needs no atomics). Window entries first: the
      // slots finishing at k + H stay listed.
      const bool wheel = cal == 2;
      auto head_of = [&](long long kk) -> int32_t* {
        return wheel ? (lane < LS ? &calh[static_cast<int>(kk & (kWheel - 1)) * LS + lane] : nullptr)
                     : &calh[static_cast<int>(kk & Rm) * 32 + lane];
      };
      auto next_of = [&](int slot) -> int {
        if (wheel) {
          const uint16_t v = wnx[slot];
          return v == 0xFFFF ? -1 : static_cast<int>(v);
        }
        return calnx[slot];
      };
      if (win) {
        int32_t* hp = head_of(k + H);
        for (int s = hp ? *hp : -1; s >= 0; s = next_of(s)) {
          if (wheel && s_f[s] != kh) continue;
          const int g = slot_worker(s);
          s_Wc[rk * G + g] += 1;
          s_Wa[rk * G + g] += s_a[s];
        }
      }
      int32_t* hb = head_of(k);
      int s = hb ? *hb : -1;
      if (!wheel) *hb = -1;
      int prev = -1;
      int rc[WPL];
BFSIM_UNROLL_W
      for (int j = 0; j < WPL; ++j) rc[j] = 0;
      int nd = 0;
      while (__any_sync(FULLMASK, s >= 0)) {
        const int nx = s >= 0 ? next_of(s) : -1;
        const bool live = s >= 0 && (!wheel || s_f[s] == static_cast<uint32_t>(k));
        if (wheel && s >= 0 && !live) prev = s;  // a later lap: stays listed
        const unsigned am = __ballot_sync(FULLMASK, live);
        int base = 0;
        if (am) {
          const int leader = __ffs(am) - 1;
          if (lane == leader) base = atomicAdd(&s_misc[0], __popc(am));
          base = __shfl_sync(FULLMASK, base, leader);
        }
        if (!live) s = nx;
        if (live) {
          const int slot = s;
          s = nx;
          if (wheel) {  // unlink
            if (prev < 0) *hb = nx;
            else wnx[prev] = static_cast<uint16_t>(nx < 0 ? 0xFFFF : nx);
          }
          const int g = WPL == 1 ? lane : slot_worker(slot);  // the walking lane owns the slot's worker
          const int i = slot - g * B;
          const int jj = g >> 5;
          const long long av = s_a[slot];
          if constexpr (WPL > 8) {  // lane arrays in local memory: index directly
            A[jj] -= av;
            s_stk[g * B + B - n[jj] + rc[jj]] = static_cast<uint16_t>(i);
            rc[jj] += 1;
          } else {
#pragma unroll
            for (int j = 0; j < WPL; ++j)
              if (j == jj) {
                A[j] -= av;
                s_stk[g * B + B - n[j] + rc[j]] = static_cast<uint16_t>(i);
                rc[j] += 1;
              }
          }
          s_f[slot] = kEmpty;
          cbuf[base + __popc(am & lanemask_lt())] = make_int2(s_x[slot], static_cast<int>(k));
          if (emit_reqs) P.reqs.finish_clock[ro + s_id[slot]] = clock;
          ++nd;
        }
      }
      __syncwarp();
      // noisy: erase_if keeps insertion order (engine.hpp:118-120); the
      // finished entries stay in the worker lists until the next draw pass
      // walks and compacts them (gen_normals)
BFSIM_UNROLL_W
      for (int j = 0; j < WPL; ++j) {
        const int g = lane + 32 * j;
        if (g >= G || rc[j] == 0) continue;
        n[j] -= rc[j];
        s_cap[g] = B - n[j];
      }
      const long long ndw = static_cast<long long>(__reduce_add_sync(FULLMASK, static_cast<unsigned>(nd)));
      done += ndw;
      act -= ndw;
    }
  };

  // --- step loop -----------------------------------------------------------
  for (;;) {
    if (OVL) {
      if (k >= total_steps) break;
    } else {
      if (done == N) break;  // all_done(), engine.hpp:171
      if (k >= total_steps) {
        status = BFSIM_PARTIAL;
        break;
      }
    }
    if (k > k_safe) {
      status = BFSIM_ERANGE;
      break;
    }
    const double cs = clock;
    if (OVL) {
      if (!topup()) {
        status = BFSIM_ESTREAM;
        break;
      }
    } else {
      reveal();
    }
    const long long free_total = static_cast<long long>(G) * B - act;
    if (n_wait > 0 && free_total > 0) {
      int U = static_cast<int>(n_wait < free_total ? n_wait : free_total);
      if constexpr (GREEDY) {
        if (k32) admit_greedy(U, free_total, std::true_type{});
        else admit_greedy(U, free_total, std::false_type{});
      } else {
        admit_fifo(U);
      }
      n_wait -= U;
      act += U;
      adm_total += U;
      if (OVL) refresh_maxcount();
BFSIM_UNROLL_W
      for (int j = 0; j < WPL; ++j) {
        int g = lane + 32 * j;
        if (g < G) s_cap[g] = B - n[j];
      }
    } else if constexpr (NOISY) {
      gen_normals(act + n_wait, false);  // views are drawn every step (engine.hpp:131)
    }
    // loads, straggler max, dt, clock (engine.hpp:136-146)
    uint32_t lmax = 0;
    const int kr = static_cast<int>(k & 31);
BFSIM_UNROLL_W
    for (int j = 0; j < WPL; ++j) {
      int g = lane + 32 * j;
      if (g < G) {
        uint32_t L = static_cast<uint32_t>(A[j] + d * k * n[j]);
        r_l[kr * rstride + g] = L;
        lmax = L > lmax ? L : lmax;
      }
    }
    const uint32_t mx = __reduce_max_sync(FULLMASK, lmax);
    const double dt = __dadd_rn(C0, __dmul_rn(TL, static_cast<double>(mx)));
    clock = __dadd_rn(clock, dt);
    if (lane == 0) {
      r_dt[kr] = dt;
      r_cs[kr] = cs;
      r_mx[kr] = mx;
      r_ac[kr] = static_cast<int32_t>(act);
      ring[k & Rm] = cs;
    }
    __syncwarp();
    if (kr == 31) {
      flush(k - 31, 32);
    } else if (s_misc[0] > cbuf_cap - G * B) {
      drain_tpot();  // completion buffer nearly full: evaluate now (ring[k] is written)
    }
    if (act > 0 || (GREEDY && !NOISY && H > 0)) retire();
    ++k;
    prefetch_fifo();
  }
  if (SM) cp_async_wait_all();
  if (lane == 0) ring[k & Rm] = clock;  // clock_start of the (unsimulated) next step
  __syncwarp();
  if (k & 31) flush(k & ~31ll, static_cast<int>(k & 31));
  else drain_tpot();

  // unrevealed requests (partial runs)
  if (!OVL && emit_reqs)
    for (long long id = nxt + lane; id < N; id += 32) {
      P.reqs.arrival_step[ro + id] = -1;
      P.reqs.start_step[ro + id] = -1;
      P.reqs.worker[ro + id] = -1;
      P.reqs.admit_clock[ro + id] = 0.0;
      P.reqs.finish_clock[ro + id] = 0.0;
    }

  if (emit_reqs && P.reqs_host.start_step) {
    // this trajectory's request slice to the page-locked host mirror,
    // coalesced, while other trajectories are still running
    __syncwarp();
    __threadfence();
    const long long nreq = N;
    auto copy = [&](auto* dst, const auto* src) {  // 4 loads in flight per lane
      long long i = lane;
      for (; i + 96 < nreq; i += 128) {
        const auto v0 = __ldcg(src + ro + i), v1 = __ldcg(src + ro + i + 32);
        const auto v2 = __ldcg(src + ro + i + 64), v3 = __ldcg(src + ro + i + 96);
        dst[ro + i] = v0;
        dst[ro + i + 32] = v1;
        dst[ro + i + 64] = v2;
        dst[ro + i + 96] = v3;
      }
      for (; i < nreq; i += 32) dst[ro + i] = __ldcg(src + ro + i);
    };
    copy(P.reqs_host.arrival_step, P.reqs.arrival_step);
    copy(P.reqs_host.start_step, P.reqs.start_step);
    copy(P.reqs_host.worker, P.reqs.worker);
    copy(P.reqs_host.admit_clock, P.reqs.admit_clock);
    copy(P.reqs_host.finish_clock, P.reqs.finish_clock);
  }
  if (emit_steps && k > scap) flags |= BFSIM_FLAG_STEP_OVERFLOW;
  if (NOISY && __any_sync(FULLMASK, ntie)) flags |= BFSIM_FLAG_NOISE_NEAR_TIE;
  if (NOISY && lane == 0) st_release(&s_ctr[2], 1u);  // the producer warp stops
  if (lane == 0) {
    bfsim_result_t r;
    r.status = status;
    r.flags = flags;
    r.steps_run = k;
    r.records = records;
    r.completed = done;
    r.admitted = adm_total;
    r.consumed = OVL ? tail : nxt;
    r.imb_total_i = imb;
    r.total_workload_i = work;
    r.tokens_i = tok;
    r.clock = clock;
    r.elapsed = elapsed;
    r.tpot_sum = tpot_sum;
    if (records == 0) {
      r.flags |= BFSIM_FLAG_EMPTY;
      r.avg_imbalance = r.throughput = r.tpot = r.energy = 0.0;
      r.imb_total = r.total_workload = r.eta_sum = 0.0;
    } else {
      // compute_metrics, metrics.hpp:106-122
      r.avg_imbalance = static_cast<double>(imb) * lsc / static_cast<double>(records);
      r.throughput = static_cast<double>(tok) / elapsed;
      r.tpot = done > 0 ? tpot_sum / static_cast<double>(done) : 0.0;
      r.energy = energy;
      r.imb_total = static_cast<double>(imb) * lsc;
      r.total_workload = static_cast<double>(work) * lsc;
      r.eta_sum = work > 0 ? static_cast<double>(imb) / static_cast<double>(work) : 0.0;
    }
    P.results[si] = r;
  }
  __syncwarp();
}

// Noisy variants run two warps per trajectory (the simulation warp and the
// draw producer), <= 144 registers a thread so 7 trajectories share an SM.
template <int MODE, int POL, int WPL, bool SMALLC, bool SM, bool NOISY, int HR, bool WIDE = false>
__global__ void __launch_bounds__(NOISY ? 64 : (WIDE ? 256 : kWarpsPerCta * 32), NOISY ? 7 : 1) step_kernel(KParams P) {
  unsigned char* smem = bfsim_dsmem;
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  if constexpr (WIDE) {
    // one trajectory per CTA: warp 0 simulates, the other warps join its
    // placement chains (wide_chain)
    __shared__ int s_qi;
    __shared__ WideChain s_w;
    __shared__ unsigned long long s_red[8][2];
    unsigned char* sm = smem;
    unsigned char* ws = P.ws + static_cast<size_t>(blockIdx.x) * P.plan.ws_stride;
    const int nthreads = static_cast<int>(blockDim.x);
    for (;;) {
      if (threadIdx.x == 0) s_qi = atomicAdd(P.queue, 1);
      __syncthreads();
      const int qi = s_qi;
      if (qi >= P.n) break;
      if (warp == 0) {
        run_traj<MODE, POL, WPL, SMALLC, SM, NOISY, HR, WIDE>(P, P.order[qi], sm, ws, &s_w, s_red);
        if (lane == 0) s_w.cmd = 0;
        __threadfence_block();
        cta_bar(nthreads);  // the helper warps leave
      } else {
        for (;;) {
          cta_bar(nthreads);
          if (s_w.cmd == 0) break;
          wide_chain(s_w, s_red, nthreads);
        }
      }
      __syncthreads();
    }
  } else if constexpr (NOISY) {
    // one trajectory per CTA: warp 0 simulates, warp 1 produces its draws
    __shared__ int s_qi;
    unsigned char* sm = smem;
    unsigned char* ws = P.ws + static_cast<size_t>(blockIdx.x) * P.plan.ws_stride;
    unsigned* ctr = at<true, unsigned>(sm, ws, P.plan.o_misc) + 1;
    for (;;) {
      if (threadIdx.x == 0) {
        s_qi = atomicAdd(P.queue, 1);
        ctr[0] = ctr[1] = ctr[2] = 0u;
      }
      __syncthreads();
      const int qi = s_qi;
      if (qi >= P.n) break;
      const int si = P.order[qi];
      if (warp == 0) {
        run_traj<MODE, POL, WPL, SMALLC, SM, NOISY, HR>(P, si, sm, ws);
      } else {
        const bfsim_scenario_t& sc = P.scen[si];
        noisy_producer(at<true, uint64_t>(sm, ws, P.plan.o_mt), at<true, int>(sm, ws, P.plan.o_nring), ctr, sc.seed,
                       sc.noise_sigma);
      }
      __syncthreads();
    }
  } else {
    const int wpc = blockDim.x >> 5;
    unsigned char* sm = smem + static_cast<size_t>(warp) * P.plan.smem_per_warp;
    unsigned char* ws = P.ws + static_cast<size_t>(blockIdx.x * wpc + warp) * P.plan.ws_stride;
    for (;;) {
      int qi = 0;
      if (lane == 0) qi = atomicAdd(P.queue, 1);
      qi = __shfl_sync(FULLMASK, qi, 0);
      if (qi >= P.n) break;
      run_traj<MODE, POL, WPL, SMALLC, SM, NOISY, HR>(P, P.order[qi], sm, ws);
    }
  }
}

template <int MODE, int POL, int WPL, bool SMALLC, bool SM, bool NOISY, int HR, bool WIDE = false>
int launch_t(const KParams& kp, int grid, int wpc, cudaStream_t s, int* occ) {
  auto fn = step_kernel<MODE, POL, WPL, SMALLC, SM, NOISY, HR, WIDE>;
  // noisy / wide: one trajectory (arena) per CTA of several warps
  size_t smem = static_cast<size_t>(kp.plan.smem_per_warp) * ((NOISY || WIDE) ? 1 : wpc);
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem));
  if (e != cudaSuccess) return static_cast<int>(e);
  if (occ) {  // occupancy query only
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(occ, fn, wpc * 32, smem);
    return static_cast<int>(e);
  }
  fn<<<grid, wpc * 32, smem, s>>>(kp);
  return static_cast<int>(cudaGetLastError());
}

// hr: register lookahead chain width (0 = shared-memory chain); the planner
// picks hr in {8, 24} only for bfio-greedy with H < hr and G <= 64.
template <int MODE, int POL, bool SMALLC, bool SM, bool NOISY>
int launch_w(int wpl, int hr, const KParams& kp, int grid, int wpc, cudaStream_t s, int* occ) {
  if constexpr (POL == BFSIM_POLICY_BFIO_GREEDY) {
    if (hr == 8 && wpl == 1) return launch_t<MODE, POL, 1, SMALLC, SM, NOISY, 8>(kp, grid, wpc, s, occ);
    if (hr == 8 && wpl == 2) return launch_t<MODE, POL, 2, SMALLC, SM, NOISY, 8>(kp, grid, wpc, s, occ);
    if (hr == 24 && wpl == 1) return launch_t<MODE, POL, 1, SMALLC, SM, NOISY, 24>(kp, grid, wpc, s, occ);
    if (hr == 24 && wpl == 2) return launch_t<MODE, POL, 2, SMALLC, SM, NOISY, 24>(kp, grid, wpc, s, occ);
    if (hr == 8 && wpl == 4) return launch_t<MODE, POL, 4, SMALLC, SM, NOISY, 8>(kp, grid, wpc, s, occ);
    if (hr == 24 && wpl == 4) return launch_t<MODE, POL, 4, SMALLC, SM, NOISY, 24>(kp, grid, wpc, s, occ);
  }
  if (hr != 0) return static_cast<int>(cudaErrorInvalidValue);
  switch (wpl) {
    case 1: return launch_t<MODE, POL, 1, SMALLC, SM, NOISY, 0>(kp, grid, wpc, s, occ);
    case 2: return launch_t<MODE, POL, 2, SMALLC, SM, NOISY, 0>(kp, grid, wpc, s, occ);
    case 4: return launch_t<MODE, POL, 4, SMALLC, SM, NOISY, 0>(kp, grid, wpc, s, occ);
    case 8: return launch_t<MODE, POL, 8, SMALLC, SM, NOISY, 0>(kp, grid, wpc, s, occ);
    case 16: return launch_t<MODE, POL, 16, SMALLC, SM, NOISY, 0>(kp, grid, wpc, s, occ);
    case 32: return launch_t<MODE, POL, 32, SMALLC, SM, NOISY, 0>(kp, grid, wpc, s, occ);
  }
  return static_cast<int>(cudaErrorInvalidValue);
}

// Wide trajectories (G > 128, bfio-greedy with a window, not noisy): own units.
template <int MODE, int POL, bool SMALLC>
int launch_wide(int wpl, const KParams& kp, int grid, int wpc, cudaStream_t s, int* occ) {
  const bool sm = kp.plan.all_smem != 0;
  switch (wpl) {
    case 8:
      return sm ? launch_t<MODE, POL, 8, SMALLC, true, false, 0, true>(kp, grid, wpc, s, occ)
                : launch_t<MODE, POL, 8, SMALLC, false, false, 0, true>(kp, grid, wpc, s, occ);
    case 16:
      return sm ? launch_t<MODE, POL, 16, SMALLC, true, false, 0, true>(kp, grid, wpc, s, occ)
                : launch_t<MODE, POL, 16, SMALLC, false, false, 0, true>(kp, grid, wpc, s, occ);
    case 32:
      return sm ? launch_t<MODE, POL, 32, SMALLC, true, false, 0, true>(kp, grid, wpc, s, occ)
                : launch_t<MODE, POL, 32, SMALLC, false, false, 0, true>(kp, grid, wpc, s, occ);
  }
  return static_cast<int>(cudaErrorInvalidValue);
}

// One instantiation unit per (mode, policy, class-set kind, noisy): both
// arena placements (all-shared / spilled) and every workers-per-lane width.
template <int MODE, int POL, bool SMALLC, bool NOISY>
int launch_unit(int wpl, int hr, const KParams& kp, int grid, int wpc, cudaStream_t s, int* occ) {
  return kp.plan.all_smem ? launch_w<MODE, POL, SMALLC, true, NOISY>(wpl, hr, kp, grid, wpc, s, occ)
                          : launch_w<MODE, POL, SMALLC, false, NOISY>(wpl, hr, kp, grid, wpc, s, occ);
}

}  // namespace detail

// Declarations of the instantiation units (engine_<mode>_<policy>*.cu).
// Only bfio-greedy uses the class bitmaps, so the FIFO units take SMALLC = true.
#define BFSIM_DECLARE_UNIT(NAME) \
  int NAME(int wpl, int hr, const KParams& kp, int grid, int wpc, cudaStream_t s, int* occ);
#define BFSIM_DEFINE_UNIT(NAME, M, P, SMALLC, NOISY)                                          \
  int NAME(int wpl, int hr, const KParams& kp, int grid, int wpc, cudaStream_t s, int* occ) {  \
    return detail::launch_unit<M, P, SMALLC, NOISY>(wpl, hr, kp, grid, wpc, s, occ);          \
  }
BFSIM_DECLARE_UNIT(launch_poisson_fcfs)
BFSIM_DECLARE_UNIT(launch_poisson_jsq)
BFSIM_DECLARE_UNIT(launch_poisson_greedy_small)
BFSIM_DECLARE_UNIT(launch_poisson_greedy_large)
BFSIM_DECLARE_UNIT(launch_poisson_greedy_noisy_small)
BFSIM_DECLARE_UNIT(launch_poisson_greedy_noisy_large)
BFSIM_DECLARE_UNIT(launch_overloaded_fcfs)
BFSIM_DECLARE_UNIT(launch_overloaded_jsq)
BFSIM_DECLARE_UNIT(launch_overloaded_greedy_small)
BFSIM_DECLARE_UNIT(launch_overloaded_greedy_large)
#define BFSIM_DECLARE_WIDE_UNIT(NAME) \
  int NAME(int wpl, const KParams& kp, int grid, int wpc, cudaStream_t s, int* occ);
#define BFSIM_DEFINE_WIDE_UNIT(NAME, M, SMALLC)                                         \
  int NAME(int wpl, const KParams& kp, int grid, int wpc, cudaStream_t s, int* occ) { \
    return detail::launch_wide<M, BFSIM_POLICY_BFIO_GREEDY, SMALLC>(wpl, kp, grid, wpc, s, occ); \
  }
BFSIM_DECLARE_WIDE_UNIT(launch_poisson_greedy_wide_small)
BFSIM_DECLARE_WIDE_UNIT(launch_poisson_greedy_wide_large)
BFSIM_DECLARE_WIDE_UNIT(launch_overloaded_greedy_wide_small)
BFSIM_DECLARE_WIDE_UNIT(launch_overloaded_greedy_wide_large)

}  // namespace bfsim
