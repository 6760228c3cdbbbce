// Host side of the batched step engine: the synthetic scenario/trace batcher
// and the IIR reducer. Plain C++ (compiled by nvcc's host compiler into
// libbfsim_gpu.so); no device code here.
//
// Traces and overloaded sample streams are generated with libstdc++'s own
// <random> engines and distributions, making them byte-identical to what the
// reference draws (SURVEY.md §2 "Synthetic generators"; north_star: traces are
// "pre-generated synthetically on the host and shared byte-for-byte").
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <limits>
#include <random>
#include <vector>

#include "bfsim_gpu.h"
#include "common.h"

namespace {

// PrefillDistribution::sample (workload.hpp:120-128): Uniform, Fixed, Empirical.
struct Prefill {
  int kind, s_max;
  const int64_t* values = nullptr;
  int64_t n_values = 0;
  int sample(std::mt19937_64& rng) const {
    if (kind == 1) return s_max;
    if (kind == 2)
      return static_cast<int>(values[std::uniform_int_distribution<std::size_t>(
          0, static_cast<std::size_t>(n_values) - 1)(rng)]);
    return std::uniform_int_distribution<int>(1, s_max)(rng);
  }
};
// DecodeDistribution::sample (workload.hpp:195-204): Geometric, Fixed, Empirical.
struct Decode {
  int kind;
  double p;
  int64_t fixed;
  const int64_t* values = nullptr;
  int64_t n_values = 0;
  long sample(std::mt19937_64& rng) const {
    if (kind == 1) return static_cast<long>(fixed);
    if (kind == 2)
      return static_cast<long>(values[std::uniform_int_distribution<std::size_t>(
          0, static_cast<std::size_t>(n_values) - 1)(rng)]);
    return 1 + std::geometric_distribution<long>(p)(rng);
  }
};

int check_dists(int prefill_kind, int s_max, int decode_kind, double p, int64_t fixed_o,
                char* err, size_t errlen) {
  // Validation mirrors PrefillDistribution::uniform / fixed_value (workload.hpp:94-108)
  // and DecodeDistribution::geometric / fixed_length (:171-184).
  if (prefill_kind != 0 && prefill_kind != 1)
    return bfsim::fail(err, errlen, BFSIM_EINVAL, "prefill: unknown distribution kind");
  if (s_max < 1)
    return bfsim::fail(err, errlen, BFSIM_EINVAL,
                       prefill_kind ? "prefill: fixed value must be >= 1"
                                    : "prefill: s_max must be >= 1");
  if (decode_kind == 0 && !(p > 0.0 && p < 1.0))
    return bfsim::fail(err, errlen, BFSIM_EINVAL, "decode: p must be in (0,1)");
  if (decode_kind == 1 && fixed_o < 1)
    return bfsim::fail(err, errlen, BFSIM_EINVAL, "decode: fixed length must be >= 1");
  if (decode_kind != 0 && decode_kind != 1)
    return bfsim::fail(err, errlen, BFSIM_EINVAL, "decode: unknown distribution kind");
  return BFSIM_OK;
}

// Descriptor -> sampler, validated as the reference's factories do
// (PrefillDistribution::empirical workload.hpp:109-118, DecodeDistribution::
// empirical :185-193: empty list, value < 1).
int make_dists(const bfsim_dist_t* pd, const bfsim_dist_t* dd, Prefill* pf, Decode* dc, char* err, size_t errlen) {
  if (!pd || !dd) return bfsim::fail(err, errlen, BFSIM_EINVAL, "null distribution");
  if (pd->kind == 2) {
    if (!pd->values || pd->n_values < 1)
      return bfsim::fail(err, errlen, BFSIM_EINVAL, "prefill: empty empirical list");
    int64_t mx = 0;
    for (int64_t i = 0; i < pd->n_values; ++i) {
      if (pd->values[i] < 1) return bfsim::fail(err, errlen, BFSIM_EINVAL, "prefill: empirical value < 1");
      if (pd->values[i] > BFSIM_MAX_CLASSES)
        return bfsim::fail(err, errlen, BFSIM_EINVAL, "prefill: empirical value exceeds the GPU class limit");
      mx = std::max(mx, pd->values[i]);
    }
    *pf = Prefill{2, static_cast<int>(mx), pd->values, pd->n_values};
  } else {
    if (pd->fixed > std::numeric_limits<int>::max())
      return bfsim::fail(err, errlen, BFSIM_EINVAL, "prefill: value exceeds int");
    int rc = check_dists(pd->kind, static_cast<int>(pd->fixed), 0, 0.5, 1, err, errlen);
    if (rc) return rc;
    *pf = Prefill{pd->kind, static_cast<int>(pd->fixed)};
  }
  if (dd->kind == 2) {
    if (!dd->values || dd->n_values < 1)
      return bfsim::fail(err, errlen, BFSIM_EINVAL, "decode: empty empirical list");
    for (int64_t i = 0; i < dd->n_values; ++i) {
      if (dd->values[i] < 1) return bfsim::fail(err, errlen, BFSIM_EINVAL, "decode: empirical value < 1");
      if (dd->values[i] > std::numeric_limits<int32_t>::max())
        return bfsim::fail(err, errlen, BFSIM_EINVAL, "decode: empirical value exceeds int32");
    }
    *dc = Decode{2, 0.0, 0, dd->values, dd->n_values};
  } else {
    int rc = check_dists(0, 1, dd->kind, dd->p, dd->fixed, err, errlen);
    if (rc) return rc;
    *dc = Decode{dd->kind, dd->p, dd->fixed};
  }
  return BFSIM_OK;
}

// sample_instance, workload.hpp:241-266: exponential gaps, then prefill, then
// decode per arrival, all from one mt19937_64(seed).
int sample_instance_impl(const Prefill& pf, const Decode& dc, double rate, double duration, uint64_t seed,
                         bfsim_request_t* out, int64_t capacity, int64_t* n_out, char* err, size_t errlen) {
  if (rate <= 0.0) return bfsim::fail(err, errlen, BFSIM_EINVAL, "sample_instance: rate must be > 0");
  if (duration <= 0.0)
    return bfsim::fail(err, errlen, BFSIM_EINVAL, "sample_instance: duration must be > 0");
  std::mt19937_64 rng(seed);
  std::exponential_distribution<double> gap(rate);
  double t = gap(rng);
  int64_t n = 0;
  while (t < duration) {
    int s = pf.sample(rng);
    long o = dc.sample(rng);
    if (o > std::numeric_limits<int32_t>::max())
      return bfsim::fail(err, errlen, BFSIM_EINVAL, "sample_instance: decode exceeds int32");
    if (out && n < capacity) {
      out[n].arrival_time = t;
      out[n].prefill = s;
      out[n].decode = static_cast<int32_t>(o);
    }
    ++n;
    t += gap(rng);
  }
  *n_out = n;
  return BFSIM_OK;
}

// run_overloaded's top-up draws prefill then decode per pending request
// (oracle.hpp:177-183) from mt19937_64(seed), independent of the policy.
int sample_stream_impl(const Prefill& pf, const Decode& dc, uint64_t seed, int64_t n, bfsim_sample_t* out,
                       char* err, size_t errlen) {
  std::mt19937_64 rng(seed);
  for (int64_t i = 0; i < n; ++i) {
    int s = pf.sample(rng);
    long o = dc.sample(rng);
    if (o > std::numeric_limits<int32_t>::max())
      return bfsim::fail(err, errlen, BFSIM_EINVAL, "sample_stream: decode exceeds int32");
    out[i].prefill = s;
    out[i].decode = static_cast<int32_t>(o);
  }
  return BFSIM_OK;
}

template <class Rec>
int prepare(const Rec* rec, int64_t n, bfsim_input_t* info, int32_t* class_base, char* err,
            size_t errlen) {
  int32_t s_max = 1, max_o = 1;
  for (int64_t i = 0; i < n; ++i) {
    if (rec[i].prefill < 1 || rec[i].decode < 1)
      return bfsim::fail(err, errlen, BFSIM_EINVAL, "input: prefill and decode must be >= 1");
    s_max = std::max(s_max, rec[i].prefill);
    max_o = std::max(max_o, rec[i].decode);
  }
  if (s_max > BFSIM_MAX_CLASSES)
    return bfsim::fail(err, errlen, BFSIM_EINVAL, "input: prefill exceeds the GPU class limit");
  info->offset = 0;
  info->length = n;
  info->class_base_offset = 0;
  info->s_max = s_max;
  info->max_decode = max_o;
  if (class_base) {
    // counting-sort layout: class_base[c] = #records with prefill < c (c = 1..s_max+1)
    std::vector<int64_t> cnt(static_cast<size_t>(s_max) + 2, 0);
    for (int64_t i = 0; i < n; ++i) cnt[rec[i].prefill] += 1;
    int64_t acc = 0;
    class_base[0] = 0;
    for (int c = 1; c <= s_max + 1; ++c) {
      class_base[c] = static_cast<int32_t>(acc);
      if (c <= s_max) acc += cnt[c];
    }
  }
  return BFSIM_OK;
}

}  // namespace

extern "C" {

int bfsim_abi_version(void) { return BFSIM_ABI_VERSION; }

int bfsim_sample_instance(int prefill_kind, int s_max, int decode_kind, double p, int64_t fixed_o,
                          double rate, double duration, uint64_t seed, bfsim_request_t* out,
                          int64_t capacity, int64_t* n_out, char* err, size_t errlen) {
  int rc = check_dists(prefill_kind, s_max, decode_kind, p, fixed_o, err, errlen);
  if (rc) return rc;
  return sample_instance_impl(Prefill{prefill_kind, s_max}, Decode{decode_kind, p, fixed_o}, rate, duration, seed,
                              out, capacity, n_out, err, errlen);
}

int bfsim_sample_instance_dist(const bfsim_dist_t* prefill, const bfsim_dist_t* decode, double rate,
                               double duration, uint64_t seed, bfsim_request_t* out, int64_t capacity,
                               int64_t* n_out, char* err, size_t errlen) {
  Prefill pf{0, 1};
  Decode dc{0, 0.5, 1};
  int rc = make_dists(prefill, decode, &pf, &dc, err, errlen);
  if (rc) return rc;
  return sample_instance_impl(pf, dc, rate, duration, seed, out, capacity, n_out, err, errlen);
}

int bfsim_sample_stream(int prefill_kind, int s_max, int decode_kind, double p, int64_t fixed_o,
                        uint64_t seed, int64_t n, bfsim_sample_t* out, char* err, size_t errlen) {
  int rc = check_dists(prefill_kind, s_max, decode_kind, p, fixed_o, err, errlen);
  if (rc) return rc;
  return sample_stream_impl(Prefill{prefill_kind, s_max}, Decode{decode_kind, p, fixed_o}, seed, n, out, err, errlen);
}

int bfsim_sample_stream_dist(const bfsim_dist_t* prefill, const bfsim_dist_t* decode, uint64_t seed, int64_t n,
                             bfsim_sample_t* out, char* err, size_t errlen) {
  Prefill pf{0, 1};
  Decode dc{0, 0.5, 1};
  int rc = make_dists(prefill, decode, &pf, &dc, err, errlen);
  if (rc) return rc;
  return sample_stream_impl(pf, dc, seed, n, out, err, errlen);
}

int bfsim_prepare_trace(const bfsim_request_t* rec, int64_t n, bfsim_input_t* info,
                        int32_t* class_base, char* err, size_t errlen) {
  for (int64_t i = 1; i < n; ++i)
    if (!(rec[i].arrival_time >= rec[i - 1].arrival_time))
      return bfsim::fail(err, errlen, BFSIM_EINVAL, "trace: arrivals must be sorted");
  if (n > 0 && !(rec[0].arrival_time >= 0.0))
    return bfsim::fail(err, errlen, BFSIM_EINVAL, "trace: negative arrival time");
  return prepare(rec, n, info, class_base, err, errlen);
}

int bfsim_prepare_stream(const bfsim_sample_t* smp, int64_t n, bfsim_input_t* info,
                         int32_t* class_base, char* err, size_t errlen) {
  return prepare(smp, n, info, class_base, err, errlen);
}

// estimate_iir reduction, oracle.hpp:290-312: mean, SEM with n-1, ratio and
// propagated relative stderr; infinite ratio when the BF-IO mean is <= 0.
int bfsim_iir_reduce(const double* fcfs, const double* bfio, int32_t trials, int32_t n_cells,
                     double* out, char* err, size_t errlen) {
  if (trials < 1) return bfsim::fail(err, errlen, BFSIM_EINVAL, "estimate_iir: trials must be >= 1");
  auto mean = [&](const double* v) {
    double m = 0.0;
    for (int32_t t = 0; t < trials; ++t) m += v[t];
    return m / static_cast<double>(trials);
  };
  auto sem = [&](const double* v) {
    if (trials < 2) return 0.0;
    double m = mean(v), acc = 0.0;
    for (int32_t t = 0; t < trials; ++t) acc += (v[t] - m) * (v[t] - m);
    return std::sqrt(acc / static_cast<double>(trials - 1)) / std::sqrt(static_cast<double>(trials));
  };
  for (int32_t c = 0; c < n_cells; ++c) {
    const double* f = fcfs + static_cast<int64_t>(c) * trials;
    const double* b = bfio + static_cast<int64_t>(c) * trials;
    double fm = mean(f), bm = mean(b), ratio, se;
    if (bm <= 0.0) {
      ratio = std::numeric_limits<double>::infinity();
      se = std::numeric_limits<double>::infinity();
    } else {
      ratio = fm / bm;
      double rf = sem(f) / fm;
      double rb = sem(b) / bm;
      se = ratio * std::sqrt(rf * rf + rb * rb);
    }
    out[4 * c + 0] = fm;
    out[4 * c + 1] = bm;
    out[4 * c + 2] = ratio;
    out[4 * c + 3] = se;
  }
  return BFSIM_OK;
}

}  // extern "C"
