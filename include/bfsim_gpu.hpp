// bfsim_gpu.hpp — reference-shaped C++ adapter over the C ABI (bfsim_gpu.h).
//
// Include AFTER the reference headers (bfsim/engine.hpp, bfsim/oracle.hpp):
// it speaks the reference's own types (SimConfig, ArrivalInstance, SimResult,
// StepRecord, RequestTiming, OverloadedSpec, IirEstimate) so a call site of
//
//   SimResult bfsim::run(const SimConfig&, const ArrivalInstance&)            engine.hpp:265
//   std::vector<StepRecord> bfsim::run_overloaded(...)                         oracle.hpp:138-143
//   IirEstimate bfsim::estimate_iir(...)                                       oracle.hpp:263-266
//
// switches to the GPU by prefixing `gpu::` and passing a context. Errors are
// rethrown as the reference's exception types (std::invalid_argument,
// std::logic_error); CUDA failures as std::runtime_error. Batched entry
// points (run_batch, estimate_iir) are where the GPU pays off: one call
// simulates every trajectory concurrently.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <limits>
#include <memory>
#include <random>
#include <stdexcept>
#include <string>
#include <tuple>
#include <vector>

#include "bfsim_gpu.h"

namespace bfsim {
namespace gpu {

inline void check(int rc, const char* err) {
  if (rc == BFSIM_OK || rc == BFSIM_PARTIAL) return;
  if (rc == BFSIM_EINVAL) throw std::invalid_argument(err);
  if (rc == BFSIM_ELOGIC) throw std::logic_error(err);
  if (rc == BFSIM_ERANGE) throw std::overflow_error(err);
  throw std::runtime_error(std::string("bfsim_gpu: ") + err);
}

// One CUDA device. Not thread-safe: one Context per host thread.
class Context {
 public:
  explicit Context(int device = 0) {
    char err[512] = {0};
    check(bfsim_ctx_create(device, &h_, err, sizeof err), err);
  }
  ~Context() { bfsim_ctx_destroy(h_); }
  Context(const Context&) = delete;
  Context& operator=(const Context&) = delete;
  bfsim_ctx_t* get() const { return h_; }

 private:
  bfsim_ctx_t* h_ = nullptr;
};

namespace detail {

inline double constant_drift(const DriftSpec& d) {
  if (d.kind != DriftSpec::Kind::Constant)
    throw std::invalid_argument("bfsim_gpu: only constant drift runs on the GPU path");
  return d.value;
}

inline bfsim_scenario_t scenario_of(const SimConfig& c, double drift, int input_id) {
  bfsim_scenario_t s{};
  s.mode = BFSIM_MODE_POISSON;
  s.policy = static_cast<int32_t>(c.policy);
  s.lookahead = static_cast<int32_t>(c.lookahead);
  s.workers = c.workers;
  s.batch = c.batch;
  s.horizon = c.horizon;
  s.input_id = input_id;
  s.drift = drift;
  s.overhead = c.overhead;
  s.per_token = c.per_token;
  s.noise_sigma = c.noise_sigma;
  s.p_idle = c.power.p_idle;
  s.p_max = c.power.p_max;
  s.mfu_sat = c.power.mfu_sat;
  s.gamma = c.power.gamma;
  s.backlog = 1.0;
  s.max_steps = c.max_steps;
  s.seed = c.seed;
  return s;
}

// Heuristic step capacity; run_batch re-runs overflowing scenarios exactly.
inline int64_t step_guess(const SimConfig& c, const std::vector<bfsim_request_t>& r) {
  if (r.empty()) return 1;
  int64_t work = 0, max_o = 0;
  for (const auto& x : r) {
    work += x.decode;
    max_o = std::max<int64_t>(max_o, x.decode);
  }
  int64_t span = static_cast<int64_t>(r.back().arrival_time / std::max(c.overhead, 1e-6));
  int64_t g = span + 3 * work / (2 * std::max<int64_t>(1, int64_t(c.workers) * c.batch)) + max_o + 64;
  return std::min<int64_t>(g, c.max_steps);
}

// Rebuild the reference's per-step id lists from per-request assignments:
// admitted in waiting-index (= id) order (engine.hpp:235-248); completed
// worker-major, then active insertion order (engine.hpp:149-156).
inline void fill_lists(std::vector<StepRecord>& steps, const std::vector<RequestTiming>& rq,
                       const std::vector<int32_t>& worker) {
  const int64_t K = static_cast<int64_t>(steps.size());
  std::vector<std::tuple<long, int, long, int>> fin;
  for (size_t i = 0; i < rq.size(); ++i) {
    const auto& t = rq[i];
    if (t.start_step >= 0 && t.start_step < K) steps[t.start_step].admitted.push_back(t.id);
    if (t.completed) {
      long f = t.start_step + t.decode_steps - 1;
      if (f < K) fin.emplace_back(f, worker[i], t.start_step, t.id);
    }
  }
  std::sort(fin.begin(), fin.end());
  for (const auto& [f, g, x, id] : fin) steps[f].completed.push_back(id);
}

}  // namespace detail

// Batched Simulation::run (engine.hpp:168-188) over independent trajectories.
inline std::vector<SimResult> run_batch(Context& ctx, const std::vector<SimConfig>& cfgs,
                                        const std::vector<const ArrivalInstance*>& insts) {
  if (cfgs.size() != insts.size()) throw std::invalid_argument("run_batch: size mismatch");
  const size_t n = cfgs.size();
  char err[1024] = {0};
  // inputs
  std::vector<std::vector<bfsim_request_t>> recs(n);
  std::vector<bfsim_input_t> inputs(n);
  std::vector<int32_t> cbase;
  std::vector<bfsim_request_t> pool;
  std::vector<bfsim_scenario_t> scen(n);
  for (size_t i = 0; i < n; ++i) {
    cfgs[i].validate();
    const auto& in = *insts[i];
    recs[i].resize(in.requests.size());
    for (size_t j = 0; j < in.requests.size(); ++j) {
      if (in.requests[j].decode > std::numeric_limits<int32_t>::max())
        throw std::invalid_argument("bfsim_gpu: decode exceeds int32");
      recs[i][j] = {in.requests[j].arrival_time, in.requests[j].prefill,
                    static_cast<int32_t>(in.requests[j].decode)};
    }
    bfsim_input_t info{};
    check(bfsim_prepare_trace(recs[i].data(), static_cast<int64_t>(recs[i].size()), &info, nullptr,
                              err, sizeof err),
          err);
    std::vector<int32_t> cb(static_cast<size_t>(info.s_max) + 2);
    check(bfsim_prepare_trace(recs[i].data(), static_cast<int64_t>(recs[i].size()), &info, cb.data(),
                              err, sizeof err),
          err);
    info.offset = static_cast<int64_t>(pool.size());
    info.class_base_offset = static_cast<int64_t>(cbase.size());
    inputs[i] = info;
    pool.insert(pool.end(), recs[i].begin(), recs[i].end());
    cbase.insert(cbase.end(), cb.begin(), cb.end());
    scen[i] = detail::scenario_of(cfgs[i], detail::constant_drift(in.drift), static_cast<int>(i));
  }
  std::vector<int64_t> cap(n);
  for (size_t i = 0; i < n; ++i) cap[i] = detail::step_guess(cfgs[i], recs[i]);
  std::vector<bfsim_result_t> res(n);
  std::vector<double> cs, dt, mx, loads, ac_clock, fin_clock;
  std::vector<int64_t> ac;
  std::vector<int32_t> arr_step, start, worker;
  for (int attempt = 0; attempt < 2; ++attempt) {
    int64_t nrec = 0, nload = 0, nreq = 0;
    for (size_t i = 0; i < n; ++i) {
      scen[i].step_offset = nrec;
      scen[i].step_capacity = cap[i];
      scen[i].load_offset = nload;
      scen[i].req_offset = nreq;
      nrec += cap[i];
      nload += cap[i] * cfgs[i].workers;
      nreq += static_cast<int64_t>(recs[i].size());
    }
    cs.assign(nrec, 0.0);
    dt.assign(nrec, 0.0);
    mx.assign(nrec, 0.0);
    ac.assign(nrec, 0);
    loads.assign(std::max<int64_t>(nload, 1), 0.0);
    arr_step.assign(std::max<int64_t>(nreq, 1), -1);
    start.assign(std::max<int64_t>(nreq, 1), -1);
    worker.assign(std::max<int64_t>(nreq, 1), -1);
    ac_clock.assign(std::max<int64_t>(nreq, 1), 0.0);
    fin_clock.assign(std::max<int64_t>(nreq, 1), 0.0);
    bfsim_step_sink_t ss{cs.data(), dt.data(), mx.data(), ac.data(), loads.data()};
    bfsim_req_sink_t rs{arr_step.data(), start.data(), worker.data(), ac_clock.data(),
                        fin_clock.data()};
    check(bfsim_run_batch(ctx.get(), scen.data(), static_cast<int64_t>(n), inputs.data(),
                          static_cast<int32_t>(n), cbase.data(), static_cast<int64_t>(cbase.size()),
                          pool.data(), static_cast<int64_t>(pool.size()), nullptr, 0, &ss, nrec,
                          nload, &rs, nreq, res.data(), err, sizeof err),
          err);
    bool again = false;
    for (size_t i = 0; i < n; ++i)
      if (res[i].flags & BFSIM_FLAG_STEP_OVERFLOW) {
        cap[i] = std::max<int64_t>(res[i].steps_run, 1);
        again = true;
      }
    if (!again) break;
  }
  std::vector<SimResult> out(n);
  for (size_t i = 0; i < n; ++i) {
    SimResult& r = out[i];
    r.config = cfgs[i];
    r.completed_all = res[i].status == BFSIM_OK;
    const int64_t K = res[i].steps_run;
    const int G = cfgs[i].workers;
    r.steps.resize(static_cast<size_t>(K));
    for (int64_t k = 0; k < K; ++k) {
      StepRecord& s = r.steps[k];
      const int64_t o = scen[i].step_offset + k;
      s.k = k;
      s.clock_start = cs[o];
      s.dt = dt[o];
      s.max_load = mx[o];
      s.active_count = ac[o];
      s.loads.assign(loads.begin() + scen[i].load_offset + k * G,
                     loads.begin() + scen[i].load_offset + (k + 1) * G);
    }
    const int64_t N = static_cast<int64_t>(recs[i].size());
    std::vector<int32_t> wk(N);
    r.requests.resize(N);
    for (int64_t j = 0; j < N; ++j) {
      const int64_t o = scen[i].req_offset + j;
      RequestTiming& t = r.requests[j];
      t.id = static_cast<int>(j);
      t.arrival_time = recs[i][j].arrival_time;
      t.arrival_step = arr_step[o];
      t.start_step = start[o];
      t.admit_clock = ac_clock[o];
      t.finish_clock = fin_clock[o];
      t.decode_steps = recs[i][j].decode;
      t.completed = start[o] >= 0 && start[o] + recs[i][j].decode - 1 < K;
      wk[j] = worker[o];
    }
    detail::fill_lists(r.steps, r.requests, wk);
  }
  return out;
}

// Simulation::run on the GPU (engine.hpp:265).
inline SimResult run(Context& ctx, const SimConfig& config, const ArrivalInstance& instance) {
  return std::move(run_batch(ctx, {config}, {&instance}).front());
}

struct OverloadedJob {
  PolicyKind policy;
  int H, G, B;
  long steps, warmup;
  std::uint64_t seed;
};

// Batched run_overloaded (oracle.hpp:138-244). The (s, o) draws the
// reference makes from mt19937_64(seed) (oracle.hpp:177-183) are generated
// here with the spec's own distributions; their order is policy-independent
// (SURVEY F11), so every job sharing a seed shares the stream.
inline std::vector<std::vector<StepRecord>> run_overloaded_batch(
    Context& ctx, const std::vector<OverloadedJob>& jobs, const OverloadedSpec& spec,
    const PowerModel& power, std::vector<std::vector<RequestTiming>>* timings = nullptr,
    std::vector<MetricsReport>* metrics = nullptr) {
  const size_t n = jobs.size();
  char err[1024] = {0};
  const double drift = detail::constant_drift(spec.drift);
  std::vector<int64_t> len(n);
  for (size_t i = 0; i < n; ++i) {
    const auto& j = jobs[i];
    double p = spec.decode.mean() > 0 ? 1.0 / spec.decode.mean() : 0.02;
    len[i] = static_cast<int64_t>(j.G) * j.B * (3 + static_cast<int64_t>((j.steps + j.warmup) * p * 1.5)) +
             4096;
  }
  std::vector<bfsim_result_t> res(n);
  std::vector<bfsim_scenario_t> scen(n);
  std::vector<double> cs, dt, mx, loads, ac_clock, fin_clock;
  std::vector<int64_t> ac;
  std::vector<int32_t> arr_step, start, worker;
  std::vector<std::vector<bfsim_sample_t>> streams(n);
  for (int attempt = 0; attempt < 8; ++attempt) {
    std::vector<bfsim_sample_t> pool;
    std::vector<bfsim_input_t> inputs(n);
    std::vector<int32_t> cbase;
    int64_t nrec = 0, nload = 0, nreq = 0;
    for (size_t i = 0; i < n; ++i) {
      const auto& j = jobs[i];
      auto& st = streams[i];
      if (static_cast<int64_t>(st.size()) < len[i]) {
        std::mt19937_64 rng(j.seed);
        st.resize(static_cast<size_t>(len[i]));
        for (auto& x : st) {
          x.prefill = spec.prefill.sample(rng);
          x.decode = static_cast<int32_t>(spec.decode.sample(rng));
        }
      }
      bfsim_input_t info{};
      check(bfsim_prepare_stream(st.data(), static_cast<int64_t>(st.size()), &info, nullptr, err,
                                 sizeof err),
            err);
      info.s_max = std::max(info.s_max, spec.prefill.s_max);
      std::vector<int32_t> cb(static_cast<size_t>(info.s_max) + 2);
      check(bfsim_prepare_stream(st.data(), static_cast<int64_t>(st.size()), &info, cb.data(), err,
                                 sizeof err),
            err);
      info.s_max = std::max(info.s_max, spec.prefill.s_max);
      cb.resize(static_cast<size_t>(info.s_max) + 2, static_cast<int32_t>(st.size()));
      info.offset = static_cast<int64_t>(pool.size());
      info.class_base_offset = static_cast<int64_t>(cbase.size());
      inputs[i] = info;
      pool.insert(pool.end(), st.begin(), st.end());
      cbase.insert(cbase.end(), cb.begin(), cb.end());
      bfsim_scenario_t s{};
      s.mode = BFSIM_MODE_OVERLOADED;
      s.policy = static_cast<int32_t>(j.policy);
      s.workers = j.G;
      s.batch = j.B;
      s.horizon = j.H;
      s.input_id = static_cast<int32_t>(i);
      s.drift = drift;
      s.overhead = spec.overhead;
      s.per_token = spec.per_token;
      s.p_idle = power.p_idle;
      s.p_max = power.p_max;
      s.mfu_sat = power.mfu_sat;
      s.gamma = power.gamma;
      s.backlog = spec.backlog;
      s.steps = j.steps;
      s.warmup = j.warmup;
      s.seed = j.seed;
      s.step_offset = nrec;
      s.step_capacity = j.steps + j.warmup;
      s.load_offset = nload;
      s.req_offset = nreq;
      nrec += s.step_capacity;
      nload += s.step_capacity * j.G;
      nreq += static_cast<int64_t>(st.size());
      scen[i] = s;
    }
    cs.assign(std::max<int64_t>(nrec, 1), 0.0);
    dt.assign(std::max<int64_t>(nrec, 1), 0.0);
    mx.assign(std::max<int64_t>(nrec, 1), 0.0);
    ac.assign(std::max<int64_t>(nrec, 1), 0);
    loads.assign(std::max<int64_t>(nload, 1), 0.0);
    arr_step.assign(nreq, -1);
    start.assign(nreq, -1);
    worker.assign(nreq, -1);
    ac_clock.assign(nreq, 0.0);
    fin_clock.assign(nreq, 0.0);
    bfsim_step_sink_t ss{cs.data(), dt.data(), mx.data(), ac.data(), loads.data()};
    bfsim_req_sink_t rs{arr_step.data(), start.data(), worker.data(), ac_clock.data(),
                        fin_clock.data()};
    int rc = bfsim_run_batch(ctx.get(), scen.data(), static_cast<int64_t>(n), inputs.data(),
                             static_cast<int32_t>(n), cbase.data(),
                             static_cast<int64_t>(cbase.size()), nullptr, 0, pool.data(),
                             static_cast<int64_t>(pool.size()), &ss, nrec, nload, &rs, nreq,
                             res.data(), err, sizeof err);
    if (rc == BFSIM_ESTREAM) {
      for (size_t i = 0; i < n; ++i)
        if (res[i].status == BFSIM_ESTREAM) len[i] *= 2;
      continue;
    }
    check(rc, err);
    break;
  }
  std::vector<std::vector<StepRecord>> out(n);
  if (timings) timings->assign(n, {});
  if (metrics) metrics->assign(n, {});
  for (size_t i = 0; i < n; ++i) {
    const auto& j = jobs[i];
    const int64_t total = j.steps + j.warmup;
    for (int64_t k = j.warmup; k < total; ++k) {
      StepRecord s;
      const int64_t o = scen[i].step_offset + k;
      s.k = k;
      s.clock_start = cs[o];
      s.dt = dt[o];
      s.max_load = mx[o];
      s.active_count = ac[o];
      s.loads.assign(loads.begin() + scen[i].load_offset + k * j.G,
                     loads.begin() + scen[i].load_offset + (k + 1) * j.G);
      out[i].push_back(std::move(s));
    }
    if (timings) {
      // ids in admission order (oracle.hpp:206); completion order (oracle.hpp:225-240)
      std::vector<std::tuple<int32_t, int64_t>> adm;
      const int64_t consumed = res[i].consumed;
      for (int64_t q = 0; q < consumed; ++q)
        if (start[scen[i].req_offset + q] >= 0) adm.emplace_back(start[scen[i].req_offset + q], q);
      std::sort(adm.begin(), adm.end());
      std::vector<std::tuple<int64_t, int32_t, int32_t, int64_t>> fin;
      for (size_t id = 0; id < adm.size(); ++id) {
        auto [x, q] = adm[id];
        int64_t f = x + streams[i][q].decode - 1;
        if (f < total) fin.emplace_back(f, worker[scen[i].req_offset + q], static_cast<int32_t>(id), q);
      }
      std::sort(fin.begin(), fin.end());
      for (const auto& [f, g, id, q] : fin) {
        RequestTiming t;
        t.id = id;
        t.admit_clock = ac_clock[scen[i].req_offset + q];
        t.finish_clock = fin_clock[scen[i].req_offset + q];
        t.decode_steps = streams[i][q].decode;
        t.completed = true;
        (*timings)[i].push_back(t);
      }
    }
    if (metrics) {
      MetricsReport& m = (*metrics)[i];
      m.avg_imbalance = res[i].avg_imbalance;
      m.throughput = res[i].throughput;
      m.tpot = res[i].tpot;
      m.energy = res[i].energy;
      m.imb_total = res[i].imb_total;
      m.total_workload = res[i].total_workload;
      m.eta_sum = res[i].eta_sum;
    }
  }
  return out;
}

// run_overloaded on the GPU (oracle.hpp:138-143).
inline std::vector<StepRecord> run_overloaded(Context& ctx, PolicyKind policy, int H, int G, int B,
                                              long steps, long warmup, const OverloadedSpec& spec,
                                              std::uint64_t seed, long /*search_limit*/ = 200000,
                                              std::vector<RequestTiming>* timings = nullptr) {
  std::vector<std::vector<RequestTiming>> tm;
  auto out = run_overloaded_batch(ctx, {{policy, H, G, B, steps, warmup, seed}}, spec, PowerModel{},
                                  timings ? &tm : nullptr);
  if (timings) *timings = std::move(tm.front());
  return std::move(out.front());
}

// estimate_iir (oracle.hpp:263-317): every (B, G, trial) x {FCFS, BF-IO H=0}
// trajectory in ONE batch on the GPU, reduced with the reference formulas.
inline IirEstimate estimate_iir(Context& ctx, const std::vector<int>& batch_sizes,
                                const std::vector<int>& worker_counts, const OverloadedSpec& spec,
                                int trials, long steps, long warmup, std::uint64_t seed) {
  if (trials < 1) throw std::invalid_argument("estimate_iir: trials must be >= 1");
  std::vector<OverloadedJob> jobs;
  for (int B : batch_sizes)
    for (int G : worker_counts)
      for (int t = 0; t < trials; ++t) {
        std::uint64_t ts = seed + 1000003ULL * static_cast<std::uint64_t>(t) +
                           17ULL * static_cast<std::uint64_t>(B) + static_cast<std::uint64_t>(G);
        jobs.push_back({PolicyKind::Fcfs, 0, G, B, steps, warmup, ts});
        jobs.push_back({PolicyKind::BfioGreedy, 0, G, B, steps, warmup, ts});
      }
  std::vector<MetricsReport> m;
  run_overloaded_batch(ctx, jobs, spec, PowerModel{}, nullptr, &m);
  const size_t cells = batch_sizes.size() * worker_counts.size();
  std::vector<double> f(cells * trials), b(cells * trials), red(cells * 4);
  for (size_t c = 0; c < cells; ++c)
    for (int t = 0; t < trials; ++t) {
      f[c * trials + t] = m[2 * (c * trials + t)].avg_imbalance;
      b[c * trials + t] = m[2 * (c * trials + t) + 1].avg_imbalance;
    }
  char err[512] = {0};
  check(bfsim_iir_reduce(f.data(), b.data(), trials, static_cast<int32_t>(cells), red.data(), err,
                         sizeof err),
        err);
  IirEstimate est;
  est.seed = seed;
  size_t c = 0;
  for (int B : batch_sizes)
    for (int G : worker_counts) {
      IirCell cell;
      cell.batch = B;
      cell.workers = G;
      cell.trials = trials;
      cell.outside_regime = std::sqrt(static_cast<double>(G)) > static_cast<double>(B);
      cell.fcfs_mean = red[4 * c];
      cell.bfio_mean = red[4 * c + 1];
      cell.ratio = red[4 * c + 2];
      cell.stderr_ = red[4 * c + 3];
      est.cells.push_back(cell);
      ++c;
    }
  return est;
}

// One policy call as the reference makes it: assign(policy, waiting,
// workers, H, search_limit), policies.hpp:372-382.
struct AssignCall {
  PolicyKind policy;
  const std::vector<RequestPreview>* waiting;
  const std::vector<WorkerView>* workers;
  int H;
};

// Many independent assign() calls in one launch (one warp each on the
// device). Returns the reference's Allocations; throws what assign() would
// (SearchLimitExceeded for bfio-exact beyond search_limit, invalid_argument
// for values the GPU path cannot take exactly).
inline std::vector<Allocation> assign_batch(Context& ctx, const std::vector<AssignCall>& calls,
                                            long search_limit = 200000,
                                            std::vector<double>* exact_costs = nullptr) {
  std::vector<bfsim_assign_call_t> c(calls.size());
  std::vector<double> pv, fu;
  std::vector<int32_t> caps, cnt;
  int64_t pairs = 0;
  for (size_t k = 0; k < calls.size(); ++k) {
    const auto& a = calls[k];
    const int G = static_cast<int>(a.workers->size());
    long capsum = 0;
    c[k] = bfsim_assign_call_t{static_cast<int32_t>(a.policy), static_cast<int32_t>(a.waiting->size()), G, a.H,
                               static_cast<int64_t>(pv.size()), static_cast<int64_t>(caps.size()),
                               static_cast<int64_t>(fu.size()), pairs};
    for (const auto& r : *a.waiting) pv.insert(pv.end(), r.w.begin(), r.w.begin() + a.H + 1);
    for (const auto& w : *a.workers) {
      caps.push_back(w.cap);
      cnt.push_back(w.active_count);
      fu.insert(fu.end(), w.future.begin(), w.future.begin() + a.H + 1);
      capsum += w.cap > 0 ? w.cap : 0;
    }
    pairs += 2 * std::min<long>(static_cast<long>(a.waiting->size()), capsum);
  }
  std::vector<int32_t> out(static_cast<size_t>(std::max<int64_t>(pairs, 1)));
  std::vector<int64_t> np(calls.size());
  std::vector<double> cost(calls.size());
  std::vector<int32_t> st(calls.size());
  char err[1024] = {0};
  int rc = bfsim_assign_batch(ctx.get(), c.data(), static_cast<int64_t>(c.size()), pv.data(),
                              static_cast<int64_t>(pv.size()), fu.data(), static_cast<int64_t>(fu.size()),
                              caps.data(), cnt.data(), static_cast<int64_t>(caps.size()), search_limit,
                              out.data(), pairs, np.data(), cost.data(), st.data(), err, sizeof err);
  if (rc == BFSIM_ELIMIT) throw SearchLimitExceeded(search_limit);
  check(rc, err);
  std::vector<Allocation> res(calls.size());
  for (size_t k = 0; k < calls.size(); ++k)
    for (int64_t j = 0; j < np[k]; ++j)
      res[k].assignments.emplace_back(out[c[k].pair_offset + 2 * j], out[c[k].pair_offset + 2 * j + 1]);
  if (exact_costs) *exact_costs = cost;
  return res;
}

}  // namespace gpu
}  // namespace bfsim
