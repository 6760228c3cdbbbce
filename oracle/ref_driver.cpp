// ORACLE / TEST INFRASTRUCTURE — not product code.
//
// Thin C-ABI driver around the UNMODIFIED reference headers
// (/root/reference/proj/include/bfsim/*.hpp). It is compiled by oracle/Makefile
// with `g++ -std=c++20 -O2 -ffp-contract=off` (F6 no FMA in dt,
// F7 GCC argument evaluation order for the noisy RNG) into oracle/_ref/libbfsim_ref.so.
// Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg load it.
//
// Every entry point calls the reference exactly the way the reference CLI
// does (tools/bfsim.cpp:118-156): sample_instance / run / run_overloaded /
// compute_metrics / estimate_iir / assign. Results are handed back through an
// opaque handle plus copy-out accessors so ctypes callers own their buffers.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <memory>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "bfsim/engine.hpp"
#include "bfsim/metrics.hpp"
#include "bfsim/oracle.hpp"
#include "bfsim/policies.hpp"
#include "bfsim/workload.hpp"
#include "bfsim_gpu.h"

namespace {

void set_err(char* err, size_t errlen, const char* msg) {
  if (err && errlen) {
    std::strncpy(err, msg, errlen - 1);
    err[errlen - 1] = 0;
  }
}

// Exception class -> bfsim_gpu.h return code.
int code_of(const std::exception_ptr& ep, char* err, size_t errlen) {
  try {
    std::rethrow_exception(ep);
  } catch (const std::invalid_argument& e) {
    set_err(err, errlen, e.what());
    return BFSIM_EINVAL;
  } catch (const std::logic_error& e) {
    set_err(err, errlen, e.what());
    return BFSIM_ELOGIC;
  } catch (const std::exception& e) {
    set_err(err, errlen, e.what());
    return 9;
  }
}

// kind 2: the reference's Empirical distributions over the lists set by
// ref_set_empirical (test infrastructure: one list pair per process)
std::vector<int> g_emp_prefill;
std::vector<long> g_emp_decode;

bfsim::PrefillDistribution make_prefill(int kind, int s_max) {
  if (kind == 2) return bfsim::PrefillDistribution::empirical(g_emp_prefill);
  return kind == 1 ? bfsim::PrefillDistribution::fixed_value(s_max)
                   : bfsim::PrefillDistribution::uniform(s_max);
}
bfsim::DecodeDistribution make_decode(int kind, double p, long fixed_o) {
  if (kind == 2) return bfsim::DecodeDistribution::empirical(g_emp_decode);
  return kind == 1 ? bfsim::DecodeDistribution::fixed_length(fixed_o)
                   : bfsim::DecodeDistribution::geometric(p);
}

bfsim::SimConfig make_config(const bfsim_scenario_t& s) {
  bfsim::SimConfig c;
  c.workers = s.workers;
  c.batch = s.batch;
  c.overhead = s.overhead;
  c.per_token = s.per_token;
  c.horizon = s.horizon;
  c.policy = static_cast<bfsim::PolicyKind>(s.policy);
  c.max_steps = s.max_steps;
  c.seed = s.seed;
  c.power.p_idle = s.p_idle;
  c.power.p_max = s.p_max;
  c.power.mfu_sat = s.mfu_sat;
  c.power.gamma = s.gamma;
  c.lookahead = static_cast<bfsim::LookaheadMode>(s.lookahead);
  c.noise_sigma = s.noise_sigma;
  return c;
}

bfsim::ArrivalInstance make_instance(const bfsim_request_t* rec, int64_t n, double drift) {
  bfsim::ArrivalInstance inst;
  inst.requests.resize(static_cast<size_t>(n));
  for (int64_t i = 0; i < n; ++i) {
    inst.requests[i].arrival_time = rec[i].arrival_time;
    inst.requests[i].prefill = rec[i].prefill;
    inst.requests[i].decode = rec[i].decode;
  }
  inst.drift = bfsim::DriftSpec::constant(drift);
  inst.source_order.resize(inst.requests.size());
  for (size_t i = 0; i < inst.source_order.size(); ++i) inst.source_order[i] = i;
  return inst;
}

struct Handle {
  std::vector<bfsim::StepRecord> steps;
  std::vector<bfsim::RequestTiming> requests;
  bool completed_all = true;
  bool has_metrics = false;
  bfsim::MetricsReport metrics;
  int G = 0;
};

}  // namespace

extern "C" {

void ref_set_empirical(const int64_t* prefill, int64_t n_prefill, const int64_t* decode, int64_t n_decode) {
  g_emp_prefill.assign(prefill, prefill + n_prefill);
  g_emp_decode.assign(decode, decode + n_decode);
}

int ref_sample_instance(int prefill_kind, int s_max, int decode_kind, double p, int64_t fixed_o,
                        double rate, double duration, uint64_t seed, bfsim_request_t* out,
                        int64_t capacity, int64_t* n_out, char* err, size_t errlen) {
  try {
    auto inst = bfsim::sample_instance(make_prefill(prefill_kind, s_max),
                                       make_decode(decode_kind, p, fixed_o), rate, duration, seed);
    *n_out = static_cast<int64_t>(inst.requests.size());
    if (out) {
      int64_t m = std::min<int64_t>(capacity, *n_out);
      for (int64_t i = 0; i < m; ++i) {
        out[i].arrival_time = inst.requests[i].arrival_time;
        out[i].prefill = inst.requests[i].prefill;
        out[i].decode = static_cast<int32_t>(inst.requests[i].decode);
      }
    }
    return 0;
  } catch (...) {
    return code_of(std::current_exception(), err, errlen);
  }
}

// bfsim::run + compute_metrics, as tools/bfsim.cpp:124-141.
void* ref_run_poisson(const bfsim_scenario_t* sc, const bfsim_request_t* trace, int64_t n,
                      int* code, char* err, size_t errlen) {
  try {
    auto h = std::make_unique<Handle>();
    auto inst = make_instance(trace, n, sc->drift);
    bfsim::SimResult res = bfsim::run(make_config(*sc), inst);
    h->G = sc->workers;
    h->completed_all = res.completed_all;
    if (!res.steps.empty()) {
      h->metrics = bfsim::compute_metrics(res);
      h->has_metrics = true;
    }
    h->steps = std::move(res.steps);
    h->requests = std::move(res.requests);
    *code = 0;
    return h.release();
  } catch (...) {
    *code = code_of(std::current_exception(), err, errlen);
    return nullptr;
  }
}

// bfsim::run_overloaded with timings + compute_metrics, as tools/bfsim.cpp:142-151.
void* ref_run_overloaded(const bfsim_scenario_t* sc, int prefill_kind, int s_max, int decode_kind,
                         double p, int64_t fixed_o, int* code, char* err, size_t errlen) {
  try {
    auto h = std::make_unique<Handle>();
    bfsim::OverloadedSpec spec;
    spec.prefill = make_prefill(prefill_kind, s_max);
    spec.decode = make_decode(decode_kind, p, fixed_o);
    spec.drift = bfsim::DriftSpec::constant(sc->drift);
    spec.overhead = sc->overhead;
    spec.per_token = sc->per_token;
    spec.backlog = sc->backlog;
    bfsim::PowerModel power;
    power.p_idle = sc->p_idle;
    power.p_max = sc->p_max;
    power.mfu_sat = sc->mfu_sat;
    power.gamma = sc->gamma;
    h->G = sc->workers;
    h->steps = bfsim::run_overloaded(static_cast<bfsim::PolicyKind>(sc->policy), sc->horizon,
                                     sc->workers, sc->batch, sc->steps, sc->warmup, spec, sc->seed,
                                     200000, &h->requests);
    if (!h->steps.empty()) {
      h->metrics = bfsim::compute_metrics(h->steps, h->requests, power);
      h->has_metrics = true;
    }
    *code = 0;
    return h.release();
  } catch (...) {
    *code = code_of(std::current_exception(), err, errlen);
    return nullptr;
  }
}

int64_t ref_res_steps(void* hp) { return static_cast<int64_t>(static_cast<Handle*>(hp)->steps.size()); }
int ref_res_completed_all(void* hp) { return static_cast<Handle*>(hp)->completed_all ? 1 : 0; }
int ref_res_has_metrics(void* hp) { return static_cast<Handle*>(hp)->has_metrics ? 1 : 0; }
int64_t ref_res_n_requests(void* hp) {
  return static_cast<int64_t>(static_cast<Handle*>(hp)->requests.size());
}

void ref_res_step_arrays(void* hp, int64_t* k, double* clock_start, double* dt, double* max_load,
                         int64_t* active_count, double* loads) {
  auto* h = static_cast<Handle*>(hp);
  for (size_t i = 0; i < h->steps.size(); ++i) {
    const auto& s = h->steps[i];
    k[i] = s.k;
    clock_start[i] = s.clock_start;
    dt[i] = s.dt;
    max_load[i] = s.max_load;
    active_count[i] = s.active_count;
    for (int g = 0; g < h->G; ++g) loads[i * h->G + g] = s.loads[g];
  }
}

// Flattened per-step id lists: which = 0 admitted, 1 completed. offsets has K+1 entries.
int64_t ref_res_list_total(void* hp, int which) {
  auto* h = static_cast<Handle*>(hp);
  int64_t t = 0;
  for (const auto& s : h->steps) t += static_cast<int64_t>(which ? s.completed.size() : s.admitted.size());
  return t;
}
void ref_res_list(void* hp, int which, int64_t* offsets, int32_t* ids) {
  auto* h = static_cast<Handle*>(hp);
  int64_t t = 0;
  for (size_t i = 0; i < h->steps.size(); ++i) {
    offsets[i] = t;
    const auto& v = which ? h->steps[i].completed : h->steps[i].admitted;
    for (int id : v) ids[t++] = id;
  }
  offsets[h->steps.size()] = t;
}

void ref_res_requests(void* hp, int32_t* id, int64_t* arrival_step, int64_t* start_step,
                      double* admit_clock, double* finish_clock, int64_t* decode_steps,
                      uint8_t* completed) {
  auto* h = static_cast<Handle*>(hp);
  for (size_t i = 0; i < h->requests.size(); ++i) {
    const auto& r = h->requests[i];
    id[i] = r.id;
    arrival_step[i] = r.arrival_step;
    start_step[i] = r.start_step;
    admit_clock[i] = r.admit_clock;
    finish_clock[i] = r.finish_clock;
    decode_steps[i] = r.decode_steps;
    completed[i] = r.completed ? 1 : 0;
  }
}

// MetricsReport field order (metrics.hpp:96-104).
void ref_res_metrics(void* hp, double* out7) {
  const auto& m = static_cast<Handle*>(hp)->metrics;
  out7[0] = m.avg_imbalance;
  out7[1] = m.throughput;
  out7[2] = m.tpot;
  out7[3] = m.energy;
  out7[4] = m.imb_total;
  out7[5] = m.total_workload;
  out7[6] = m.eta_sum;
}

void ref_res_free(void* hp) { delete static_cast<Handle*>(hp); }

// Per-step policy operator assign(), policies.hpp:372-382. Pairs (waiting idx,
// worker) in the reference's output order. cost (may be NULL) = horizon cost of
// the resulting allocation (predict_loads + horizon_cost, policies.hpp:143-172).
int ref_assign(int policy, int n_waiting, const double* previews, int G, const int32_t* caps,
               const int32_t* active_counts, const double* futures, int H, int64_t limit,
               int32_t* pairs, int64_t* n_pairs, double* cost, char* err, size_t errlen) {
  try {
    std::vector<bfsim::RequestPreview> waiting(static_cast<size_t>(n_waiting));
    for (int i = 0; i < n_waiting; ++i)
      waiting[i].w.assign(previews + static_cast<size_t>(i) * (H + 1),
                          previews + static_cast<size_t>(i + 1) * (H + 1));
    std::vector<bfsim::WorkerView> workers(static_cast<size_t>(G));
    for (int g = 0; g < G; ++g) {
      workers[g].cap = caps[g];
      workers[g].active_count = active_counts[g];
      workers[g].future.assign(futures + static_cast<size_t>(g) * (H + 1),
                               futures + static_cast<size_t>(g + 1) * (H + 1));
    }
    bfsim::Allocation a =
        bfsim::assign(static_cast<bfsim::PolicyKind>(policy), waiting, workers, H, limit);
    *n_pairs = static_cast<int64_t>(a.assignments.size());
    for (size_t j = 0; j < a.assignments.size(); ++j) {
      pairs[2 * j] = a.assignments[j].first;
      pairs[2 * j + 1] = a.assignments[j].second;
    }
    if (cost) *cost = bfsim::horizon_cost(bfsim::predict_loads(workers, waiting, a, H));
    return 0;
  } catch (...) {
    return code_of(std::current_exception(), err, errlen);
  }
}

// estimate_iir, oracle.hpp:263-317. out: 8 doubles per cell
// {B, G, fcfs_mean, bfio_mean, ratio, stderr, trials, outside_regime}.
int ref_estimate_iir(const int32_t* b_list, int nb, const int32_t* g_list, int ng, int prefill_kind,
                     int s_max, int decode_kind, double p, int64_t fixed_o, double drift,
                     double overhead, double per_token, double backlog, int trials, int64_t steps,
                     int64_t warmup, uint64_t seed, double* out, char* err, size_t errlen) {
  try {
    bfsim::OverloadedSpec spec;
    spec.prefill = make_prefill(prefill_kind, s_max);
    spec.decode = make_decode(decode_kind, p, fixed_o);
    spec.drift = bfsim::DriftSpec::constant(drift);
    spec.overhead = overhead;
    spec.per_token = per_token;
    spec.backlog = backlog;
    auto est = bfsim::estimate_iir(std::vector<int>(b_list, b_list + nb),
                                   std::vector<int>(g_list, g_list + ng), spec, trials, steps,
                                   warmup, seed);
    for (size_t c = 0; c < est.cells.size(); ++c) {
      const auto& cell = est.cells[c];
      double* o = out + 8 * c;
      o[0] = cell.batch;
      o[1] = cell.workers;
      o[2] = cell.fcfs_mean;
      o[3] = cell.bfio_mean;
      o[4] = cell.ratio;
      o[5] = cell.stderr_;
      o[6] = cell.trials;
      o[7] = cell.outside_regime ? 1.0 : 0.0;
    }
    return 0;
  } catch (...) {
    return code_of(std::current_exception(), err, errlen);
  }
}

// CPU baseline: run the reference (run + compute_metrics, tools/bfsim.cpp:124-141)
// over n_scen Poisson scenarios on `threads` host threads, one scenario per
// task. Trace construction (ArrivalInstance) is done before the clock starts.
// Returns wall seconds; worker_steps receives sum over scenarios of G*K.
double ref_bench_poisson(const bfsim_scenario_t* scen, int64_t n_scen, const bfsim_input_t* inputs,
                         const bfsim_request_t* traces, int threads, int64_t* worker_steps) {
  std::vector<bfsim::ArrivalInstance> inst(static_cast<size_t>(n_scen));
  for (int64_t i = 0; i < n_scen; ++i) {
    const bfsim_input_t& in = inputs[scen[i].input_id];
    inst[i] = make_instance(traces + in.offset, in.length, scen[i].drift);
  }
  std::atomic<int64_t> next{0}, ws{0};
  auto body = [&]() {
    for (;;) {
      int64_t i = next.fetch_add(1);
      if (i >= n_scen) break;
      bfsim::SimResult res = bfsim::run(make_config(scen[i]), inst[i]);
      volatile double sink = 0.0;
      if (!res.steps.empty()) sink = bfsim::compute_metrics(res).avg_imbalance;
      (void)sink;
      ws.fetch_add(static_cast<int64_t>(res.steps.size()) * scen[i].workers);
    }
  };
  auto t0 = std::chrono::steady_clock::now();
  std::vector<std::thread> pool;
  for (int t = 0; t < threads; ++t) pool.emplace_back(body);
  for (auto& t : pool) t.join();
  auto t1 = std::chrono::steady_clock::now();
  *worker_steps = ws.load();
  return std::chrono::duration<double>(t1 - t0).count();
}


// CPU baseline for run_overloaded (oracle.hpp:138-244) + compute_metrics:
// each scenario runs the reference loop, drawing its own samples from
// mt19937_64(seed); one scenario per task on `threads` host threads.
// Returns wall seconds; worker_steps receives sum of G * (warmup + steps).
double ref_bench_overloaded(const bfsim_scenario_t* scen, int64_t n_scen, int prefill_kind, int s_max,
                            int decode_kind, double p, int64_t fixed_o, int threads,
                            int64_t* worker_steps) {
  std::atomic<int64_t> next{0}, ws{0};
  auto body = [&]() {
    for (;;) {
      int64_t i = next.fetch_add(1);
      if (i >= n_scen) break;
      const bfsim_scenario_t& sc = scen[i];
      bfsim::OverloadedSpec spec;
      spec.prefill = make_prefill(prefill_kind, s_max);
      spec.decode = make_decode(decode_kind, p, fixed_o);
      spec.drift = bfsim::DriftSpec::constant(sc.drift);
      spec.overhead = sc.overhead;
      spec.per_token = sc.per_token;
      spec.backlog = sc.backlog;
      bfsim::PowerModel power;
      power.p_idle = sc.p_idle;
      power.p_max = sc.p_max;
      power.mfu_sat = sc.mfu_sat;
      power.gamma = sc.gamma;
      std::vector<bfsim::RequestTiming> timings;
      auto steps = bfsim::run_overloaded(static_cast<bfsim::PolicyKind>(sc.policy), sc.horizon,
                                         sc.workers, sc.batch, sc.steps, sc.warmup, spec, sc.seed,
                                         200000, &timings);
      volatile double sink = 0.0;
      if (!steps.empty()) sink = bfsim::compute_metrics(steps, timings, power).avg_imbalance;
      (void)sink;
      ws.fetch_add(static_cast<int64_t>(sc.steps + sc.warmup) * sc.workers);
    }
  };
  auto t0 = std::chrono::steady_clock::now();
  std::vector<std::thread> pool;
  for (int t = 0; t < threads; ++t) pool.emplace_back(body);
  for (auto& t : pool) t.join();
  auto t1 = std::chrono::steady_clock::now();
  *worker_steps = ws.load();
  return std::chrono::duration<double>(t1 - t0).count();
}

}  // extern "C"
