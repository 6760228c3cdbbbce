// GPU path through the reference-shaped C++ adapter (include/bfsim_gpu.hpp)
// against the UNMODIFIED reference (bfsim::run / run_overloaded /
// estimate_iir) in the same binary. Restates the reference's own test
// expectations (proj/tests/engine_test.cpp, oracle_test.cpp, acceptance C04)
// plus randomized whole-trajectory equality. Prints one PASS/FAIL line per
// check; exit code = number of failures. Needs a B200 (run from pytest -m gpu).
#include <cstdio>
#include <random>
#include <sstream>
#include <string>

#include "bfsim/engine.hpp"
#include "bfsim/metrics.hpp"
#include "bfsim/oracle.hpp"
#include "bfsim_gpu.hpp"

using namespace bfsim;

static int failures = 0;
static void report(const std::string& name, bool ok) {
  std::printf("%-58s %s\n", name.c_str(), ok ? "PASS" : "FAIL");
  if (!ok) ++failures;
}

static bool same_steps(const std::vector<StepRecord>& a, const std::vector<StepRecord>& b) {
  if (a.size() != b.size()) return false;
  for (size_t k = 0; k < a.size(); ++k) {
    const auto &x = a[k], &y = b[k];
    if (x.k != y.k || x.clock_start != y.clock_start || x.dt != y.dt || x.max_load != y.max_load ||
        x.active_count != y.active_count || x.loads != y.loads)
      return false;
  }
  return true;
}

static bool same_result(const SimResult& g, const SimResult& r) {
  if (!same_steps(g.steps, r.steps) || g.completed_all != r.completed_all) return false;
  for (size_t k = 0; k < g.steps.size(); ++k)
    if (g.steps[k].admitted != r.steps[k].admitted || g.steps[k].completed != r.steps[k].completed)
      return false;
  if (g.requests.size() != r.requests.size()) return false;
  for (size_t i = 0; i < g.requests.size(); ++i) {
    const auto &a = g.requests[i], &b = r.requests[i];
    if (a.id != b.id || a.arrival_step != b.arrival_step || a.start_step != b.start_step ||
        a.admit_clock != b.admit_clock || a.finish_clock != b.finish_clock ||
        a.decode_steps != b.decode_steps || a.completed != b.completed)
      return false;
  }
  if (!r.steps.empty()) {
    MetricsReport mg = compute_metrics(g), mr = compute_metrics(r);
    if (mg.avg_imbalance != mr.avg_imbalance || mg.throughput != mr.throughput ||
        mg.tpot != mr.tpot || mg.energy != mr.energy || mg.eta_sum != mr.eta_sum)
      return false;
  }
  return true;
}

static ArrivalInstance make_instance(std::vector<ArrivalRecord> rows, DriftSpec drift = DriftSpec::unit()) {
  ArrivalInstance inst;
  inst.requests = std::move(rows);
  inst.drift = drift;
  inst.source_order.resize(inst.requests.size());
  for (size_t i = 0; i < inst.source_order.size(); ++i) inst.source_order[i] = i;
  return inst;
}

static SimConfig small(int G, int B, PolicyKind p = PolicyKind::Fcfs) {
  SimConfig c;
  c.workers = G;
  c.batch = B;
  c.policy = p;
  return c;
}

int main() {
  gpu::Context ctx(0);

  {  // engine_test.cpp:82-94 hand trace
    auto inst = make_instance({{0.0, 2, 3}});
    SimResult g = gpu::run(ctx, small(1, 1), inst);
    bool ok = g.steps.size() == 3 && g.steps[0].loads[0] == 2.0 && g.steps[1].loads[0] == 3.0 &&
              g.steps[2].loads[0] == 4.0 && g.total_workload_processed() == 9.0 && g.completed_all &&
              g.requests[0].start_step == 0 && g.requests[0].completed;
    report("engine_test SingleRequestHandTrace (loads 2,3,4)", ok);
  }
  {  // engine_test.cpp:111-118
    auto inst = make_instance({{0.0, 2, 100}});
    SimConfig c = small(1, 1);
    c.max_steps = 10;
    SimResult g = gpu::run(ctx, c, inst);
    report("engine_test MaxStepsGivesPartialResult", g.steps.size() == 10 && !g.completed_all);
  }
  {  // engine_test.cpp:75-80
    ArrivalInstance inst;
    SimResult g = gpu::run(ctx, small(2, 2), inst);
    report("engine_test EmptyInstance", g.steps.empty() && g.completed_all);
  }
  {  // engine_test.cpp:142-154
    auto inst = make_instance({{0.0, 3, 4}, {0.0, 2, 2}});
    SimResult g = gpu::run(ctx, small(2, 1), inst);
    bool ok = g.completed_all;
    for (const auto& r : g.requests) {
      long fs = -1;
      for (const auto& s : g.steps)
        for (int id : s.completed)
          if (id == r.id) fs = s.k;
      ok = ok && fs == r.start_step + r.decode_steps - 1;
    }
    report("engine_test ProgressCompletionStep", ok);
  }
  {  // engine_test.cpp:131-140 workload conservation
    auto inst = sample_instance(PrefillDistribution::uniform(16), DecodeDistribution::geometric(0.15),
                                60.0, 4.0, 13);
    double expected = inst.total_workload();
    bool ok = true;
    for (PolicyKind p : {PolicyKind::Fcfs, PolicyKind::Jsq, PolicyKind::BfioGreedy}) {
      SimResult g = gpu::run(ctx, small(4, 4, p), inst);
      ok = ok && g.completed_all && g.total_workload_processed() == expected;
    }
    report("engine_test WorkloadConservationAcrossPolicies", ok);
  }
  {  // randomized whole-trajectory equality, one GPU batch
    std::mt19937_64 rng(2601);
    std::vector<SimConfig> cfgs;
    std::vector<ArrivalInstance> insts;
    for (int t = 0; t < 40; ++t) {
      int G = 1 + static_cast<int>(rng() % 24), B = 1 + static_cast<int>(rng() % 12);
      SimConfig c = small(G, B, std::vector<PolicyKind>{PolicyKind::Fcfs, PolicyKind::Jsq,
                                                        PolicyKind::BfioGreedy}[rng() % 3]);
      c.horizon = std::vector<int>{0, 0, 1, 4, 20}[rng() % 5];
      c.lookahead = std::vector<LookaheadMode>{LookaheadMode::Perfect, LookaheadMode::TruncatedAtH,
                                               LookaheadMode::Noisy}[rng() % 3];
      c.noise_sigma = std::vector<double>{0.5, 2.0, 7.0}[rng() % 3];
      c.seed = rng();
      double drift = static_cast<double>(rng() % 3);
      auto inst = sample_instance(PrefillDistribution::uniform(2 + static_cast<int>(rng() % 100)),
                                  DecodeDistribution::geometric(0.03 + 0.3 * (rng() % 100) / 100.0),
                                  (5.0 + rng() % 20) * G * B / 8.0, 0.5 + (rng() % 20) / 10.0,
                                  rng(), DriftSpec::constant(drift));
      cfgs.push_back(c);
      insts.push_back(std::move(inst));
    }
    std::vector<const ArrivalInstance*> ptrs;
    for (auto& i : insts) ptrs.push_back(&i);
    auto gres = gpu::run_batch(ctx, cfgs, ptrs);
    bool ok = true;
    for (size_t i = 0; i < cfgs.size(); ++i) ok = ok && same_result(gres[i], run(cfgs[i], insts[i]));
    report("gpu::run_batch == bfsim::run (40 random trajectories, perfect/truncated/noisy)", ok);
  }
  {  // oracle_test.cpp:99-107
    OverloadedSpec spec;
    spec.prefill = PrefillDistribution::uniform(8);
    spec.decode = DecodeDistribution::geometric(0.2);
    auto steps = gpu::run_overloaded(ctx, PolicyKind::Fcfs, 0, 3, 4, 100, 20, spec, 99);
    bool ok = steps.size() == 100u;
    for (const auto& s : steps) ok = ok && s.active_count == 12;
    report("oracle_test RunOverloaded MaintainsFullBatches", ok);
  }
  {  // run_overloaded equality incl. timings
    bool ok = true;
    std::mt19937_64 rng(7);
    for (int t = 0; t < 12 && ok; ++t) {
      OverloadedSpec spec;
      spec.prefill = PrefillDistribution::uniform(2 + static_cast<int>(rng() % 63));
      spec.decode = DecodeDistribution::geometric(0.05 + 0.3 * (rng() % 100) / 100.0);
      spec.drift = DriftSpec::constant(static_cast<double>(rng() % 2));
      PolicyKind p = std::vector<PolicyKind>{PolicyKind::Fcfs, PolicyKind::Jsq, PolicyKind::BfioGreedy}[rng() % 3];
      int H = std::vector<int>{0, 2, 20}[rng() % 3];
      int G = 1 + static_cast<int>(rng() % 9), B = 1 + static_cast<int>(rng() % 9);
      long steps = 20 + static_cast<long>(rng() % 150), warm = static_cast<long>(rng() % 40);
      uint64_t seed = rng();
      std::vector<RequestTiming> tg, tr;
      auto sg = gpu::run_overloaded(ctx, p, H, G, B, steps, warm, spec, seed, 200000, &tg);
      auto sr = run_overloaded(p, H, G, B, steps, warm, spec, seed, 200000, &tr);
      ok = same_steps(sg, sr) && tg.size() == tr.size();
      for (size_t i = 0; ok && i < tg.size(); ++i)
        ok = tg[i].id == tr[i].id && tg[i].admit_clock == tr[i].admit_clock &&
             tg[i].finish_clock == tr[i].finish_clock && tg[i].decode_steps == tr[i].decode_steps;
      if (ok && !sr.empty()) {
        MetricsReport mg = compute_metrics(sg, tg, PowerModel{}), mr = compute_metrics(sr, tr, PowerModel{});
        ok = mg.avg_imbalance == mr.avg_imbalance && mg.tpot == mr.tpot && mg.energy == mr.energy;
      }
    }
    report("gpu::run_overloaded == run_overloaded (12 random, timings)", ok);
  }
  {  // oracle_test.cpp:117-127 + equality of estimate_iir
    OverloadedSpec spec;
    spec.prefill = PrefillDistribution::uniform(8);
    spec.decode = DecodeDistribution::geometric(0.2);
    IirEstimate one = gpu::estimate_iir(ctx, {4}, {1}, spec, 3, 50, 10, 5);
    report("oracle_test EstimateIir SingleWorkerRatioIsOne",
           one.cells.size() == 1 && one.cells[0].fcfs_mean == 0.0 && one.cells[0].bfio_mean == 0.0 &&
               std::isinf(one.cells[0].ratio));
    IirEstimate g = gpu::estimate_iir(ctx, {2, 4}, {2, 3}, spec, 4, 60, 15, 11);
    IirEstimate r = estimate_iir({2, 4}, {2, 3}, spec, 4, 60, 15, 11);
    bool ok = g.cells.size() == r.cells.size();
    for (size_t c = 0; ok && c < g.cells.size(); ++c)
      ok = g.cells[c].fcfs_mean == r.cells[c].fcfs_mean && g.cells[c].bfio_mean == r.cells[c].bfio_mean &&
           g.cells[c].ratio == r.cells[c].ratio && g.cells[c].stderr_ == r.cells[c].stderr_ &&
           g.cells[c].outside_regime == r.cells[c].outside_regime;
    report("gpu::estimate_iir == estimate_iir (2x2 grid, 4 trials)", ok);
  }
  {  // the reference's own writers over GPU results are
     // byte-identical (steps.csv engine.hpp:270-281, summary metrics.hpp:129-136,
     // iir.csv oracle.hpp:321-330) -- the adapter returns the reference's types
    auto inst = sample_instance(PrefillDistribution::uniform(64), DecodeDistribution::geometric(0.02), 2000.0,
                                1.0, 1, DriftSpec::unit());
    bool ok = true;
    for (PolicyKind p : {PolicyKind::Fcfs, PolicyKind::BfioGreedy}) {
      SimConfig c = small(8, 64, p);
      c.horizon = p == PolicyKind::BfioGreedy ? 20 : 0;
      c.lookahead = LookaheadMode::Noisy;
      c.noise_sigma = 2.0;
      c.seed = 5;
      SimResult g = gpu::run(ctx, c, inst), r = run(c, inst);
      std::ostringstream a, b;
      write_step_csv(a, g);
      write_summary(a, compute_metrics(g));
      write_step_csv(b, r);
      write_summary(b, compute_metrics(r));
      ok = ok && a.str() == b.str();
    }
    OverloadedSpec spec;
    spec.prefill = PrefillDistribution::uniform(16);
    spec.decode = DecodeDistribution::geometric(0.1);
    std::ostringstream a, b;
    write_iir_csv(a, gpu::estimate_iir(ctx, {2, 8}, {2, 16}, spec, 3, 80, 20, 9));
    write_iir_csv(b, estimate_iir({2, 8}, {2, 16}, spec, 3, 80, 20, 9));
    ok = ok && a.str() == b.str();
    report("write_step_csv / write_summary / write_iir_csv byte-identical (C1, noisy H=20)", ok);
  }
  {  // the policy operator: gpu::assign_batch == assign() on random steps,
     // every policy (policies_test.cpp random_step shapes, :27-55)
    std::mt19937_64 rng(4242);
    std::vector<std::vector<RequestPreview>> ws;
    std::vector<std::vector<WorkerView>> vs;
    std::vector<gpu::AssignCall> calls;
    std::vector<int> hs;
    for (int t = 0; t < 2000; ++t) {
      int H = static_cast<int>(rng() % 3), G = 1 + static_cast<int>(rng() % 3), n = static_cast<int>(rng() % 7);
      std::vector<WorkerView> v(static_cast<size_t>(G));
      for (auto& w : v) {
        w.cap = static_cast<int>(rng() % 4);
        w.active_count = static_cast<int>(rng() % 3);
        for (int h = 0; h <= H; ++h) w.future.push_back(static_cast<double>(rng() % 20));
      }
      std::vector<RequestPreview> q(static_cast<size_t>(n));
      for (auto& r : q)
        for (int h = 0; h <= H; ++h) r.w.push_back(static_cast<double>(rng() % 10));
      ws.push_back(std::move(q));
      vs.push_back(std::move(v));
      hs.push_back(H);
    }
    for (size_t t = 0; t < ws.size(); ++t)
      calls.push_back({std::vector<PolicyKind>{PolicyKind::Fcfs, PolicyKind::Jsq, PolicyKind::BfioExact,
                                               PolicyKind::BfioGreedy}[t % 4],
                       &ws[t], &vs[t], hs[t]});
    auto got = gpu::assign_batch(ctx, calls);
    bool ok = got.size() == calls.size();
    for (size_t t = 0; ok && t < calls.size(); ++t)
      ok = got[t].assignments == assign(calls[t].policy, ws[t], vs[t], hs[t], 200000).assignments;
    bool threw = false;
    std::vector<WorkerView> v4(4);
    for (auto& w : v4) {
      w.cap = 4;
      w.future = {0.0};
    }
    std::vector<RequestPreview> q12(12);
    for (auto& r : q12) r.w = {1.0};
    try {
      gpu::assign_batch(ctx, {{PolicyKind::BfioExact, &q12, &v4, 0}}, 100);
    } catch (const SearchLimitExceeded&) {
      threw = true;
    }
    report("gpu::assign_batch == assign (2000 random steps, 4 policies) + SearchLimitExceeded", ok && threw);
  }
  {  // acceptance_test.cpp:178-180 (C04) through the GPU path
    OverloadedSpec spec;
    spec.prefill = PrefillDistribution::uniform(64);
    spec.decode = DecodeDistribution::geometric(0.02);
    spec.drift = DriftSpec::constant(0.0);
    std::vector<gpu::OverloadedJob> jobs;
    for (uint64_t seed = 1; seed <= 10; ++seed)
      for (PolicyKind p : {PolicyKind::Fcfs, PolicyKind::Jsq, PolicyKind::BfioGreedy})
        jobs.push_back({p, 0, 8, 16, 5000, 500, seed});
    std::vector<MetricsReport> m;
    gpu::run_overloaded_batch(ctx, jobs, spec, PowerModel{}, nullptr, &m);
    double f = 0, j = 0, b = 0;
    for (size_t i = 0; i < jobs.size(); i += 3) {
      f += m[i].avg_imbalance;
      j += m[i + 1].avg_imbalance;
      b += m[i + 2].avg_imbalance;
    }
    report("acceptance C04: BF-IO <= 0.5 FCFS, JSQ <= FCFS (GPU)", b <= 0.5 * f && j <= f);
  }
  std::printf("failures=%d\n", failures);
  return failures;
}
