// bfsim_gpu: the reference CLI's experiment subcommands (proj/tools/bfsim.cpp:
// run, compare, sweep-h, sweep-g, iir, validate-trace) on the B200 step engine.
//
// Same flags, config-file keys, output files and exit codes as the reference
// CLI (tools/bfsim.cpp:28-377; 0 success, 1 usage/config error, 2 partial
// completion). What changes is the execution: every simulation a subcommand
// needs goes to the GPU in ONE batch through the reference-shaped adapter
// (include/bfsim_gpu.hpp -> the C ABI): compare = one trajectory per policy,
// sweep-h = one per H, sweep-g = two per G, iir = the whole (B, G, trial)
// grid. The per-step records and request timings come back bit-exact, and
// the metrics are the reference's own compute_metrics over them
// (metrics.hpp:106-126), so summary.txt / compare.csv / sweep_*.csv /
// steps.csv are byte-identical to the CPU reference's.
//
// Built with -DBFSIM_CLI_CPU the same program runs the unmodified reference
// functions instead (bfsim::run / run_overloaded / estimate_iir): the CPU
// side of the CLI parity test (tests/test_gpu_cli.py). The CLI11 option
// parser of the reference is not vendored here; flags are parsed directly.
#include <cstdio>
#include <cstdlib>
#include <filesystem>
#include <fstream>
#include <functional>
#include <iostream>
#include <map>
#include <sstream>
#include <string>
#include <vector>

#include "bfsim/engine.hpp"
#include "bfsim/metrics.hpp"
#include "bfsim/oracle.hpp"
#include "bfsim/policies.hpp"
#include "bfsim/workload.hpp"
#ifndef BFSIM_CLI_CPU
#include "bfsim_gpu.hpp"
#endif

namespace fs = std::filesystem;
using namespace bfsim;

namespace {

struct ExperimentConfig {  // tools/bfsim.cpp:28-43
  SimConfig sim;
  std::string policy_name = "fcfs";
  std::string trace;
  std::string mode = "poisson";
  double rate = 50.0;
  double duration = 10.0;
  long steps = 2000;
  long warmup = 200;
  int prefill_max = 64;
  double geo_p = 0.02;
  double drift = 1.0;
  std::string out = ".";
  bool emit_steps = false;
};

#ifndef BFSIM_CLI_CPU
gpu::Context& device() {  // one context (device 0) for the process
  static gpu::Context ctx(0);
  return ctx;
}
#endif

struct RunOutput {
  MetricsReport metrics;
  bool completed_all = true;
  std::vector<StepRecord> steps;
};

struct Job {  // one simulation of a subcommand
  ExperimentConfig cfg;
  PolicyKind policy;
  int horizon;
};

ArrivalInstance instance_of(const ExperimentConfig& cfg) {  // tools/bfsim.cpp:124-133
  ArrivalInstance inst;
  if (!cfg.trace.empty()) {
    inst = load_trace(cfg.trace);
    inst.drift = DriftSpec::constant(cfg.drift);
  } else {
    inst = sample_instance(PrefillDistribution::uniform(cfg.prefill_max), DecodeDistribution::geometric(cfg.geo_p),
                           cfg.rate, cfg.duration, cfg.sim.seed, DriftSpec::constant(cfg.drift));
  }
  return inst;
}

OverloadedSpec spec_of(const ExperimentConfig& cfg) {  // tools/bfsim.cpp:143-148
  OverloadedSpec spec;
  spec.prefill = PrefillDistribution::uniform(cfg.prefill_max);
  spec.decode = DecodeDistribution::geometric(cfg.geo_p);
  spec.drift = DriftSpec::constant(cfg.drift);
  spec.overhead = cfg.sim.overhead;
  spec.per_token = cfg.sim.per_token;
  return spec;
}

// run_one (tools/bfsim.cpp:118-156) for a whole list of jobs at once.
std::vector<RunOutput> run_jobs(const std::vector<Job>& jobs) {
  std::vector<RunOutput> out(jobs.size());
  std::vector<size_t> pois, ovl;
  for (size_t i = 0; i < jobs.size(); ++i) {
    const auto& c = jobs[i].cfg;
    if (!c.trace.empty() || c.mode == "poisson") pois.push_back(i);
    else if (c.mode == "overloaded") ovl.push_back(i);
    else throw std::runtime_error("config: mode must be 'poisson' or 'overloaded'");
  }
  // Poisson / trace jobs: instances are shared by identical workloads
  std::vector<ArrivalInstance> insts;
  std::vector<SimConfig> cfgs;
  std::vector<const ArrivalInstance*> ptrs;
  insts.reserve(pois.size());
  for (size_t i : pois) {
    SimConfig sim = jobs[i].cfg.sim;
    sim.policy = jobs[i].policy;
    sim.horizon = jobs[i].horizon;
    cfgs.push_back(sim);
    insts.push_back(instance_of(jobs[i].cfg));
  }
  for (auto& in : insts) ptrs.push_back(&in);
#ifdef BFSIM_CLI_CPU
  std::vector<SimResult> res;
  for (size_t j = 0; j < cfgs.size(); ++j) res.push_back(run(cfgs[j], *ptrs[j]));
#else
  // bfio-exact (an exponential search per step) stays on the CPU reference
  // (SURVEY §8(b)); everything else is one GPU batch
  gpu::Context& ctx = device();
  std::vector<SimConfig> gcfgs;
  std::vector<const ArrivalInstance*> gptrs;
  for (size_t j = 0; j < cfgs.size(); ++j)
    if (cfgs[j].policy != PolicyKind::BfioExact) {
      gcfgs.push_back(cfgs[j]);
      gptrs.push_back(ptrs[j]);
    }
  std::vector<SimResult> gres = gcfgs.empty() ? std::vector<SimResult>{} : gpu::run_batch(ctx, gcfgs, gptrs);
  std::vector<SimResult> res;
  for (size_t j = 0, q = 0; j < cfgs.size(); ++j)
    res.push_back(cfgs[j].policy == PolicyKind::BfioExact ? run(cfgs[j], *ptrs[j]) : std::move(gres[q++]));
#endif
  for (size_t j = 0; j < pois.size(); ++j) {
    RunOutput& o = out[pois[j]];
    o.completed_all = res[j].completed_all;
    o.metrics = res[j].steps.empty() ? MetricsReport{} : compute_metrics(res[j]);
    o.steps = std::move(res[j].steps);
  }
  // overloaded jobs: the workload flags (hence the OverloadedSpec) and the
  // power model are shared by every job of a subcommand
  if (ovl.empty()) return out;
  const ExperimentConfig& c0 = jobs[ovl.front()].cfg;
#ifdef BFSIM_CLI_CPU
  for (size_t i : ovl) {
    const auto& c = jobs[i].cfg;
    std::vector<RequestTiming> timings;
    out[i].steps = run_overloaded(jobs[i].policy, jobs[i].horizon, c.sim.workers, c.sim.batch, c.steps, c.warmup,
                                  spec_of(c), c.sim.seed, c.sim.search_limit, &timings);
    out[i].metrics = compute_metrics(out[i].steps, timings, c.sim.power);
  }
#else
  std::vector<gpu::OverloadedJob> oj;
  for (size_t i : ovl) {
    const auto& c = jobs[i].cfg;
    oj.push_back({jobs[i].policy, jobs[i].horizon, c.sim.workers, c.sim.batch, c.steps, c.warmup, c.sim.seed});
  }
  std::vector<std::vector<RequestTiming>> timings;
  auto steps = gpu::run_overloaded_batch(ctx, oj, spec_of(c0), c0.sim.power, &timings);
  for (size_t j = 0; j < ovl.size(); ++j) {
    out[ovl[j]].steps = std::move(steps[j]);
    out[ovl[j]].metrics = compute_metrics(out[ovl[j]].steps, timings[j], c0.sim.power);
  }
#endif
  return out;
}

void write_config_echo(std::ostream& os, const ExperimentConfig& cfg) {  // tools/bfsim.cpp:158-165
  os << "policy=" << cfg.policy_name << "\n"
     << "seed=" << cfg.sim.seed << "\n"
     << "workers=" << cfg.sim.workers << "\n"
     << "batch=" << cfg.sim.batch << "\n"
     << "horizon=" << cfg.sim.horizon << "\n"
     << "mode=" << (cfg.trace.empty() ? cfg.mode : "trace") << "\n";
}

int cmd_run(const ExperimentConfig& cfg) {
  RunOutput out = std::move(run_jobs({{cfg, policy_from_name(cfg.policy_name), cfg.sim.horizon}}).front());
  fs::create_directories(cfg.out);
  {
    std::ofstream os(fs::path(cfg.out) / "summary.txt");
    write_config_echo(os, cfg);
    write_summary(os, out.metrics);
  }
  if (cfg.emit_steps) {
    std::ofstream os(fs::path(cfg.out) / "steps.csv");
    os << "k,clock_start,dt,max_load,active_count";
    for (int g = 0; g < cfg.sim.workers; ++g) os << ",load_" << g;
    os << "\n";
    os.precision(17);
    for (const auto& s : out.steps) {
      os << s.k << ',' << s.clock_start << ',' << s.dt << ',' << s.max_load << ',' << s.active_count;
      for (double l : s.loads) os << ',' << l;
      os << "\n";
    }
  }
  return out.completed_all ? 0 : 2;
}

void metric_row(std::ostream& os, const MetricsReport& m) {
  os << m.avg_imbalance << ',' << m.throughput << ',' << m.tpot << ',' << m.energy;
}

int cmd_compare(const ExperimentConfig& cfg, const std::vector<std::string>& policies) {
  if (policies.size() < 2) {
    std::cerr << "compare: need at least two policies\n";
    return 1;
  }
  std::vector<Job> jobs;
  for (const auto& name : policies) jobs.push_back({cfg, policy_from_name(name), cfg.sim.horizon});
  auto outs = run_jobs(jobs);
  fs::create_directories(cfg.out);
  std::ofstream os(fs::path(cfg.out) / "compare.csv");
  os << "policy,avg_imbalance,throughput,tpot,energy\n";
  os.precision(17);
  bool all_complete = true;
  for (size_t i = 0; i < policies.size(); ++i) {
    all_complete = all_complete && outs[i].completed_all;
    os << policies[i] << ',';
    metric_row(os, outs[i].metrics);
    os << "\n";
  }
  return all_complete ? 0 : 2;
}

int cmd_sweep_h(const ExperimentConfig& cfg, const std::vector<int>& h_list) {
  PolicyKind policy = policy_from_name(cfg.policy_name);
  std::vector<Job> jobs;
  for (int h : h_list) jobs.push_back({cfg, policy, h});
  auto outs = run_jobs(jobs);
  fs::create_directories(cfg.out);
  std::ofstream os(fs::path(cfg.out) / "sweep_h.csv");
  os << "H,avg_imbalance,throughput,tpot,energy\n";
  os.precision(17);
  bool all_complete = true;
  for (size_t i = 0; i < h_list.size(); ++i) {
    all_complete = all_complete && outs[i].completed_all;
    os << h_list[i] << ',';
    metric_row(os, outs[i].metrics);
    os << "\n";
  }
  return all_complete ? 0 : 2;
}

int cmd_sweep_g(const ExperimentConfig& cfg, const std::vector<int>& g_list) {
  std::vector<Job> jobs;
  for (int g : g_list) {
    ExperimentConfig c = cfg;
    c.sim.workers = g;
    jobs.push_back({c, PolicyKind::Fcfs, cfg.sim.horizon});
    jobs.push_back({c, PolicyKind::BfioGreedy, cfg.sim.horizon});
  }
  auto outs = run_jobs(jobs);
  fs::create_directories(cfg.out);
  std::ofstream os(fs::path(cfg.out) / "sweep_g.csv");
  os << "G,policy,avg_imbalance,throughput,tpot,energy,saving_pct\n";
  os.precision(17);
  bool all_complete = true;
  for (size_t i = 0; i < g_list.size(); ++i) {
    const RunOutput &fcfs = outs[2 * i], &bfio = outs[2 * i + 1];
    all_complete = all_complete && fcfs.completed_all && bfio.completed_all;
    double saving =
        fcfs.metrics.energy > 0.0 ? 100.0 * (fcfs.metrics.energy - bfio.metrics.energy) / fcfs.metrics.energy : 0.0;
    os << g_list[i] << ",fcfs,";
    metric_row(os, fcfs.metrics);
    os << ",0\n" << g_list[i] << ",bfio-greedy,";
    metric_row(os, bfio.metrics);
    os << ',' << saving << "\n";
  }
  return all_complete ? 0 : 2;
}

int cmd_iir(const ExperimentConfig& cfg, const std::vector<int>& b_list, const std::vector<int>& g_list,
            int trials) {
#ifdef BFSIM_CLI_CPU
  IirEstimate est = estimate_iir(b_list, g_list, spec_of(cfg), trials, cfg.steps, cfg.warmup, cfg.sim.seed);
#else
  IirEstimate est = gpu::estimate_iir(device(), b_list, g_list, spec_of(cfg), trials, cfg.steps, cfg.warmup,
                                      cfg.sim.seed);
#endif
  fs::create_directories(cfg.out);
  std::ofstream os(fs::path(cfg.out) / "iir.csv");
  write_iir_csv(os, est);
  return 0;
}

int cmd_validate_trace(const std::string& path) {
  ArrivalInstance inst = load_trace(path);
  std::cout << "trace ok: " << inst.requests.size() << " requests\n";
  return 0;
}

// ---- arguments (the reference's option names, tools/bfsim.cpp:292-336) ----
std::vector<int> int_list(const std::string& v) {
  std::vector<int> out;
  std::stringstream ss(v);
  std::string tok;
  while (std::getline(ss, tok, ',')) out.push_back(std::stoi(tok));
  return out;
}
std::vector<std::string> str_list(const std::string& v) {
  std::vector<std::string> out;
  std::stringstream ss(v);
  std::string tok;
  while (std::getline(ss, tok, ',')) out.push_back(tok);
  return out;
}

// flat key=value config file, '#' comments (tools/bfsim.cpp:46-65); the keys
// map to the flags, which take precedence (:69-110)
void load_config(const std::string& path, std::map<std::string, std::string>& kv) {
  std::ifstream in(path);
  if (!in) throw std::runtime_error("config: cannot open " + path);
  std::string line;
  std::size_t lineno = 0;
  auto trim = [](std::string s) {
    std::size_t a = s.find_first_not_of(" \t"), b = s.find_last_not_of(" \t");
    return a == std::string::npos ? std::string{} : s.substr(a, b - a + 1);
  };
  while (std::getline(in, line)) {
    ++lineno;
    std::size_t first = line.find_first_not_of(" \t");
    if (first == std::string::npos || line[first] == '#') continue;
    std::size_t eq = line.find('=');
    if (eq == std::string::npos) throw std::runtime_error("config: missing '=' at line " + std::to_string(lineno));
    kv[trim(line.substr(0, eq))] = trim(line.substr(eq + 1));
  }
}

bool apply(ExperimentConfig& cfg, const std::string& key, const std::string& val) {
  if (key == "workers") cfg.sim.workers = std::stoi(val);
  else if (key == "batch") cfg.sim.batch = std::stoi(val);
  else if (key == "seed") cfg.sim.seed = std::stoull(val);
  else if (key == "policy") cfg.policy_name = val;
  else if (key == "horizon") cfg.sim.horizon = std::stoi(val);
  else if (key == "max_steps") cfg.sim.max_steps = std::stol(val);
  else if (key == "overhead") cfg.sim.overhead = std::stod(val);
  else if (key == "per_token") cfg.sim.per_token = std::stod(val);
  else if (key == "search_limit") cfg.sim.search_limit = std::stol(val);
  else if (key == "trace") cfg.trace = val;
  else if (key == "mode") cfg.mode = val;
  else if (key == "rate") cfg.rate = std::stod(val);
  else if (key == "duration") cfg.duration = std::stod(val);
  else if (key == "steps") cfg.steps = std::stol(val);
  else if (key == "warmup") cfg.warmup = std::stol(val);
  else if (key == "prefill_max") cfg.prefill_max = std::stoi(val);
  else if (key == "geo_p") cfg.geo_p = std::stod(val);
  else if (key == "drift") cfg.drift = std::stod(val);
  else if (key == "power.p_idle") cfg.sim.power.p_idle = std::stod(val);
  else if (key == "power.p_max") cfg.sim.power.p_max = std::stod(val);
  else if (key == "power.mfu_sat") cfg.sim.power.mfu_sat = std::stod(val);
  else if (key == "power.gamma") cfg.sim.power.gamma = std::stod(val);
  else if (key == "out") cfg.out = val;
  else if (key == "emit_steps") cfg.emit_steps = (val == "1" || val == "true");
  else return false;
  return true;
}

int usage() {
  std::cerr << "usage: bfsim_gpu {run|compare|sweep-h|sweep-g|iir|validate-trace} [--flag value ...]\n";
  return 1;
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2) return usage();
  const std::string sub = argv[1];
  ExperimentConfig cfg;
  std::string config_path, trace_path;
  std::vector<std::string> policies;
  std::vector<int> h_list, g_list, b_list;
  int trials = 20;
  std::map<std::string, std::string> given;  // flag keys given on the command line
  try {
    for (int i = 2; i < argc; ++i) {
      std::string a = argv[i];
      if (sub == "validate-trace" && a.rfind("--", 0) != 0) {
        trace_path = a;
        continue;
      }
      if (a.rfind("--", 0) != 0) return usage();
      std::string key = a.substr(2);
      if (key == "emit-steps") {
        cfg.emit_steps = true;
        given["emit_steps"] = "1";
        continue;
      }
      if (i + 1 >= argc) return usage();
      std::string val = argv[++i];
      if (key == "config") config_path = val;
      else if (key == "policies") policies = str_list(val);
      else if (key == "h-list") h_list = int_list(val);
      else if (key == "g-list") g_list = int_list(val);
      else if (key == "b-list") b_list = int_list(val);
      else if (key == "trials") trials = std::stoi(val);
      else {
        for (char& ch : key)
          if (ch == '-') ch = '_';
        if (!apply(cfg, key, val)) return usage();
        given[key] = val;
      }
    }
    if (!config_path.empty()) {
      std::map<std::string, std::string> kv;
      load_config(config_path, kv);
      for (const auto& [k, v] : kv) {
        if (given.count(k)) continue;
        if (!apply(cfg, k, v)) throw std::runtime_error("config: unknown key '" + k + "'");
      }
    }
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << "\n";
    return 1;
  }
  try {
    if (sub == "validate-trace") return trace_path.empty() ? usage() : cmd_validate_trace(trace_path);
    if (sub == "run") return cmd_run(cfg);
    if (sub == "compare") return cmd_compare(cfg, policies);
    if (sub == "sweep-h") {
      if (h_list.empty()) {
        std::cerr << "sweep-h: --h-list must be nonempty\n";
        return 1;
      }
      return cmd_sweep_h(cfg, h_list);
    }
    if (sub == "sweep-g") {
      if (g_list.empty()) {
        std::cerr << "sweep-g: --g-list must be nonempty\n";
        return 1;
      }
      return cmd_sweep_g(cfg, g_list);
    }
    if (sub == "iir") {
      if (b_list.empty() || g_list.empty()) {
        std::cerr << "iir: --b-list and --g-list must be nonempty\n";
        return 1;
      }
      return cmd_iir(cfg, b_list, g_list, trials);
    }
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << "\n";
    return 1;
  }
  return usage();
}
