/*
 * bfsim_gpu.h — C ABI of the B200-native batched BF-IO step engine.
 *
 * This is the drop-in boundary for the per-step hot path of the reference
 * simulator (arXiv 2601.17855, /root/reference/proj/include/bfsim). The
 * reference evaluates one trajectory at a time through
 *
 *   SimResult run(const SimConfig&, const ArrivalInstance&)        engine.hpp:265
 *   std::vector<StepRecord> run_overloaded(PolicyKind, int H, int G, int B,
 *       long steps, long warmup, const OverloadedSpec&, uint64_t seed,
 *       long search_limit, std::vector<RequestTiming>* timings)    oracle.hpp:138-143
 *   MetricsReport compute_metrics(steps, requests, power)          metrics.hpp:106-126
 *   Allocation assign(PolicyKind, waiting, workers, H, limit)      policies.hpp:372-374
 *   IirEstimate estimate_iir(...)                                  oracle.hpp:263-317
 *
 * The GPU path evaluates many independent trajectories ("scenarios") in one
 * call. Every entry point takes plain pointers and sizes; no exception crosses
 * the ABI. Return codes map onto the reference's exception classes so the C++
 * wrapper (bfsim_gpu.hpp) rethrows exactly what the reference would throw:
 *
 *   BFSIM_OK          0  success
 *   BFSIM_EINVAL      1  std::invalid_argument   (engine.hpp:31-36, workload.hpp:65,74,
 *                                                  metrics_power.hpp:17-21)
 *   BFSIM_ELOGIC      2  std::logic_error        (engine.hpp:236-242)
 *   BFSIM_ECUDA       3  CUDA / NCCL failure (no reference analogue)
 *   BFSIM_PARTIAL     4  max_steps reached, completed_all == false (engine.hpp:171-173;
 *                        CLI exit 2 at tools/bfsim.cpp:192). Per-scenario status only.
 *   BFSIM_ESTREAM     5  overloaded sample stream exhausted: the host batcher
 *                        extends the stream and re-runs (never user visible from
 *                        the C++ wrapper)
 *   BFSIM_ELIMIT      6  SearchLimitExceeded (bfio-exact, policies.hpp:174-178)
 *   BFSIM_ERANGE      7  a GPU-path integer range was exceeded at run time (the
 *                        per-slot a = s - drift*x is int32: drift * steps must stay
 *                        below 2^31). No reference analogue (the reference's doubles
 *                        lose exactness instead); std::overflow_error in the wrapper.
 *
 * A context is bound to one CUDA device and is not thread-safe: use one
 * context per host thread (the reference: one Simulation owns its state,
 * engine.hpp:93-95; distinct simulations may run concurrently).
 */
#ifndef BFSIM_GPU_H_
#define BFSIM_GPU_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BFSIM_ABI_VERSION 1

#define BFSIM_OK 0
#define BFSIM_EINVAL 1
#define BFSIM_ELOGIC 2
#define BFSIM_ECUDA 3
#define BFSIM_PARTIAL 4
#define BFSIM_ESTREAM 5
#define BFSIM_ELIMIT 6 /* bfio-exact: SearchLimitExceeded (policies.hpp:174-178), a std::runtime_error */
#define BFSIM_ERANGE 7 /* GPU integer state range exceeded (drift * steps >= 2^31) */

/* PolicyKind, policies.hpp:16 (same numbering). */
#define BFSIM_POLICY_FCFS 0
#define BFSIM_POLICY_JSQ 1
#define BFSIM_POLICY_BFIO_EXACT 2 /* CPU-only (exponential search); GPU returns EINVAL */
#define BFSIM_POLICY_BFIO_GREEDY 3

/* LookaheadMode, policies.hpp:36 (same numbering). */
#define BFSIM_LOOKAHEAD_PERFECT 0
#define BFSIM_LOOKAHEAD_TRUNCATED 1
#define BFSIM_LOOKAHEAD_NOISY 2

/* Trajectory loop: Simulation::run (engine.hpp:168) or run_overloaded (oracle.hpp:138). */
#define BFSIM_MODE_POISSON 0
#define BFSIM_MODE_OVERLOADED 1

/* Result flags. */
#define BFSIM_FLAG_STEP_OVERFLOW 1u  /* more steps than step_capacity: records truncated */
#define BFSIM_FLAG_NOISE_NEAR_TIE 2u /* a noisy draw landed within 1e-12 of a lround tie */
#define BFSIM_FLAG_EMPTY 4u          /* zero step records (metrics left at zero, as tools/bfsim.cpp:133-137) */

/* One arrival: ArrivalRecord (workload.hpp:217-221) as a 16-byte record.
 * decode is int32 (the reference's long); the host batcher rejects o > INT32_MAX. */
typedef struct bfsim_request_t {
  double arrival_time;
  int32_t prefill;
  int32_t decode;
} bfsim_request_t;

/* One pre-generated overloaded sample: the (prefill.sample, decode.sample) pair
 * that run_overloaded draws at oracle.hpp:179-180, in draw order. */
typedef struct bfsim_sample_t {
  int32_t prefill;
  int32_t decode;
} bfsim_sample_t;

/* Per-input statistics the batcher computes once per trace / stream
 * (bfsim_prepare_input). class_base_offset indexes the class_base pool:
 * class_base[class_base_offset + c] = #records with prefill < c, c = 1..s_max+1
 * (a counting-sort layout used for the per-prefill-class waiting deques). */
typedef struct bfsim_input_t {
  int64_t offset;            /* first record in the trace or stream pool */
  int64_t length;            /* N (poisson) or stream length (overloaded) */
  int64_t class_base_offset; /* into the class_base pool */
  int32_t s_max;             /* largest prefill present */
  int32_t max_decode;        /* largest decode present */
} bfsim_input_t;

/* One scenario = one trajectory: SimConfig (engine.hpp:17-37) or the
 * run_overloaded argument list + OverloadedSpec (oracle.hpp:121-143). */
typedef struct bfsim_scenario_t {
  int32_t mode;      /* BFSIM_MODE_* */
  int32_t policy;    /* BFSIM_POLICY_* */
  int32_t lookahead; /* BFSIM_LOOKAHEAD_* (poisson only; overloaded is always perfect) */
  int32_t workers;   /* G */
  int32_t batch;     /* B */
  int32_t horizon;   /* H */
  int32_t input_id;  /* index into the bfsim_input_t table */
  int32_t reserved0;  /* ignored on input (the library's dyadic-drift shift) */
  double drift;       /* DriftSpec::constant(value): a non-negative integer, or dyadic m / 2^e
                         (e <= 16, s_max * 2^e <= 262143), exact like the reference's fp64 profile */
  double overhead;    /* C     */
  double per_token;   /* t_ell */
  double noise_sigma; /* Noisy lookahead sigma */
  double p_idle, p_max, mfu_sat, gamma; /* PowerModel, metrics_power.hpp:11-22 */
  double backlog;     /* OverloadedSpec::backlog */
  int64_t max_steps;  /* poisson step cap */
  int64_t steps;      /* overloaded measured steps */
  int64_t warmup;     /* overloaded warm-up steps */
  uint64_t seed;      /* SimConfig::seed (noisy lookahead RNG) */
  /* output slices (ignored when the corresponding sink is NULL) */
  int64_t step_offset;   /* first record in the step sink */
  int64_t step_capacity; /* records available at step_offset */
  int64_t load_offset;   /* first double in step sink `loads` (capacity * workers) */
  int64_t req_offset;    /* first entry in the request sink (input length entries) */
} bfsim_scenario_t;

/* Per-scenario outcome. The seven doubles avg_imbalance..eta_sum are
 * MetricsReport (metrics.hpp:96-104) computed as compute_metrics does. */
typedef struct bfsim_result_t {
  int32_t status; /* BFSIM_OK / BFSIM_PARTIAL / error code */
  uint32_t flags; /* BFSIM_FLAG_* */
  int64_t steps_run;  /* steps simulated (overloaded: warmup + steps) */
  int64_t records;    /* step records (poisson: steps_run; overloaded: steps) */
  int64_t completed;  /* completed requests (overloaded: includes warm-up) */
  int64_t admitted;   /* admitted requests */
  int64_t consumed;   /* overloaded: samples drawn from the stream */
  int64_t imb_total_i;      /* exact integer sum of G*max - sum over records (dyadic drift m / 2^e:
                               in units of 2^-e) */
  int64_t total_workload_i; /* exact integer sum of loads over records (same units) */
  int64_t tokens_i;         /* exact sum of active_count over records */
  double avg_imbalance, throughput, tpot, energy, imb_total, total_workload, eta_sum;
  double clock;   /* simulated clock after the last step */
  double elapsed; /* sum of dt over records */
  double tpot_sum;
} bfsim_result_t;

/* Per-step StepRecord sink (engine.hpp:39-48), SoA. Index step_offset + k;
 * loads at load_offset + k*G + g. Overloaded mode writes every simulated step
 * (warm-up included) so the caller can drop the first `warmup`. */
typedef struct bfsim_step_sink_t {
  double* clock_start;
  double* dt;
  double* max_load;
  int64_t* active_count;
  double* loads;
} bfsim_step_sink_t;

/* Per-request RequestTiming sink (engine.hpp:50-59), SoA, indexed by
 * req_offset + (trace index | stream sample index). -1 = never happened.
 * Overloaded ids are admission order (oracle.hpp:206): sort admitted samples by
 * (start_step, sample index). */
typedef struct bfsim_req_sink_t {
  int32_t* arrival_step; /* poisson reveal step (k_i) */
  int32_t* start_step;   /* x_i */
  int32_t* worker;       /* worker g the request was placed on */
  double* admit_clock;
  double* finish_clock; /* 0.0 when not completed */
} bfsim_req_sink_t;

typedef struct bfsim_ctx bfsim_ctx_t;

/* ---- context ---------------------------------------------------------- */
int bfsim_abi_version(void);
int bfsim_ctx_create(int device, bfsim_ctx_t** out, char* err, size_t errlen);
void bfsim_ctx_destroy(bfsim_ctx_t* ctx);
int bfsim_ctx_device(const bfsim_ctx_t* ctx);

/* ---- host batcher: synthetic inputs (byte-identical to the reference) ---- */
/* sample_instance(uniform(s_max), geometric(p), rate, duration, seed), workload.hpp:241-266.
 * prefill_kind: 0 uniform(s_max), 1 fixed(s_max). decode_kind: 0 geometric(p), 1 fixed(fixed_o).
 * Two-call: with out == NULL returns the count in *n_out; otherwise fills up to capacity. */
int bfsim_sample_instance(int prefill_kind, int s_max, int decode_kind, double p, int64_t fixed_o,
                          double rate, double duration, uint64_t seed, bfsim_request_t* out,
                          int64_t capacity, int64_t* n_out, char* err, size_t errlen);
/* The first n (prefill, decode) pairs run_overloaded draws from mt19937_64(seed)
 * (oracle.hpp:177-183). Policy-independent; only the number consumed varies. */
int bfsim_sample_stream(int prefill_kind, int s_max, int decode_kind, double p, int64_t fixed_o,
                        uint64_t seed, int64_t n, bfsim_sample_t* out, char* err, size_t errlen);
/* Any PrefillDistribution / DecodeDistribution (workload.hpp:87-215), including
 * the Empirical kinds (:109-118, :185-193):
 *   prefill kind 0 uniform(fixed = s_max), 1 fixed_value(fixed), 2 empirical(values)
 *   decode  kind 0 geometric(p), 1 fixed_length(fixed), 2 empirical(values)
 * An empirical draw is values[uniform_int_distribution<size_t>(0, n_values - 1)(rng)];
 * validation and messages follow the reference's factories. */
typedef struct bfsim_dist_t {
  int32_t kind;
  int32_t reserved;
  int64_t fixed;         /* uniform s_max / fixed value */
  double p;              /* geometric success probability */
  const int64_t* values; /* empirical list (kind 2) */
  int64_t n_values;
} bfsim_dist_t;
int bfsim_sample_instance_dist(const bfsim_dist_t* prefill, const bfsim_dist_t* decode, double rate,
                               double duration, uint64_t seed, bfsim_request_t* out, int64_t capacity,
                               int64_t* n_out, char* err, size_t errlen);
int bfsim_sample_stream_dist(const bfsim_dist_t* prefill, const bfsim_dist_t* decode, uint64_t seed, int64_t n,
                             bfsim_sample_t* out, char* err, size_t errlen);
/* Input statistics + class_base for a trace (records) or stream (samples).
 * class_base must hold s_max + 2 entries; call with class_base == NULL to learn s_max. */
int bfsim_prepare_trace(const bfsim_request_t* rec, int64_t n, bfsim_input_t* info,
                        int32_t* class_base, char* err, size_t errlen);
int bfsim_prepare_stream(const bfsim_sample_t* smp, int64_t n, bfsim_input_t* info,
                         int32_t* class_base, char* err, size_t errlen);

/* ---- batched step engine ------------------------------------------------ */
/* Host-pointer entry (the end-to-end path): copies inputs H2D, runs every
 * scenario, copies outputs D2H. Any sink pointer may be NULL. Step sinks in
 * page-locked host memory (cudaHostAlloc / cudaHostRegister) are written by
 * the kernels directly (zero-copy, overlapped with the simulation). Returns
 * the first error over scenarios (per-scenario status in results[i].status). */
int bfsim_run_batch(bfsim_ctx_t* ctx, const bfsim_scenario_t* scen, int64_t n_scen,
                    const bfsim_input_t* inputs, int32_t n_inputs, const int32_t* class_base,
                    int64_t n_class_base, const bfsim_request_t* traces, int64_t n_trace_records,
                    const bfsim_sample_t* streams, int64_t n_stream_samples,
                    const bfsim_step_sink_t* steps, int64_t n_step_records, int64_t n_load_values,
                    const bfsim_req_sink_t* reqs, int64_t n_req_entries, bfsim_result_t* results,
                    char* err, size_t errlen);

/* Device-pointer entry (inputs already resident in HBM): every pointer is a
 * device pointer except `scen_host`/`inputs_host` (validated and planned on
 * the host). Enqueued on `stream` (a cudaStream_t; NULL = legacy default);
 * returns after enqueueing. Results land in `results_dev`. */
int bfsim_run_batch_device(bfsim_ctx_t* ctx, const bfsim_scenario_t* scen_host, int64_t n_scen,
                           const bfsim_input_t* inputs_host, int32_t n_inputs,
                           const int32_t* class_base_dev, const bfsim_request_t* traces_dev,
                           const bfsim_sample_t* streams_dev, const bfsim_step_sink_t* steps_dev,
                           const bfsim_req_sink_t* reqs_dev, bfsim_result_t* results_dev,
                           void* stream, char* err, size_t errlen);

/* Kernel launches enqueued by the last bfsim_run_batch* call on this context
 * (the bench's gpu_launches claim) and the device time of its step kernels
 * in milliseconds (CUDA events on the launching stream; 0 when unavailable). */
int64_t bfsim_last_launch_count(const bfsim_ctx_t* ctx);
double bfsim_last_step_kernel_ms(const bfsim_ctx_t* ctx);

/* ---- batched policy operator ------------------------------------------- */
/* One assign() call (policies.hpp:372-382): `n_waiting` previews w[0..H]
 * (row-major doubles at preview_offset), G worker views (cap and active_count
 * at worker_offset, future[0..H] row-major at future_offset). The pairs
 * (waiting index, worker) land at pair_offset, 2 int32 each, in the order the
 * reference returns them; up to 2 * min(n_waiting, sum cap) int32. */
typedef struct bfsim_assign_call_t {
  int32_t policy;    /* BFSIM_POLICY_*, all four including bfio-exact */
  int32_t n_waiting;
  int32_t workers;   /* G, 1..32 (bfio-exact: 1..16) */
  int32_t horizon;   /* H, 0..64 (bfio-exact: 0..16) */
  int64_t preview_offset;
  int64_t worker_offset;
  int64_t future_offset;
  int64_t pair_offset;
} bfsim_assign_call_t;

/* Many independent assign() calls, one warp each on the device -- the
 * policy-level boundary the reference's unit tests and acceptance C01/C02
 * call (tests/policies_test.cpp, acceptance_test.cpp:117-169). Values must be
 * integers in [0, 2^31) (exact arithmetic). Per call: n_pairs,
 * cost (bfio-exact's cost_out, else 0) and status (BFSIM_OK or
 * BFSIM_ELIMIT when more than search_limit full allocations exist). */
int bfsim_assign_batch(bfsim_ctx_t* ctx, const bfsim_assign_call_t* calls, int64_t n_calls,
                       const double* previews, int64_t n_previews, const double* futures,
                       int64_t n_futures, const int32_t* caps, const int32_t* active_counts,
                       int64_t n_workers, int64_t search_limit, int32_t* pairs, int64_t n_pairs_cap,
                       int64_t* n_pairs, double* cost, int32_t* status, char* err, size_t errlen);

/* Reducer for estimate_iir (oracle.hpp:284-312): per cell, per-trial mean
 * imbalances of FCFS and BF-IO -> mean, SEM (n-1), ratio, propagated stderr.
 * out: 4 doubles per cell {fcfs_mean, bfio_mean, ratio, stderr}. */
int bfsim_iir_reduce(const double* fcfs_trial_means, const double* bfio_trial_means, int32_t trials,
                     int32_t n_cells, double* out, char* err, size_t errlen);

/* ---- device-side input generation ----------------------- */
/* One synthetic input: sample_instance(prefill, decode, rate, duration, seed)
 * (workload.hpp:241-266), or -- for the stream calls -- the first `samples`
 * (prefill, decode) pairs run_overloaded draws from mt19937_64(seed)
 * (oracle.hpp:177-183; rate/duration ignored). Empirical value lists are host
 * pointers. Output is byte-identical to bfsim_sample_instance_dist /
 * bfsim_sample_stream_dist (same libstdc++ draws, glibc's own log). */
typedef struct bfsim_gen_spec_t {
  bfsim_dist_t prefill;
  bfsim_dist_t decode;
  double rate;
  double duration;
  uint64_t seed;
} bfsim_gen_spec_t;
/* Pool sizes the generators need: records (traces: a Poisson(rate*duration)
 * bound per trace, mean + 12 sd + 64; streams: samples each) and class_base
 * entries (largest possible prefill + 2 each). stream_samples < 0 = traces. */
int bfsim_generate_bounds(const bfsim_gen_spec_t* specs, int32_t n, int64_t stream_samples, int64_t* n_records,
                          int64_t* n_class_base, char* err, size_t errlen);
/* Generate n traces into device memory (one warp per trace), with their
 * class_base tables; fills inputs_out[n] on the host (what bfsim_prepare_trace
 * computes), ready for bfsim_run_batch_device. Synchronizes `stream` (the
 * lengths are needed on the host to plan the run). */
int bfsim_generate_traces(bfsim_ctx_t* ctx, const bfsim_gen_spec_t* specs, int32_t n, bfsim_request_t* traces_dev,
                          int64_t n_records, int32_t* class_base_dev, int64_t n_class_base,
                          bfsim_input_t* inputs_out, void* stream, char* err, size_t errlen);
int bfsim_generate_streams(bfsim_ctx_t* ctx, const bfsim_gen_spec_t* specs, int32_t n, int64_t samples,
                           bfsim_sample_t* streams_dev, int64_t n_samples_cap, int32_t* class_base_dev,
                           int64_t n_class_base, bfsim_input_t* inputs_out, void* stream, char* err,
                           size_t errlen);
/* Host twin of the device's glibc log (csrc/libm_log.cuh), for the tests. */
void bfsim_libm_log_host(const double* x, double* y, int64_t n);

#ifdef __cplusplus
}
#endif

#endif /* BFSIM_GPU_H_ */
