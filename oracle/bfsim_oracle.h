/*
 * ORACLE / TEST INFRASTRUCTURE — not product code.
 *
 * Plain-C restatement of the reference hot path (arXiv 2601.17855,
 * /root/reference/proj/include/bfsim). Only tests/, __graft_entry__.smoke()
 * and bench.py's CPU-baseline leg may load liboracle.so. The product path
 * (paper_2601_17855_b200) never links or calls it.
 *
 * Parity pinning: the restatement is checked against the unmodified reference
 * headers compiled into oracle/_ref/libbfsim_ref.so (tests/test_oracle_vs_ref.py)
 * and against committed fixtures generated from that build
 * (tests/golden/make_golden.py). It shares only the plain record layouts of
 * include/bfsim_gpu.h.
 */
#ifndef BFSIM_ORACLE_H_
#define BFSIM_ORACLE_H_

#include <stdint.h>

#include "../include/bfsim_gpu.h"

#ifdef __cplusplus
extern "C" {
#endif

/* mt19937_64 as libstdc++ implements std::mersenne_twister_engine
 * (bits/random.h / random.tcc), plus generate_canonical<double,53>
 * (random.tcc:3349-3381) and normal_distribution's polar method
 * (random.tcc:1809-1844) with a fresh distribution object per call. */
typedef struct oracle_mt64_t {
  uint64_t mt[312];
  int idx;
} oracle_mt64_t;
void oracle_mt64_seed(oracle_mt64_t* g, uint64_t seed);
uint64_t oracle_mt64_next(oracle_mt64_t* g);
double oracle_canonical(oracle_mt64_t* g);
double oracle_normal(oracle_mt64_t* g, double mean, double sigma);

/* Simulation::run (engine.hpp:168-188) + compute_metrics (metrics.hpp:106-126).
 * Step sink arrays have step_cap entries (loads: step_cap*G); request sink
 * arrays have n entries. Any output pointer may be NULL.
 * Returns BFSIM_OK, BFSIM_PARTIAL (max_steps hit) or BFSIM_EINVAL. */
int oracle_run_poisson(const bfsim_scenario_t* sc, const bfsim_request_t* trace, int64_t n,
                       int64_t step_cap, double* clock_start, double* dt, double* max_load,
                       int64_t* active_count, double* loads, int32_t* arrival_step,
                       int32_t* start_step, int32_t* worker, double* admit_clock,
                       double* finish_clock, bfsim_result_t* res);

/* run_overloaded (oracle.hpp:138-244) over a pre-generated (s,o) stream (F11),
 * + compute_metrics(steps, timings, power). Step sinks receive ALL simulated
 * steps (warm-up included); metrics use steps >= warmup as the reference.
 * Per-sample sinks (stream_len entries) get start_step / worker. Timings are
 * emitted in the reference's completion order (oracle.hpp:225-240).
 * Returns BFSIM_OK, BFSIM_EINVAL or BFSIM_ESTREAM (stream too short). */
int oracle_run_overloaded(const bfsim_scenario_t* sc, const bfsim_sample_t* stream,
                          int64_t stream_len, int32_t s_max, int64_t step_cap,
                          double* clock_start, double* dt, double* max_load,
                          int64_t* active_count, double* loads, int32_t* start_step,
                          int32_t* worker, int64_t timing_cap, int32_t* t_id, double* t_admit,
                          double* t_finish, int64_t* t_decode, int64_t* n_timings,
                          bfsim_result_t* res);

/* assign() (policies.hpp:372-382) for fcfs / jsq / bfio-greedy on one step.
 * previews: n_waiting x (H+1); futures: G x (H+1). pairs: 2*U int32 in the
 * reference's output order. Returns BFSIM_OK or BFSIM_EINVAL (bfio-exact). */
int oracle_assign(int policy, int n_waiting, const double* previews, int G, const int32_t* caps,
                  const int32_t* active_counts, const double* futures, int H, int32_t* pairs,
                  int64_t* n_pairs);

#ifdef __cplusplus
}
#endif

#endif
