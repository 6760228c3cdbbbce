#!/usr/bin/env python
"""Benchmark of the batched BF-IO step engine (BASELINE.json metric: simulated
worker-steps/s, % of HBM roofline, vs the host-CPU reference).

Workload (BASELINE.json configs[1], "C2"): per GPU, 256 seeds of
sample_instance(U[1,64] prefill, Geo(0.02) decode, lambda = 4000/s, 2.5 s,
drift 1) ~ 9.8k requests each, every seed simulated under bfio-greedy (H=0)
and jsq on G=16 workers with batch cap B=64 -> 512 trajectories per GPU.
One bench "step" = one pass of the hot path over that batch: every trajectory
simulated to completion with full outputs (per-step StepRecords, per-request
timings, MetricsReport).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N > 1 runs under torchrun (one rank per GPU, NCCL); seeds are sharded per
rank (weak scaling); time = max over ranks of the device-timed region.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

RATE, DURATION, S_MAX, GEO_P = 4000.0, 2.5, 64, 0.02
G, B = 16, 64
SEEDS_PER_GPU = 256
POLICIES = (("bfio-greedy", 3, 0), ("jsq", 1, 0))
WORKLOAD = "C2: G=16, B=64, 256 seeds x {bfio-greedy H=0, jsq}, lambda=4000/s x 2.5 s (~9.8k requests/trace)"
METRIC = "simulated worker-steps/sec (1/2/4/8 B200) + % HBM roofline vs host-CPU ref"
UNIT = "worker-steps/s"


def algorithmic_bytes(n_requests, workers, steps):
    """SURVEY.md §8(d), emit mode: trace 16 B/request read once; per step
    8*G (f64 loads) + 32 (clock_start, dt, max_load, active_count); per request
    24 (start step, worker, admit clock, finish clock); 56 B of metrics."""
    return 16 * n_requests + (8 * workers + 32) * steps + 24 * n_requests + 56


def env_rank():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("LOCAL_RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))


def make_workload(rank):
    from paper_2601_17855_b200 import abi, host

    traces, scen = [], []
    for j in range(SEEDS_PER_GPU):
        seed = rank * SEEDS_PER_GPU + j + 1
        traces.append(host.sample_instance(seed, rate=RATE, duration=DURATION, s_max=S_MAX, p=GEO_P))
        for name, pol, H in POLICIES:
            scen.append(abi.scenario(policy=pol, workers=G, batch=B, horizon=H, input_id=j, drift=1.0, seed=seed))
    return traces, np.array(scen, abi.scenario_dtype)


class ClockSampler:
    """Samples SM clock and throttle reasons via NVML while the timed region runs."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
        0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
        0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting",
    }

    def __init__(self, device):
        self.device = device
        self.samples, self.reasons = [], set()
        self.max_mhz = None
        self._stop = threading.Event()
        self._t = None

    def __enter__(self):
        try:
            import pynvml

            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.device)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)

            def loop():
                while not self._stop.is_set():
                    try:
                        self.samples.append(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM))
                        r = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                        for bit, name in self.REASONS.items():
                            if r & bit and bit != 0x1:
                                self.reasons.add(name)
                    except Exception:
                        pass
                    self._stop.wait(0.05)

            self._t = threading.Thread(target=loop, daemon=True)
            self._t.start()
        except Exception as e:  # NVML unavailable: report it
            self.reasons.add(f"nvml_unavailable:{type(e).__name__}")
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join()

    def summary(self):
        med = statistics.median(self.samples) if self.samples else None
        return {"sm_mhz": med, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": len(self.samples)}


def measured_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def ncu_traffic():
    """dram bytes per launch of the greedy step kernel from the committed ncu capture."""
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return d.get("dram_bytes_per_launch"), d.get("kernel")
    except Exception:
        return None, None


def cpu_baseline(scen, traces, seconds_target=20.0):
    """The reference (oracle/_ref, the unmodified headers) on the host cores:
    run() + compute_metrics per scenario, one scenario per thread, all threads."""
    from oracle.oracle import RefLib, ref_available
    from paper_2601_17855_b200 import host

    if not ref_available():
        return None
    ref = RefLib()
    pool = host.InputPool(traces)
    threads = os.cpu_count() or 1
    # size the sample: first pass on a small prefix, then enough for ~seconds_target
    n0 = min(len(scen), 2 * threads)
    sec0, ws0 = ref.bench_poisson(scen[:n0], pool.inputs, pool.records, threads)
    rate0 = ws0 / max(sec0, 1e-9)
    per_scen = ws0 / n0
    n = int(min(len(scen), max(n0, seconds_target * rate0 / max(per_scen, 1))))
    sec, ws = ref.bench_poisson(scen[:n], pool.inputs, pool.records, threads)
    return {"value": ws / sec, "unit": UNIT, "cores": threads, "kind": "reference",
            "sample": f"{n} of {len(scen)} scenarios of the same batch (seeds 1..{(n + 1) // 2}, both policies), "
                      f"{ws} worker-steps in {sec:.2f} s on {threads} host threads "
                      f"(oracle/_ref: reference headers, g++ -O2 -ffp-contract=off)"}


def run_reference(args):
    rank, local, world = env_rank()
    if rank != 0:
        return 0
    from oracle.oracle import RefLib, ref_available
    from paper_2601_17855_b200 import host

    if not ref_available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libbfsim_ref.so not built"}))
        return 0
    traces, scen = make_workload(0)
    pool = host.InputPool(traces)
    ref = RefLib()
    threads = os.cpu_count() or 1
    per_step = max(threads, 32)  # bounded sample of the batch per step
    tot_ws, tot_s = 0, 0.0
    cursor = 0
    for i in range(args.warmup + args.steps):
        idx = [(cursor + j) % len(scen) for j in range(per_step)]
        cursor += per_step
        sec, ws = ref.bench_poisson(scen[idx], pool.inputs, pool.records, threads)
        if i >= args.warmup:
            tot_ws += ws
            tot_s += sec
    value = tot_ws / tot_s
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot_s / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int64/f64",
        "data": "synthetic", "config": {"workload": WORKLOAD, "sample_per_step": per_step},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "reference",
                         "sample": f"{per_step} scenarios per step of the {len(scen)}-scenario batch, run()+compute_metrics"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))
    return 0


def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_2601_17855_b200 import abi, host

    rank, local, world = env_rank()
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)

    traces, scen = make_workload(rank)
    pool = host.InputPool(traces)
    ctx = host.Context(local)
    n_req = pool.inputs["length"][scen["input_id"]].astype(np.int64)

    # calibration pass (metrics only) -> exact step counts -> exact sinks
    cal = host.DeviceBatch(ctx, scen, pool, emit_steps=False, emit_requests=False)
    cal.run()
    torch.cuda.synchronize(dev)
    K = cal.result_array()["steps_run"].astype(np.int64)
    db = host.DeviceBatch(ctx, scen, pool, emit_steps=True, emit_requests=True, step_capacity=np.maximum(K, 1))
    worker_steps = int((K * scen["workers"]).sum())
    alg = int(sum(algorithmic_bytes(int(n), int(g), int(k)) for n, g, k in zip(n_req, scen["workers"], K)))
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)  # > 126 MB L2

    for _ in range(args.warmup):
        db.run()
    barrier()
    evs = []
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            db.run()
            e1.record()
            evs.append((e0, e1))
        barrier()
    launches = ctx.last_launches * args.steps
    ms = sum(a.elapsed_time(b) for a, b in evs)
    res = db.result_array()
    assert (res["status"] == abi.OK).all(), "a trajectory did not complete"

    # each policy family timed alone (CUDA events); the bfio-greedy one is the
    # dominant kernel and carries the roofline
    def time_alone(idx, reps=5):
        b = host.DeviceBatch(ctx, scen[idx], pool, emit_steps=True, emit_requests=True,
                             step_capacity=np.maximum(K[idx], 1))
        b.run()
        evs = []
        for _ in range(reps):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            b.run()
            e1.record()
            evs.append((e0, e1))
        torch.cuda.synchronize(dev)
        return statistics.mean(a.elapsed_time(b_) for a, b_ in evs)

    per_policy_ms = {}
    for name, pol, _ in POLICIES:
        per_policy_ms[name] = time_alone(np.nonzero(scen["policy"] == pol)[0])
    gi = np.nonzero(scen["policy"] == abi.BFIO_GREEDY)[0]
    g_ms = per_policy_ms["bfio-greedy"]
    g_alg = int(sum(algorithmic_bytes(int(n_req[i]), int(scen["workers"][i]), int(K[i])) for i in gi))

    # end to end through the host-pointer C ABI: pinned host buffers, H2D of
    # traces + D2H of every output inside each timed call
    pb = host.PinnedBatch(ctx, scen, pool, step_capacity=np.maximum(K, 1))
    pb.run()
    barrier()
    e2e_evs = []
    for _ in range(args.steps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        r2 = pb.run()
        e1.record()
        e2e_evs.append((e0, e1))
    barrier()
    e2e_ms = sum(a.elapsed_time(b) for a, b in e2e_evs)
    assert np.array_equal(r2["imb_total_i"], res["imb_total_i"])

    # cross-rank: max time (device-timed), total work; the final metric
    # reduction over NCCL (parallel.gather_results / allreduce_exact)
    from paper_2601_17855_b200 import parallel

    t = torch.tensor([ms, e2e_ms], dtype=torch.float64, device=dev)
    w = torch.tensor([worker_steps], dtype=torch.int64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.all_reduce(w, op=dist.ReduceOp.SUM)
    exact = parallel.allreduce_exact(res, device=dev)
    allres = parallel.gather_results(res, rank * scen.shape[0], world * scen.shape[0], device=dev)
    w = torch.tensor([int(w[0]), exact[0], exact[1]], dtype=torch.int64)
    ms_max, e2e_max = float(t[0]), float(t[1])
    total_ws = int(w[0]) * args.steps
    value = total_ws / (ms_max / 1e3)
    e2e_value = total_ws / (e2e_max / 1e3)

    if rank == 0:
        peak, peak_src = measured_peak()
        achieved = g_alg / (g_ms / 1e3) / 1e9
        traffic, traffic_kernel = ncu_traffic()
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            cpu = cpu_baseline(scen, traces)
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "int64/f64", "data": "synthetic",
            "config": {
                "workload": WORKLOAD, "workers": G, "batch": B, "seeds_per_gpu": SEEDS_PER_GPU,
                "trajectories_per_gpu": int(scen.shape[0]), "requests_per_gpu": int(n_req.sum() // 2),
                "simulated_steps_per_gpu": int(K.sum()), "outputs": "StepRecords + request timings + MetricsReport",
                "l2": "flushed between timed iterations (256 MiB device write, outside the events)",
                "parallelism": f"scenario shards x{world} (no data-path collective; NCCL all-reduce of metrics)",
            },
            "roofline": {
                "bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                "traffic": traffic,
                "kernel": "step_kernel<Poisson, bfio-greedy> (256 trajectories, timed alone, CUDA events)",
                "kernel_ms": g_ms, "algorithmic_bytes": g_alg, "peak_source": peak_src,
                "traffic_source": traffic_kernel,
            },
            "per_policy_kernel_ms": per_policy_ms,
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": pb.h2d_bytes,
                    "d2h_bytes_per_step": pb.d2h_bytes, "ms_per_step": e2e_max / args.steps},
            "gpu_launches": int(launches),
            "clocks": clk.summary(),
            "imbalance_check": {"imb_total_i_sum": int(w[1]), "total_workload_i_sum": int(w[2]),
                                "trajectories_gathered": int(allres.shape[0])},
        }
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()
    ctx.close()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=("ours", "reference"))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
