#!/usr/bin/env python
"""Benchmark of the batched BF-IO step engine (BASELINE.json metric: simulated
worker-steps/s, % of HBM roofline, vs the host-CPU reference).

Default workload (BASELINE.json configs[1], "C2"): per GPU, 256 seeds of
sample_instance(U[1,64] prefill, Geo(0.02) decode, lambda = 4000/s, 2.5 s,
drift 1) ~ 9.8k requests each, every seed simulated under bfio-greedy (H=0)
and jsq on G=16 workers with batch cap B=64 -> 512 trajectories per GPU.
One bench "step" = one pass of the hot path over that batch: every trajectory
simulated to completion with full outputs (per-step StepRecords, per-request
timings, MetricsReport).

The other BASELINE configs are available as supplementary lines
(--config c1|c3|c4|c5; see CONFIGS below and DESIGN.md §6).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config c2]

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

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "simulated worker-steps/sec (1/2/4/8 B200) + % HBM roofline vs host-CPU ref"
UNIT = "worker-steps/s"


def env_rank():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("LOCAL_RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))


# --------------------------------------------------------------------------
# Workloads. Each returns a dict: scen (scenario table), inputs (traces or
# streams), emit (full outputs?), workload text, groups (label -> mask) for
# per-family kernel timing, and the CPU-baseline sampler.


def _poisson(traces, rows, workload, emit, cpu_n, extra=None):
    from paper_2601_17855_b200 import abi

    scen = np.array(rows, abi.scenario_dtype)
    groups = {}
    for s_idx, s in enumerate(scen):
        lab = f"{abi.POLICY_LABELS[int(s['policy'])]}" + (f" H={int(s['horizon'])}" if s["horizon"] else "")
        if s["lookahead"] == abi.NOISY and s["noise_sigma"] > 0 and s["horizon"] > 0:
            lab += f" noisy sigma={float(s['noise_sigma']):g}"
        groups.setdefault(lab, []).append(s_idx)
    return dict(kind="poisson", scen=scen, inputs=traces, emit=emit, workload=workload, groups=groups,
                cpu_n=cpu_n, extra=extra or {})


def wl_c1(rank, args):
    """BASELINE configs[0]: single trace, G=8, B=64, ~2k requests (lambda=2000/s,
    1 s, seed 1): bfio-greedy H=0/H=20 vs fcfs (the reference's stand-in for
    round-robin, SURVEY §7 hard part 7)."""
    from paper_2601_17855_b200 import abi, host

    tr = host.sample_instance(1 + rank, rate=2000.0, duration=1.0, s_max=64, p=0.02)
    rows = [abi.scenario(policy=p, workers=8, batch=64, horizon=H, input_id=0, drift=1.0)
            for p, H in ((abi.BFIO_GREEDY, 0), (abi.BFIO_GREEDY, 20), (abi.FCFS, 0))]
    return _poisson([tr], rows, "C1: G=8, B=64, 1 trace (lambda=2000/s x 1 s, N=1957) x {bfio-greedy H=0, H=20, fcfs}",
                    True, 3)


def wl_c2(rank, args):
    """BASELINE configs[1] (the headline)."""
    from paper_2601_17855_b200 import abi, host

    seeds = args.seeds or 256
    traces, rows = [], []
    for j in range(seeds):
        seed = rank * seeds + j + 1
        traces.append(host.sample_instance(seed, rate=4000.0, duration=2.5, s_max=64, p=0.02))
        for pol in (abi.BFIO_GREEDY, abi.JSQ):
            rows.append(abi.scenario(policy=pol, workers=16, batch=64, horizon=0, input_id=j, drift=1.0, seed=seed))
    return _poisson(traces, rows, f"C2: G=16, B=64, {seeds} seeds x {{bfio-greedy H=0, jsq}}, lambda=4000/s x 2.5 s "
                                  "(~9.8k requests/trace)", True, None)


def wl_c3(rank, args):
    """BASELINE configs[2]: G=64, B=64, 100k requests (lambda=8000/s x 12.5 s),
    1k seeds, bfio-greedy H=20 with Noisy lookahead sigma=2."""
    from paper_2601_17855_b200 import abi, host

    seeds = args.seeds or 1000
    traces, rows = [], []
    for j in range(seeds):
        seed = rank * seeds + j + 1
        traces.append(host.sample_instance(seed, rate=8000.0, duration=12.5, s_max=64, p=0.02))
        rows.append(abi.scenario(policy=abi.BFIO_GREEDY, workers=64, batch=64, horizon=20, input_id=j, drift=1.0,
                                 lookahead=abi.NOISY, noise_sigma=2.0, seed=seed))
    return _poisson(traces, rows, f"C3: G=64, B=64, {seeds} seeds x bfio-greedy H=20 Noisy(sigma=2), "
                                  "lambda=8000/s x 12.5 s (~100k requests/trace), metrics-only outputs", False, 16)


def wl_c5(rank, args):
    """BASELINE configs[4]: fleet scale. A shared pool of 64 traces
    (lambda=8000/s x 125 s, ~1M requests each); scenarios = trace x
    {fcfs, jsq, bfio-greedy H=0, bfio-greedy H=20 Noisy sigma=2 (seeded)}, G=B=64,
    metrics-only. 65,536 scenarios over 8 GPUs is 8,192 per GPU; --scenarios
    sets the per-GPU count (default 1,024, a stated subset)."""
    from paper_2601_17855_b200 import abi, host

    n_traces = 64
    per_gpu = args.scenarios or 1024
    traces = [host.sample_instance(t + 1, rate=8000.0, duration=125.0, s_max=64, p=0.02) for t in range(n_traces)]
    combos = [(abi.FCFS, 0, abi.PERFECT), (abi.JSQ, 0, abi.PERFECT), (abi.BFIO_GREEDY, 0, abi.PERFECT),
              (abi.BFIO_GREEDY, 20, abi.NOISY)]
    rows = []
    for j in range(per_gpu):
        g = rank * per_gpu + j  # global scenario index
        tid = g % n_traces
        pol, H, la = combos[(g // n_traces) % len(combos)]
        rows.append(abi.scenario(policy=pol, workers=64, batch=64, horizon=H, input_id=tid, drift=1.0, lookahead=la,
                                 noise_sigma=2.0 if la == abi.NOISY else 0.0, seed=1 + g))
    return _poisson(traces, rows, f"C5: {per_gpu} scenarios/GPU of the 65,536-scenario grid (64 shared traces x "
                                  "~1M requests, lambda=8000/s x 125 s; fcfs/jsq/greedy H0/greedy H20 noisy), "
                                  "G=B=64, metrics-only outputs", False, 16)


def wl_c4(rank, args):
    """BASELINE configs[3]: run_overloaded worker-count sweep G=8..1024, B=64,
    4 policies (fcfs, jsq, bfio-greedy H=0 at drift 0; bfio-greedy H=20 at
    drift 1, acceptance C05), 2000+200 steps, OverloadedSpec defaults. Seed s is
    shared by every G (one pre-generated (s,o) stream per seed).
    --seeds sets seeds per G (default 32 of the config's 4k)."""
    from paper_2601_17855_b200 import abi, host

    seeds = args.seeds or 32
    Gs = [int(x) for x in (args.workers or "8,16,32,64,128,256,512,1024").split(",")]
    B, steps, warm, p = 64, 2000, 200, 0.02
    n = int(max(Gs) * B * (2 + (steps + warm) * p * 1.3)) + 8192
    streams = [host.sample_stream(rank * seeds + j + 1, n, s_max=64, p=p) for j in range(seeds)]
    combos = [(abi.FCFS, 0, 0.0), (abi.JSQ, 0, 0.0), (abi.BFIO_GREEDY, 0, 0.0), (abi.BFIO_GREEDY, 20, 1.0)]
    rows, groups = [], {}
    for G in Gs:
        for pol, H, drift in combos:
            lab = f"G={G} {abi.POLICY_LABELS[pol]}" + (f" H={H}" if H else "")
            for j in range(seeds):
                groups.setdefault(lab, []).append(len(rows))
                rows.append(abi.scenario(mode=abi.OVERLOADED, policy=pol, workers=G, batch=B, horizon=H, drift=drift,
                                         steps=steps, warmup=warm, seed=rank * seeds + j + 1, input_id=j))
    scen = np.array(rows, abi.scenario_dtype)
    return dict(kind="overloaded", scen=scen, inputs=streams, emit=False, groups=groups, cpu_n=None,
                workload=f"C4: run_overloaded G in {Gs}, B=64, {seeds} seeds/G x {{fcfs, jsq, bfio-greedy H=0 (drift 0), "
                         "bfio-greedy H=20 (drift 1)}}, 2000+200 steps, metrics-only outputs",
                extra={"workers": Gs})


CONFIGS = {"c1": wl_c1, "c2": wl_c2, "c3": wl_c3, "c4": wl_c4, "c5": wl_c5}


def algorithmic_bytes(wl, n_inputs_len, scen, K):
    """trace 16 B/request (Poisson) or 8 B/sample consumed
    (overloaded) read once; in emit mode per step 8*G (f64 loads) + 32
    (clock_start, dt, max_load, active_count) and per request 24 (start step,
    worker, admit clock, finish clock); 56 B of metrics per scenario."""
    G = scen["workers"].astype(np.int64)
    if wl["kind"] == "poisson":
        n = n_inputs_len
        b = 16 * n + 56
        if wl["emit"]:
            b = b + (8 * G + 32) * K + 24 * n
        return b
    return 8 * n_inputs_len + 56  # overloaded: n_inputs_len = samples consumed


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
                    self._stop.wait(0.02)

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


def ncu_traffic(config):
    """dram bytes per launch of the dominant step kernel from the committed ncu
    capture, plus that capture's issue-slot and warp activity (the kernel is
    latency-bound: these say how far from issue-bound it is)."""
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(p) as f:
            d = json.load(f)
        d = d.get(config, d if config == "c2" else {})
        return d.get("dram_bytes_per_launch"), d.get("kernel"), {
            "issue_active": d.get("issue_active"), "warps_active": d.get("warps_active")}
    except Exception:
        return None, None, {}


# --------------------------------------------------------------- CPU baseline
def cpu_baseline(wl, pool, seconds_target=20.0):
    """The reference (oracle/_ref, the unmodified headers) on the host cores:
    run() / run_overloaded() + compute_metrics per scenario, one scenario per
    thread, all threads; a bounded sample of the same workload."""
    from oracle.oracle import RefLib, ref_available

    if not ref_available():
        return None
    ref = RefLib()
    threads = os.cpu_count() or 1
    scen = wl["scen"]
    if wl["kind"] == "overloaded":
        # per G: `threads` scenarios, step prefix scaled so the sample stays bounded
        tot_s, tot_ws, desc = 0.0, 0, []
        for G in wl["extra"]["workers"]:
            idx = np.nonzero(scen["workers"] == G)[0]
            sub = scen[idx][:: max(1, len(idx) // threads)][:threads].copy()
            scale = max(1, G // 32)
            sub["steps"] = np.maximum(20, sub["steps"] // (scale * scale))
            sub["warmup"] = np.maximum(5, sub["warmup"] // (scale * scale))
            sec, ws = ref.bench_overloaded(sub, threads)
            tot_s += sec
            tot_ws += ws
            desc.append(f"G={G}: {len(sub)} runs x {int(sub['warmup'][0])}+{int(sub['steps'][0])} steps, "
                        f"{ws / sec:.3g} ws/s")
        return {"value": tot_ws / tot_s, "unit": UNIT, "cores": threads, "kind": "reference",
                "sample": "run_overloaded step prefixes, all 4 policies mixed; " + "; ".join(desc)}
    n0 = min(len(scen), wl["cpu_n"] or 2 * threads)
    sec0, ws0 = ref.bench_poisson(scen[:n0], pool.inputs, pool.records, threads)
    n = n0
    if wl["cpu_n"] is None:
        rate0 = ws0 / max(sec0, 1e-9)
        per_scen = ws0 / n0
        n = int(min(len(scen), max(n0, seconds_target * rate0 / max(per_scen, 1))))
        sec, ws = ref.bench_poisson(scen[:n], pool.inputs, pool.records, threads)
    else:
        sec, ws = sec0, ws0
    return {"value": ws / sec, "unit": UNIT, "cores": threads, "kind": "reference",
            "sample": f"{n} of {len(scen)} scenarios of the same batch, {ws} worker-steps in {sec:.2f} s on "
                      f"{threads} host threads (oracle/_ref: reference headers, g++ -O2 -ffp-contract=off)"}


def run_reference(args):
    rank, local, world = env_rank()
    if rank != 0:
        return 0
    from oracle.oracle import RefLib, ref_available
    from paper_2601_17855_b200 import host

    if not ref_available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libbfsim_ref.so not built"}))
        return 0
    wl = CONFIGS[args.config](0, args)
    scen = wl["scen"]
    ref = RefLib()
    threads = os.cpu_count() or 1
    tot_ws, tot_s = 0, 0.0
    cursor = 0
    if wl["kind"] == "overloaded":
        pool = None
        per_step = threads
    else:
        pool = host.InputPool(wl["inputs"])
        per_step = max(threads, 32) if wl["cpu_n"] is None else wl["cpu_n"]
    for i in range(args.warmup + args.steps):
        idx = [(cursor + j) % len(scen) for j in range(per_step)]
        cursor += per_step
        if wl["kind"] == "overloaded":
            sub = scen[idx].copy()
            big = sub["workers"] >= 256
            sub["steps"][big] = 40
            sub["warmup"][big] = 10
            sec, ws = ref.bench_overloaded(sub, threads)
        else:
            sec, ws = ref.bench_poisson(scen[idx], pool.inputs, pool.records, threads)
        if i >= args.warmup:
            tot_ws += ws
            tot_s += sec
    value = tot_ws / tot_s
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot_s / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int64/f64",
        "data": "synthetic", "config": {"workload": wl["workload"], "sample_per_step": per_step},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "reference",
                         "sample": f"{per_step} scenarios per step of the {len(scen)}-scenario batch, "
                                   "run()/run_overloaded() + compute_metrics"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))
    return 0


# --------------------------------------------------------------- our engine
def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_2601_17855_b200 import abi, host, parallel

    rank, local, world = env_rank()
    # one process per GPU; the modulo and the backend override only matter
    # for exercising the multi-rank path on a single-GPU box (gloo)
    local = local % max(1, torch.cuda.device_count())
    if world > 1:
        torch.cuda.set_device(local)
        backend = os.environ.get("BFSIM_DIST_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)

    wl = CONFIGS[args.config](rank, args)
    scen = wl["scen"]
    pool = host.InputPool(wl["inputs"])
    ctx = host.Context(local)
    emit = wl["emit"]
    n_in = pool.inputs["length"][scen["input_id"]].astype(np.int64)

    # calibration pass (metrics only) -> exact step counts -> exact sinks
    cal = host.DeviceBatch(ctx, scen, pool, emit_steps=False, emit_requests=False)
    cal.run()
    torch.cuda.synchronize(dev)
    cres = cal.result_array()
    K = cres["steps_run"].astype(np.int64)
    del cal
    db = host.DeviceBatch(ctx, scen, pool, emit_steps=emit, emit_requests=emit,
                          step_capacity=np.maximum(K, 1) if emit else None)
    worker_steps = int((K * scen["workers"]).sum())
    read_len = n_in if wl["kind"] == "poisson" else cres["consumed"].astype(np.int64)
    alg = algorithmic_bytes(wl, read_len, scen, K)
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
    assert np.array_equal(res["imb_total_i"], cres["imb_total_i"]), "runs disagree"

    # each kernel family timed alone (CUDA events on the launching stream);
    # the slowest carries the roofline
    def time_alone(idx, reps=3):
        b = host.DeviceBatch(ctx, scen[idx], pool, emit_steps=emit, emit_requests=emit,
                             step_capacity=np.maximum(K[idx], 1) if emit else None)
        b.run()
        e = []
        for _ in range(reps):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            b.run()
            e1.record()
            e.append((e0, e1))
        torch.cuda.synchronize(dev)
        return statistics.mean(a.elapsed_time(b_) for a, b_ in e)

    per_group = {}
    if not args.no_groups:
        for lab, idx in wl["groups"].items():
            per_group[lab] = time_alone(np.asarray(idx))
    dom = max(per_group, key=per_group.get) if per_group else None
    dom_idx = np.asarray(wl["groups"][dom]) if dom else np.arange(len(scen))
    dom_ms = per_group[dom] if dom else ms / args.steps
    dom_alg = int(alg[dom_idx].sum())

    # end to end through the host-pointer C ABI: pinned host buffers, H2D of
    # the inputs + D2H of every output inside each timed call
    pb = host.PinnedBatch(ctx, scen, pool, step_capacity=np.maximum(K, 1) if emit else None, emit_requests=emit)
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
    t = torch.tensor([ms, e2e_ms], dtype=torch.float64, device=dev)
    w = torch.tensor([worker_steps], dtype=torch.int64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.all_reduce(w, op=dist.ReduceOp.SUM)
    exact = parallel.allreduce_exact(res, device=dev)
    allres = parallel.gather_results(res, rank * scen.shape[0], world * scen.shape[0], device=dev)
    ms_max, e2e_max = float(t[0]), float(t[1])
    total_ws = int(w[0]) * args.steps
    value = total_ws / (ms_max / 1e3)
    e2e_value = total_ws / (e2e_max / 1e3)

    if rank == 0:
        peak, peak_src = measured_peak()
        achieved = dom_alg / (dom_ms / 1e3) / 1e9
        traffic, traffic_kernel, activity = ncu_traffic(args.config)
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            cpu = cpu_baseline(wl, pool)
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "int64/f64", "data": "synthetic",
            "config": {
                "workload": wl["workload"], "config": args.config,
                "trajectories_per_gpu": int(scen.shape[0]), "inputs_per_gpu": len(wl["inputs"]),
                "records_per_gpu": int(pool.records.shape[0]),
                "simulated_steps_per_gpu": int(K.sum()), "worker_steps_per_gpu": worker_steps,
                "outputs": "StepRecords + request timings + MetricsReport" if emit else "MetricsReport (+exact sums)",
                "l2": "flushed between timed iterations (256 MiB device write, outside the events)",
                "parallelism": f"scenario shards x{world} (no data-path collective; NCCL all-reduce of metrics)",
            },
            "roofline": {
                "bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                "traffic": traffic,
                "kernel": f"step_kernel family '{dom}' ({len(dom_idx)} trajectories, timed alone, CUDA events)",
                "kernel_ms": dom_ms, "algorithmic_bytes": dom_alg, "peak_source": peak_src,
                "traffic_source": traffic_kernel,
                "ncu_activity": activity,
            },
            "per_family_kernel_ms": per_group,
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": pb.h2d_bytes,
                    "d2h_bytes_per_step": pb.d2h_bytes, "ms_per_step": e2e_max / args.steps},
            "gpu_launches": int(launches),
            "clocks": clk.summary(),
            "imbalance_check": {"imb_total_i_sum": int(exact[0]), "total_workload_i_sum": int(exact[1]),
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
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--seeds", type=int, default=None, help="seeds per GPU (c2/c3) or per G (c4)")
    ap.add_argument("--scenarios", type=int, default=None, help="scenarios per GPU (c5)")
    ap.add_argument("--workers", default=None, help="comma-separated G list (c4)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-groups", action="store_true", help="skip the per-family kernel timings")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
