"""BASELINE configs[4] (C5) at its stated size on one B200: all 65,536
scenarios of the fleet grid once (bench.py's C5 line runs a prefix of the grid
so that a bench run stays within minutes).

The 64 shared traces (sample_instance, lambda = 8000/s x 125 s, ~1M requests
each) are generated in HBM by the device generator (bfsim_generate_traces,
SURVEY §8(f2)); scenario g = trace g % 64 x {fcfs, jsq, bfio-greedy H=0,
bfio-greedy H=20 Noisy sigma=2 (seed 1+g)}, G = B = 64, metrics-only outputs
(bench.wl_c5). The grid runs in chunks of --chunk scenarios, one
bfsim_run_batch_device call each, device-timed with CUDA events. Prints one
JSON line: worker-steps, device seconds, rate, statuses, exact metric sums.

    python tools/c5_full_grid.py [--scenarios 65536] [--chunk 8192] [--out gpurun_out/c5_full.json]
"""
import argparse
import json
import os
import sys
import time
import types

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2601_17855_b200 import abi, host  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--scenarios", type=int, default=65536)
    ap.add_argument("--chunk", type=int, default=8192)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    wl = bench.wl_c5(0, 1, types.SimpleNamespace(scenarios=a.scenarios))
    scen = wl["scen"]
    ctx = host.Context(0)
    t0 = time.perf_counter()
    pool = host.DevicePool(ctx, wl["specs"])
    torch.cuda.synchronize()
    gen_s = time.perf_counter() - t0
    res_all = np.zeros(scen.shape[0], abi.result_dtype)
    dev_ms = 0.0
    per_chunk = []
    for lo in range(0, scen.shape[0], a.chunk):
        sub = scen[lo:lo + a.chunk].copy()
        db = host.DeviceBatch(ctx, sub, pool, emit_steps=False, emit_requests=False)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        db.run()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        dev_ms += ms
        r = db.result_array()
        res_all[lo:lo + sub.shape[0]] = r
        ws = int((r["steps_run"].astype(np.int64) * sub["workers"]).sum())
        per_chunk.append({"first": lo, "n": int(sub.shape[0]), "ms": ms, "worker_steps": ws})
        print(f"chunk {lo}: {sub.shape[0]} scenarios, {ms:.0f} ms, {ws / (ms / 1e3):.3g} ws/s", flush=True)
        del db
    ws_total = int((res_all["steps_run"].astype(np.int64) * scen["workers"]).sum())
    line = {
        "config": "C5 full grid", "workload": wl["workload"].replace(f"0..{a.scenarios - 1}", f"all {a.scenarios}"),
        "scenarios": int(scen.shape[0]), "trace_records": int(pool.inputs["length"].sum()),
        "trace_generation_s": gen_s, "device_s": dev_ms / 1e3, "worker_steps": ws_total,
        "worker_steps_per_s": ws_total / (dev_ms / 1e3),
        "status_ok": int((res_all["status"] == abi.OK).sum()),
        "imb_total_i_sum": int(res_all["imb_total_i"].sum()),
        "total_workload_i_sum": int(res_all["total_workload_i"].sum()),
        "completed_sum": int(res_all["completed"].sum()), "chunks": per_chunk,
    }
    print(json.dumps(line))
    if a.out:
        with open(a.out, "w") as f:
            json.dump(line, f, indent=1)
    ctx.close()


if __name__ == "__main__":
    main()
