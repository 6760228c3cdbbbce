"""Where the C2 end-to-end time goes: total (events around the C-ABI call) vs
the step kernels inside it (bfsim_last_step_kernel_ms) vs host-side time."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import bench
from paper_2601_17855_b200 import host


class A:
    seeds = None


wl = bench.wl_c2(0, A)
pool = host.InputPool(wl["inputs"])
ctx = host.Context(0)
cal = host.DeviceBatch(ctx, wl["scen"], pool, emit_steps=False, emit_requests=False)
cal.run()
torch.cuda.synchronize()
K = cal.result_array()["steps_run"].astype(np.int64)
pb = host.PinnedBatch(ctx, wl["scen"], pool, step_capacity=np.maximum(K, 1))
for _ in range(3):
    pb.run()
for _ in range(5):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    pb.run()
    e1.record()
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    print(f"events {e0.elapsed_time(e1):.3f} ms  wall {1e3 * (t1 - t0):.3f} ms  kernels {ctx.last_kernel_ms:.3f} ms")
db = host.DeviceBatch(ctx, wl["scen"], pool, emit_steps=True, emit_requests=True, step_capacity=np.maximum(K, 1))
db.run()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
db.run()
e1.record()
torch.cuda.synchronize()
print(f"device-resident: {e0.elapsed_time(e1):.3f} ms")
