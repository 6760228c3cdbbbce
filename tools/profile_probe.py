"""Small single-launch workloads for ncu captures (scratch probe; not the bench).

    python tools/profile_probe.py c4fcfs|c4greedy|c3perfect|c3noisy|c2greedy
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2601_17855_b200 import abi, host

which = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 8
if which.startswith("c4"):
    G = 256 if "g256" in which else 1024
    pol = abi.FCFS if which == "c4fcfs" else abi.BFIO_GREEDY
    H, drift = (20, 1.0) if "h20" in which else (0, 0.0)
    steps, warm = 150, 50
    ln = int(G * 64 * (2 + (steps + warm) * 0.02 * 1.3)) + 4096
    inputs = [host.sample_stream(s, ln, s_max=64, p=0.02) for s in range(1, n + 1)]
    scs = [abi.scenario(mode=abi.OVERLOADED, policy=pol, workers=G, batch=64, steps=steps, warmup=warm, seed=s,
                        horizon=H, drift=drift, input_id=i) for i, s in enumerate(range(1, n + 1))]
elif which.startswith("c3"):
    noisy = which == "c3noisy"
    inputs = [host.sample_instance(s, rate=8000.0, duration=2.0, s_max=64, p=0.02) for s in range(1, n + 1)]
    scs = [abi.scenario(policy=abi.BFIO_GREEDY, workers=64, batch=64, horizon=20,
                        lookahead=abi.NOISY if noisy else abi.PERFECT, noise_sigma=2.0 if noisy else 0.0, seed=s,
                        input_id=i) for i, s in enumerate(range(1, n + 1))]
else:
    inputs = [host.sample_instance(s, rate=4000.0, duration=2.5, s_max=64, p=0.02) for s in range(1, n + 1)]
    scs = [abi.scenario(policy=abi.BFIO_GREEDY, workers=16, batch=64, seed=s, input_id=i)
           for i, s in enumerate(range(1, n + 1))]
scs = np.array(scs, abi.scenario_dtype)
ctx = host.Context(0)
db = host.DeviceBatch(ctx, scs, host.InputPool(inputs), emit_steps=True, emit_requests=True)
db.run()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
db.run()
e1.record()
torch.cuda.synchronize()
res = db.result_array()
K = res["steps_run"].astype(np.int64)
print(which, "traj", len(scs), "steps", int(K.sum()), "ms", e0.elapsed_time(e1),
      "us/step/traj", 1e3 * e0.elapsed_time(e1) / max(1, K.max()), "status", np.unique(res["status"]))
