"""C3 at full scale (1000 seeds x 100k requests), one launch, metrics only (ncu target)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2601_17855_b200 import abi, host

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
dur = float(sys.argv[2]) if len(sys.argv) > 2 else 12.5
trs = [host.sample_instance(s, rate=8000.0, duration=dur, s_max=64, p=0.02) for s in range(1, n + 1)]
scs = np.array([abi.scenario(policy=abi.BFIO_GREEDY, workers=64, batch=64, horizon=20, lookahead=abi.NOISY,
                             noise_sigma=2.0, seed=s, input_id=i) for i, s in enumerate(range(1, n + 1))],
               abi.scenario_dtype)
ctx = host.Context(0)
db = host.DeviceBatch(ctx, scs, host.InputPool(trs), emit_steps=False, emit_requests=False)
db.run()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
db.run()
e1.record()
torch.cuda.synchronize()
res = db.result_array()
print("traj", n, "steps", int(res["steps_run"].sum()), "ms", e0.elapsed_time(e1))
