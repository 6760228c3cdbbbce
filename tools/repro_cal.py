"""Repro: the calendar test batch (several kernel groups at once) under compute-sanitizer."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2601_17855_b200 import abi, host

ctx = host.Context(0)
sel = [int(x) for x in sys.argv[1].split(",")] if len(sys.argv) > 1 else None
cases = ((128, 40, abi.FCFS, 0, abi.PERFECT), (100, 50, abi.JSQ, 0, abi.PERFECT),
         (96, 48, abi.BFIO_GREEDY, 0, abi.PERFECT), (64, 80, abi.BFIO_GREEDY, 6, abi.PERFECT),
         (70, 64, abi.BFIO_GREEDY, 20, abi.TRUNCATED), (300, 16, abi.BFIO_GREEDY, 3, abi.PERFECT),
         (64, 72, abi.BFIO_GREEDY, 20, abi.NOISY), (520, 9, abi.BFIO_GREEDY, 0, abi.PERFECT))
scs, trs = [], []
for t, (G, B, pol, H, la) in enumerate(cases):
    if sel is not None and t not in sel:
        continue
    s = abi.scenario(policy=pol, workers=G, batch=B, horizon=H, lookahead=la,
                     noise_sigma=2.0 if la == abi.NOISY else 0.0, seed=t + 1)
    s["input_id"] = len(trs)
    scs.append(s)
    trs.append(host.sample_instance(100 + t, rate=G * B * 1.5, duration=0.8, s_max=64, p=0.05))
br = ctx.run_batch(np.array(scs, abi.scenario_dtype), host.InputPool(trs), emit_steps=True, emit_requests=True)
print("ok", br.res["steps_run"])
