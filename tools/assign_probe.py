"""One bfsim_assign_batch launch for an ncu capture (scratch probe; not the
bench): 20,000 bfio-greedy calls (G=32, 64 waiting, H=16) and 2,000
bfio-exact calls (acceptance C01 shapes), CUDA-event timed.

    python tools/assign_probe.py [greedy|exact]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

from paper_2601_17855_b200 import abi, host

which = sys.argv[1] if len(sys.argv) > 1 else "greedy"
rng = np.random.default_rng(5)
calls = []
if which == "greedy":
    for _ in range(20000):
        G, n, H = 32, 64, 16
        calls.append((abi.BFIO_GREEDY, rng.integers(1, 64, (n, H + 1)).astype(np.float64),
                      rng.integers(0, 4, G).astype(np.int32), rng.integers(0, 60, G).astype(np.int32),
                      rng.integers(0, 4000, (G, H + 1)).astype(np.float64)))
else:
    for _ in range(2000):
        G, n, H = 3, 6, 2
        calls.append((abi.BFIO_EXACT, rng.integers(1, 10, (n, H + 1)).astype(np.float64),
                      rng.integers(0, 3, G).astype(np.int32), rng.integers(0, 3, G).astype(np.int32),
                      rng.integers(0, 20, (G, H + 1)).astype(np.float64)))
ctx = host.Context(0)
host.assign_batch(ctx, calls)
t = time.perf_counter()
out = host.assign_batch(ctx, calls)
print(which, len(calls), "calls", "%.2f ms host-timed" % (1e3 * (time.perf_counter() - t)),
      "statuses", sorted(set(int(o[2]) for o in out)))
