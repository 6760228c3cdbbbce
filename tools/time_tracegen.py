"""Time the device generator on the C3 pass (1,000 traces, lambda = 8000/s x
12.5 s) against the host batcher (one trace, scaled). Prints one JSON line."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2601_17855_b200 import host  # noqa: E402

ctx = host.Context(0)
specs = [dict(seed=s, rate=8000.0, duration=12.5, s_max=64, p=0.02) for s in range(1000)]
host.DevicePool(ctx, specs[:8])  # warm-up (module load, allocator)
ts = []
for _ in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    pool = host.DevicePool(ctx, specs)
    torch.cuda.synchronize()
    ts.append(time.perf_counter() - t0)
n = int(pool.inputs["length"].sum())
t0 = time.perf_counter()
h = host.sample_instance(0, rate=8000.0, duration=12.5, s_max=64, p=0.02)
th = time.perf_counter() - t0
print(json.dumps({"device_s": min(ts), "records": n, "device_records_per_s": n / min(ts),
                  "host_1trace_s": th, "host_records_per_s_1thread": h.shape[0] / th}))
