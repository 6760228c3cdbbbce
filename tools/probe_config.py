"""Quick device timing of one BASELINE config shape (scratch probe, not the bench)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2601_17855_b200 import abi, host

def run(name, scs, traces, emit=False, reps=3):
    pool = host.InputPool(traces)
    ctx = host.Context(0)
    db = host.DeviceBatch(ctx, scs, pool, emit_steps=emit, emit_requests=emit)
    db.run(); torch.cuda.synchronize()
    res = db.result_array()
    K = res["steps_run"].astype(np.int64)
    ws = int((K * scs["workers"]).sum())
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); db.run(); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ms = min(ts)
    print(f"{name}: {len(scs)} traj, {int(K.sum())} steps, {ws} worker-steps, {ms:.2f} ms -> {ws/ms*1e3:.3e} ws/s; "
          f"status {np.unique(res['status'])} flags {np.unique(res['flags'])}", flush=True)
    ctx.close()
    return res

which = sys.argv[1] if len(sys.argv) > 1 else "c3"
nseeds = int(sys.argv[2]) if len(sys.argv) > 2 else 148
if which == "c3":
    t0 = time.time()
    trs = [host.sample_instance(s, rate=8000.0, duration=12.5, s_max=64, p=0.02) for s in range(1, nseeds + 1)]
    print("gen", time.time() - t0, "s", sum(t.shape[0] for t in trs), "requests", flush=True)
    for sigma, la in ((2.0, abi.NOISY), (0.0, abi.PERFECT)):
        scs = np.array([abi.scenario(policy=abi.BFIO_GREEDY, workers=64, batch=64, horizon=20, lookahead=la,
                                     noise_sigma=sigma, seed=s, input_id=i) for i, s in enumerate(range(1, nseeds + 1))],
                       abi.scenario_dtype)
        run(f"C3 greedy H20 la={la} sigma={sigma}", scs, trs)
elif which == "c4":
    for G in [int(x) for x in sys.argv[3].split(",")]:
        B, steps, warm = 64, 2000, 200
        n = int(G * B * (2 + (steps + warm) * 0.02 * 1.3)) + 4096
        sts = [host.sample_stream(s, n, s_max=64, p=0.02) for s in range(1, nseeds + 1)]
        for pol, H, drift in ((abi.FCFS, 0, 0.0), (abi.JSQ, 0, 0.0), (abi.BFIO_GREEDY, 0, 0.0), (abi.BFIO_GREEDY, 20, 1.0)):
            scs = np.array([abi.scenario(mode=abi.OVERLOADED, policy=pol, workers=G, batch=B, horizon=H, drift=drift,
                                         steps=steps, warmup=warm, seed=s, input_id=i)
                            for i, s in enumerate(range(1, nseeds + 1))], abi.scenario_dtype)
            run(f"C4 G={G} pol={pol} H={H}", scs, sts)
