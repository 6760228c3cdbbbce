"""Repro: several wide trajectories in one group (Poisson and overloaded), vs the oracle."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2601_17855_b200 import abi, host
from oracle.oracle import OracleLib

orc = OracleLib()
ctx = host.Context(0)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 8
G = int(sys.argv[2]) if len(sys.argv) > 2 else 300
trs = [host.sample_instance(7 + i, rate=G * 16 * 1.5, duration=0.5, s_max=64, p=0.05) for i in range(n)]
scs = [abi.scenario(policy=abi.BFIO_GREEDY, workers=G, batch=16, horizon=3, input_id=i) for i in range(n)]
br = ctx.run_batch(np.array(scs, abi.scenario_dtype), host.InputPool(trs), emit_steps=True, emit_requests=True)
bad = 0
for i in range(n):
    rc, res, st, rq = orc.run_poisson(br.scen[i], trs[i])
    bad += not np.array_equal(br.steps(i)["loads"], st.loads)
print("poisson ok, mismatches:", bad)
