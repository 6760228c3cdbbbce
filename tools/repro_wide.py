"""Small wide-chain repro cases (G > 128 with a window), checked against the oracle."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2601_17855_b200 import abi, host
from oracle.oracle import OracleLib

orc = OracleLib()
ctx = host.Context(0)
cases = [(300, 16, 3), (513, 3, 3), (256, 20, 20), (129, 40, 5)]
for G, B, H in cases:
    tr = host.sample_instance(7, rate=G * B * 1.5, duration=0.5, s_max=64, p=0.05)
    sc = abi.scenario(policy=abi.BFIO_GREEDY, workers=G, batch=B, horizon=H, input_id=0)
    try:
        br = ctx.run_batch(np.array([sc], abi.scenario_dtype), host.InputPool([tr]), emit_steps=True, emit_requests=True)
    except Exception as e:
        print("FAIL", G, B, H, e)
        sys.exit(1)
    rc, res, st, rq = orc.run_poisson(br.scen[0], tr)
    ok = np.array_equal(br.steps(0)["loads"], st.loads)
    print(G, B, H, "loads equal:", ok, int(br.res[0]["steps_run"]), int(res["steps_run"]))
