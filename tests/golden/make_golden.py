"""Generate the golden fixtures from the UNMODIFIED reference build
(oracle/_ref/libbfsim_ref.so, compiled from /root/reference by oracle/Makefile).

    python tests/golden/make_golden.py

Writes tests/golden/c1_reference.npz (BASELINE C1: the seed-1 trace and the
reference's per-step loads, clocks and MetricsReport for fcfs, bfio-greedy H=0
and H=20), tests/golden/iir_c06.npy (acceptance C06's estimate_iir grid) and
tests/golden/assign_steps.json (assign() on random steps, all four policies,
with bfio-exact's cost). The fixtures pin parity without the reference
present (the GPU box has no /root/reference)."""
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import numpy as np  # noqa: E402

from oracle.oracle import RefLib  # noqa: E402
from paper_2601_17855_b200 import abi  # noqa: E402


def main():
    ref = RefLib()
    tr = ref.sample_instance(s_max=64, p=0.02, rate=2000.0, duration=1.0, seed=1)
    out = {"trace": tr}
    for name, pol, H in (("fcfs", abi.FCFS, 0), ("greedy_h0", abi.BFIO_GREEDY, 0), ("greedy_h20", abi.BFIO_GREEDY, 20)):
        rc, err, (st, rq, m, done) = ref.run_poisson(abi.scenario(policy=pol, workers=8, batch=64, horizon=H), tr)
        assert rc == 0, err
        out[f"{name}_loads"] = st.loads
        out[f"{name}_clock"] = st.clock_start
        out[f"{name}_metrics"] = np.array([m[k] for k in abi.METRIC_FIELDS])
    np.savez_compressed(os.path.join(HERE, "c1_reference.npz"), **out)
    np.save(os.path.join(HERE, "iir_c06.npy"), ref.estimate_iir([8, 32], [4, 16], 20, 1500, 300, 606))
    rng = np.random.default_rng(424242)
    steps = []
    for t in range(400):
        pol = (abi.FCFS, abi.JSQ, abi.BFIO_EXACT, abi.BFIO_GREEDY)[t % 4]
        H = int(rng.integers(0, 3))
        G = int(rng.integers(1, 4))
        n = int(rng.integers(0, 7))
        caps = rng.integers(0, 4, G).astype(np.int32)
        cnt = rng.integers(0, 3, G).astype(np.int32)
        fut = rng.integers(0, 20, (G, H + 1)).astype(np.float64)
        pv = rng.integers(0, 10, (n, H + 1)).astype(np.float64)
        rc, pairs, cost = ref.assign(pol, pv, caps, cnt, fut, H)
        assert rc == 0
        steps.append(dict(policy=pol, H=H, previews=pv.tolist(), caps=caps.tolist(), counts=cnt.tolist(),
                          futures=fut.tolist(), pairs=pairs, cost=cost))
    with open(os.path.join(HERE, "assign_steps.json"), "w") as f:
        json.dump(steps, f)
    print("golden fixtures written")


if __name__ == "__main__":
    main()
