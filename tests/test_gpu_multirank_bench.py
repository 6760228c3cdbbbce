"""The bench's multi-rank path (torchrun, one process per GPU) on one B200:
two ranks share the device and talk over gloo (BFSIM_DIST_BACKEND=gloo; the
NCCL path needs one GPU per rank). The gathered per-scenario result rows must
equal a single-rank run of the same scenarios byte for byte:

* C2, weak scaling: rank r runs seeds r*S+1 .. (r+1)*S, so 2 ranks x S seeds
  = 1 rank x 2S seeds.
* C5, strong scaling: the fixed scenario grid is split across the ranks
  (parallel.shard_range), so 2 ranks and 1 rank run the identical grid.

Timing fields differ run to run; the result rows (MetricsReport, exact sums,
status, step counts) may not."""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

from paper_2601_17855_b200 import abi

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
COMPARE = ("status", "steps_run", "records", "completed", "admitted", "imb_total_i", "total_workload_i",
           "tokens_i", "clock", "elapsed", "avg_imbalance", "throughput", "imb_total", "total_workload",
           "eta_sum")


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _bench(tmp_path, name, args, nproc):
    out = str(tmp_path / f"{name}.npy")
    base = [os.path.join(ROOT, "bench.py"), "--steps", "1", "--warmup", "3", "--no-cpu-baseline", "--no-groups",
            "--dump-results", out, *args]
    env = dict(os.environ, BFSIM_DIST_BACKEND="gloo")
    if nproc == 1:
        cmd = [sys.executable, *base]
    else:
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
               "--master-addr", "127.0.0.1", "--master-port", str(_port()), *base, "--gpus", str(nproc)]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads([l for l in r.stdout.splitlines() if l.startswith("{")][-1])
    return line, np.load(out)


def _same(a, b):
    assert a.shape == b.shape
    for k in COMPARE:
        np.testing.assert_array_equal(a[k], b[k], err_msg=k)
    for k in ("energy", "tpot"):  # summation order is fixed per trajectory: equal too
        np.testing.assert_array_equal(a[k], b[k], err_msg=k)


def test_two_ranks_weak_c2(tmp_path):
    l2, r2 = _bench(tmp_path, "c2_two", ["--config", "c2", "--seeds", "4"], 2)
    l1, r1 = _bench(tmp_path, "c2_one", ["--config", "c2", "--seeds", "8"], 1)
    assert l2["n_gpus"] == 2 and l2["scaling"] == "weak"
    assert r2.shape[0] == 16 and (r2["status"] == abi.OK).all()
    _same(r2, r1)
    assert l2["imbalance_check"] == l1["imbalance_check"]


def test_two_ranks_strong_c5(tmp_path):
    l2, r2 = _bench(tmp_path, "c5_two", ["--config", "c5", "--scenarios", "8"], 2)
    l1, r1 = _bench(tmp_path, "c5_one", ["--config", "c5", "--scenarios", "8"], 1)
    assert l2["scaling"] == "strong"
    _same(r2, r1)
