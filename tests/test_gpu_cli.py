"""The reference CLI's subcommands (proj/tools/bfsim.cpp) on the GPU engine:
tools/_bin/bfsim_gpu against the same program over the unmodified reference
(tools/_bin/bfsim_cpu, -DBFSIM_CLI_CPU). Every output file (summary.txt,
steps.csv, compare.csv, sweep_h.csv, sweep_g.csv, iir.csv) must be
byte-identical, and the exit codes (0 ok, 1 usage/config error, 2 partial)
equal. Both binaries are built by __graft_entry__.build() where the reference
headers exist and travel to the GPU box."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "tools", "_bin")


def _run(which, args, out):
    exe = os.path.join(BIN, which)
    if not os.path.exists(exe):
        pytest.skip("tools/_bin not built (needs the reference headers at build time)")
    r = subprocess.run([exe, *args, "--out", str(out)], capture_output=True, text=True, timeout=600)
    return r.returncode, r.stdout


def _both(tmp_path, name, args):
    g, c = tmp_path / f"{name}_gpu", tmp_path / f"{name}_cpu"
    rg, og = _run("bfsim_gpu", args, g)
    rc, oc = _run("bfsim_cpu", args, c)
    assert rg == rc, (rg, rc, og, oc)
    files = sorted(os.listdir(c)) if os.path.isdir(c) else []
    assert files == (sorted(os.listdir(g)) if os.path.isdir(g) else [])
    for f in files:
        a, b = open(g / f, "rb").read(), open(c / f, "rb").read()
        assert a == b, f"{name}: {f} differs"
    return rg, files


COMMON = ["--workers", "8", "--batch", "16", "--rate", "600", "--duration", "1.5", "--seed", "3"]


@pytest.mark.parametrize("name,args,code", [
    ("run_greedy", ["run", *COMMON, "--policy", "bfio-greedy", "--horizon", "4", "--emit-steps"], 0),
    ("run_fcfs", ["run", *COMMON, "--policy", "fcfs", "--emit-steps"], 0),
    ("run_partial", ["run", *COMMON, "--policy", "jsq", "--max-steps", "40"], 2),
    ("run_overloaded", ["run", "--mode", "overloaded", "--workers", "8", "--batch", "8", "--steps", "150",
                        "--warmup", "30", "--policy", "bfio-greedy", "--horizon", "3", "--seed", "5",
                        "--emit-steps"], 0),
    ("compare", ["compare", *COMMON, "--policies", "fcfs,jsq,bfio-greedy"], 0),
    ("sweep_h", ["sweep-h", *COMMON, "--policy", "bfio-greedy", "--h-list", "0,2,5"], 0),
    ("sweep_g", ["sweep-g", "--batch", "16", "--rate", "600", "--duration", "1.0", "--g-list", "4,8,12"], 0),
    ("sweep_g_ovl", ["sweep-g", "--mode", "overloaded", "--batch", "8", "--steps", "120", "--warmup", "20",
                     "--g-list", "4,8"], 0),
    ("iir", ["iir", "--b-list", "4,8", "--g-list", "4,8", "--trials", "3", "--steps", "150", "--warmup", "30"], 0),
    ("compare_one", ["compare", *COMMON, "--policies", "fcfs"], 1),
    ("bad_policy", ["run", *COMMON, "--policy", "round-robin"], 1),
])
def test_cli_matches_reference(tmp_path, name, args, code):
    rc, files = _both(tmp_path, name, args)
    assert rc == code
    if code != 1:
        assert files


def test_cli_trace_and_config(tmp_path):
    trace = tmp_path / "t.csv"
    trace.write_text("# a hand-written trace\narrival_time,prefill,decode\n0.0,3,5\n0.001,7,2\n0.0005,2,9\n"
                     "0.02,64,30\n0.05,1,1\n")
    rc, files = _both(tmp_path, "trace", ["run", "--trace", str(trace), "--workers", "2", "--batch", "2",
                                          "--policy", "bfio-greedy", "--horizon", "2", "--emit-steps"])
    assert rc == 0 and "steps.csv" in files
    cfg = tmp_path / "c.cfg"
    cfg.write_text("# config file (tools/bfsim.cpp:46-65)\nworkers = 6\nbatch=4\npolicy=jsq\nrate=300\n"
                   "duration=1\npower.gamma=0.5\n")
    rc, files = _both(tmp_path, "config", ["run", "--config", str(cfg), "--workers", "5"])
    assert rc == 0
    assert "workers=5" in open(tmp_path / "config_gpu" / "summary.txt").read()
    for exe in ("bfsim_gpu", "bfsim_cpu"):
        r = subprocess.run([os.path.join(BIN, exe), "validate-trace", str(trace)], capture_output=True, text=True)
        assert r.returncode == 0 and r.stdout == "trace ok: 5 requests\n"
