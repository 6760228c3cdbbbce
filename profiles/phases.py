"""Group an ncu source-page capture of the step kernel by engine phase
(line ranges of the lambdas in engine_impl.cuh): python profiles/phases.py rep.ncu-rep"""
import re
import subprocess
import sys
from collections import defaultdict

sys.path.insert(0, __file__.rsplit("/", 1)[0])
from hotlines import main as _unused  # noqa: F401  (same CSV format)

SRC = __file__.rsplit("/", 2)[0] + "/paper_2601_17855_b200/csrc/engine_impl.cuh"
MARKS = [
    (r"^__device__ __forceinline__ uint64_t mt_temper", "noisy: producer warp (mt19937_64, polar)"),
    (r"^template <bool SM, class T>", "setup / other"),
    (r"^struct WideChain", "wide chain (G > 128)"),
    (r"^template <int MODE, int POL, int WPL, bool SMALLC, bool SM, bool NOISY, int HR, bool WIDE = false>", "setup / other"),
    (r"auto drain_tpot = ", "accounting (flush, TPOT)"),
    (r"auto reveal = ", "reveal"),
    (r"auto topup = ", "overloaded top-up"),
    (r"auto refresh_maxcount = ", "overloaded top-up"),
    (r"auto place = ", "place"),
    (r"auto gen_normals = ", "noisy: normals"),
    (r"auto waiting_ranks = ", "noisy: waiting ranks"),
    (r"auto noisy_views = ", "noisy: views"),
    (r"auto prefetch_fifo = ", "fifo admission"),
    (r"auto admit_greedy = ", "greedy: setup"),
    (r"    if \(phase1\) \{", "greedy: phase 1 (water filling)"),
    (r"    // Order the U admitted items", "greedy: ordering"),
    (r"    if \(H == 0\) \{", "greedy: phase 2 H=0"),
    (r"      // general H: lookahead views", "greedy: phase 2 H>0"),
    (r"  auto retire = ", "retire"),
    (r"  // --- step loop", "step loop (loads, dt, clock)"),
    (r"^template <int MODE, int POL, int WPL, bool SMALLC, bool SM, bool NOISY, int HR>\n__global__", "kernel"),
]


def ranges():
    lines = open(SRC).read().splitlines()
    marks = []
    for i, l in enumerate(lines, 1):
        for pat, name in MARKS:
            if re.search(pat.split("\n")[0], l):
                marks.append((i, name))
    marks.sort()
    return marks


def phase_of(marks, ln):
    cur = "setup / other"
    for i, name in marks:
        if ln >= i:
            cur = name
    return cur


def main():
    rep = sys.argv[1]
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    import csv
    rows = list(csv.reader(out.splitlines()))
    marks = ranges()
    tot = defaultdict(float)
    ins = defaultdict(float)
    hdr = None
    cur = None
    fname = None
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            hdr = r
            si = hdr.index("Warp Stall Sampling (All Samples)")
            ei = hdr.index("Instructions Executed")
            continue
        if hdr is None or len(r) < len(hdr):
            continue
        if r[0].strip():
            cur = (fname, int(r[0]))
        if cur is None:
            continue
        try:
            s = float(r[si] or 0)
            e = float(r[ei] or 0)
        except ValueError:
            continue
        key = phase_of(marks, cur[1]) if cur[0] == "engine_impl.cuh" else "intrinsics (" + cur[0] + ")"
        tot[key] += s
        ins[key] += e
    t = sum(tot.values()) or 1
    ti = sum(ins.values()) or 1
    print("stall-samples  warp-instructions  phase")
    for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
        print(f"{100 * v / t:12.1f}%  {100 * ins[k] / ti:16.1f}%  {k}")
    print(f"total warp instructions: {ti:.4g}")


if __name__ == "__main__":
    main()
