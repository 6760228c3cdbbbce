"""Per-CUDA-source-line L2 sector traffic (global + local) of an ncu capture:
python profiles/l2lines.py rep.ncu-rep [top]. Used to find where a kernel's
DRAM traffic comes from (L2 sectors are the upper bound of its DRAM bytes)."""
import csv
import re
import subprocess
import sys
from collections import defaultdict


def num(v):
    m = re.match(r"[0-9.eE+]+", v.strip())
    return float(m.group(0)) if m else 0.0


def main():
    rep = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout.splitlines()
    hdr, fname, cur = None, None, None
    glob, loc, src, ops = defaultdict(float), defaultdict(float), {}, defaultdict(set)
    for r in csv.reader(out):
        if not r:
            continue
        if r[0] in ("File Path", "File Name"):
            fname = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            hdr = {h: i for i, h in enumerate(r)}
            continue
        if hdr is None or len(r) < len(hdr):
            continue
        if r[0].strip():
            cur = (fname, int(r[0]))
            src[cur] = r[1].strip()[:100]
        if cur is None:
            continue
        g = r[hdr["L2 Theoretical Sectors Global"]].strip()
        l = r[hdr["L2 Theoretical Sectors Local"]].strip()
        glob[cur] += num(g)
        loc[cur] += num(l)
        op = r[hdr["Access Operation"]].strip()
        if op:
            ops[cur].add(op)
    tot = sum(glob.values()) + sum(loc.values())
    print(f"total L2 sectors {tot:.4g} ({tot * 32 / 1e9:.2f} GB)")
    keys = sorted(set(glob) | set(loc), key=lambda k: -(glob[k] + loc[k]))[:top]
    for k in keys:
        s = glob[k] + loc[k]
        print(f"{100 * s / tot:5.1f}%  {s * 32 / 1e9:7.2f} GB  local {loc[k] * 32 / 1e9:6.2f}  {k[0]}:{k[1]}  "
              f"{','.join(sorted(ops[k]))}  {src.get(k, '')}")


if __name__ == "__main__":
    main()
