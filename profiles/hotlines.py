"""Aggregate an ncu source page (--page source --csv --print-source cuda,sass)
into per-CUDA-source-line warp-stall samples: python profiles/hotlines.py rep.ncu-rep [top]."""
import csv
import subprocess
import sys
from collections import defaultdict


def main():
    rep = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout.splitlines()
    rows = list(csv.reader(out))
    hdr = None
    line_samples = defaultdict(float)
    line_exec = defaultdict(float)
    src = {}
    cur_line = None
    fname = None
    stall_cols = {}
    stall_tot = defaultdict(lambda: defaultdict(float))
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
            stall_cols = {h: i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h}
            continue
        if hdr is None or len(r) < len(hdr):
            continue
        if r[0].strip():
            cur_line = (fname, int(r[0]))
            src[cur_line] = r[1].strip()[:90]
        if cur_line is None:
            continue
        try:
            s = float(r[si] or 0)
            e = float(r[ei] or 0)
        except ValueError:
            continue
        line_samples[cur_line] += s
        line_exec[cur_line] += e
        for h, i in stall_cols.items():
            try:
                stall_tot[cur_line][h] += float(r[i] or 0)
            except ValueError:
                pass
    tot = sum(line_samples.values()) or 1.0
    print(f"total samples {tot:.0f}")
    for ln, s in sorted(line_samples.items(), key=lambda kv: -kv[1])[:top]:
        st = sorted(stall_tot[ln].items(), key=lambda kv: -kv[1])[:3]
        sts = " ".join(f"{k[6:]}={v/s*100:.0f}%" for k, v in st if s)
        print(f"{s/tot*100:5.1f}% {ln[0]}:{ln[1]:<5} exec={line_exec[ln]:.3g} [{sts}] {src.get(ln, '')}")


if __name__ == "__main__":
    main()
