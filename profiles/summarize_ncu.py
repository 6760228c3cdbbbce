"""Summarise ncu reports captured under gpurun into profiles/ (run here, no GPU).

    python profiles/summarize_ncu.py gpurun_out/prof_greedy_r01.ncu-rep [...]
"""
import csv
import json
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "launch__shared_mem_per_block_dynamic", "smsp__inst_executed.sum",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__cycles_active.avg", "sm__cycles_elapsed.avg", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_bytes.sum", "l1tex__t_bytes.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units, vals = rows[0], rows[1], rows[2]
    d = {h: (v, u) for h, u, v in zip(hdr, units, vals)}
    return d


def to_bytes(v, u):
    f = float(v)
    return f * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)


def hot_lines(rep, n=15):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr = rows[2]
    si = hdr.index("Warp Stall Sampling (All Samples)")
    lines = [r for r in rows[3:] if len(r) > si and r[2] == "-"]
    tot = sum(float(r[si] or 0) for r in lines) or 1.0
    lines.sort(key=lambda r: -float(r[si] or 0))
    return [(round(100 * float(r[si]) / tot, 1), int(r[0]), r[1].strip()[:90]) for r in lines[:n]]


def main():
    summary = {}
    for rep in sys.argv[1:]:
        d = raw(rep)
        name = d["Kernel Name"][0]
        s = {k: d[k][0] + " " + d[k][1] for k in KEYS if k in d}
        rd = to_bytes(*d["dram__bytes_read.sum"])
        wr = to_bytes(*d["dram__bytes_write.sum"])
        s["dram_bytes_per_launch"] = rd + wr
        s["hot_lines"] = hot_lines(rep)
        summary[rep.split("/")[-1]] = {"kernel": name, **s}
    print(json.dumps(summary, indent=1))


if __name__ == "__main__":
    main()
