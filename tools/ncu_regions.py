"""Summarise an ncu report: key pipe/stall metrics and stall samples per source file/line.

usage: python tools/ncu_regions.py REPORT.ncu-rep [top_lines]
"""
import collections
import csv
import io
import subprocess
import sys


def ncu(rep, *args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


def main():
    rep = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 8
    rows = list(csv.reader(io.StringIO(ncu(rep, "--page", "raw", "--csv"))))
    h, v = rows[0], rows[2]
    keys = ["gpu__time_duration.sum", "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
            "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__issue_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
            "dram__bytes_read.sum", "dram__bytes_write.sum"]
    for k in keys:
        if k in h:
            print(f"{k:70s} {v[h.index(k)]}")
    st = [(n, v[i]) for i, n in enumerate(h) if n.startswith("smsp__average_warps_issue_stalled_")
          and n.endswith("_per_issue_active.ratio")]
    st.sort(key=lambda x: -float(x[1] or 0))
    print("stalls/issue:", ", ".join(f"{n[34:-23]} {float(x):.2f}" for n, x in st[:9]))
    rows = list(csv.reader(io.StringIO(ncu(rep, "--page", "source", "--csv", "--print-source", "cuda,sass"))))
    f = None
    tot = collections.Counter()
    by = collections.defaultdict(collections.Counter)
    for r in rows:
        if r and r[0] == "File Path":
            f = r[1].split("/")[-1]
            continue
        if len(r) < 6:
            continue
        try:
            ln, s = int(r[0]), int(r[4] or 0)
        except ValueError:
            continue
        tot[f] += s
        by[f][(ln, r[1].strip()[:80])] += s
    T = sum(tot.values()) or 1
    for f, s in tot.most_common():
        print(f"== {f} {s / T:.3f}")
        for (ln, src), c in by[f].most_common(top):
            if c / T >= 0.004:
                print(f"   {c / T:.3f} L{ln}: {src}")


if __name__ == "__main__":
    main()
