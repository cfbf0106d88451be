"""Summaries committed under profiles/ from a gpurun_out/ ncu launch list (--csv --log-file) and a
full capture (.ncu-rep).  Usage: python tools/summarize_ncu.py launches.csv [full.ncu-rep]"""
import csv
import subprocess
import sys
from collections import defaultdict


def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    tot, cnt = defaultdict(float), defaultdict(int)
    for r in rows[1:]:
        if r[mi] != "gpu__time_duration.sum":
            continue
        v = float(r[vi].replace(",", ""))
        unit = r[hdr.index("Metric Unit")]
        us = v / 1e3 if unit in ("ns", "nsecond") else v * 1e3 if unit in ("ms", "msecond") else v
        tot[r[ki]] += us
        cnt[r[ki]] += 1
    s = sum(tot.values())
    print("# count  total_us  share  kernel")
    for kname in sorted(tot, key=tot.get, reverse=True):
        print(f"{cnt[kname]:5d} {tot[kname]:10.1f} {100*tot[kname]/s:5.1f}%  {kname[:100]}")


METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "launch__grid_size",
           "launch__block_size", "launch__registers_per_thread",
           "smsp__issue_active.avg.pct_of_peak_sustained_active",
           "sm__throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__throughput.avg.pct_of_peak_sustained_active",
           "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active",
           "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
           "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
           "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
           "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
           "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"]


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units, vals = rows[0], rows[1], rows[2]
    print(f"Kernel Name  {vals[hdr.index('Kernel Name')]}")
    for mname in METRICS:
        if mname in hdr:
            i = hdr.index(mname)
            print(f"{mname:70s} {vals[i]} {units[i]}")


if __name__ == "__main__":
    launches(sys.argv[1])
    if len(sys.argv) > 2:
        full(sys.argv[2])
