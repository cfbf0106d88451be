"""profiles/r02_ncu_full_summary.txt and profiles/traffic.json from the raw-page CSVs that
tools/jobs/ncu_captures.sh brings back (gpurun_out/ncu/*.raw.csv).  Usage: python tools/summarize_ncu_raw.py"""
import csv
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT / "tools"))
import summarize_ncu as s  # noqa: E402

HEADER = """Round-2 ncu --set full --clock-control none --import-source on captures (one B200) of the final
kernels (tools/jobs/ncu_captures.sh: reports stay on the box, `ncu -i REP --page raw --csv` comes
back; the values below are from those raw pages, tools/summarize_ncu_raw.py).

* r02_tc_window_cfg3: the bench's timed call — the resident tensor-core launch of km_lloyd(C0, 20)
  at cfg3 (2M x 25 x 16), i.e. passes 1..20 of the first-K trajectory (tools/profile_window.py).
* r02_tc_steady_cfg3: the resident launch of km_lloyd(C0, 400) at cfg3 (passes 1..400, mostly
  steady state; tools/profile_steady.py cfg3 400 50, ncu -s 1 -c 1 selects that launch).
* r02_tc_steady_k64: the same for 2M x 25 x 64 (cfg5's K), passes 1..300.
* r02_sums_cfg3: the cluster-sums kernel of the first pass at cfg3 (2M rows).
* r02_full_first (earlier kernel, not re-captured): KM_FULL_FIRST_PASS=1 at cfg3, the fused full
  first pass.  Warp-stall sampling: 21.8 % of all samples on the transform's wait for the raw-tile
  full barrier — the epilogue holds every raw slot until its Δ is done and its twelve warps adding
  2M rows are the bound (~200 us vs 49 us labels-only pass + 67 us cluster sums), hence the split
  first pass for n >= 500k.
"""
EXTRA = ["l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smsp__inst_executed.sum", "sm__cycles_elapsed.avg"]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}

parts, traffic = [HEADER], {}
for r in ["r02_tc_window_cfg3", "r02_tc_steady_cfg3", "r02_tc_steady_k64", "r02_sums_cfg3"]:
    rows = list(csv.reader(open(ROOT / "gpurun_out" / "ncu" / f"{r}.raw.csv")))
    hdr, units, vals = rows[0], rows[1], rows[2]
    out = [f"===== {r}", f"Kernel Name  {vals[hdr.index('Kernel Name')]}"]
    for m in s.METRICS + EXTRA:
        if m in hdr:
            i = hdr.index(m)
            out.append(f"{m:70s} {vals[i]} {units[i]}")
    parts.append("\n".join(out) + "\n")

    def b(name):
        i = hdr.index(name)
        return float(vals[i].replace(",", "")) * SCALE[units[i]]

    traffic[r] = b("dram__bytes_read.sum") + b("dram__bytes_write.sum")
(ROOT / "profiles" / "r02_ncu_full_summary.txt").write_text("\n".join(parts))
t = {"cfg3": round(traffic["r02_tc_window_cfg3"] / 20, 1), "cfg5": round(traffic["r02_tc_steady_k64"] / 300 * 32, 1),
     "_unit": "dram bytes per Lloyd pass",
     "_source": "profiles/r02_ncu_full_summary.txt: cfg3 = the bench window's resident launch (20 passes), "
                "(dram__bytes_read.sum + dram__bytes_write.sum) / passes; cfg5 = the 2M x 25 x 64 resident launch "
                "(300 passes) per pass, scaled by 32 to 64M rows"}
(ROOT / "profiles" / "traffic.json").write_text(json.dumps(t, indent=1))
print(t)
