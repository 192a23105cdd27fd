"""Summarise an ncu report: key metrics, stall reasons, source hot spots.
Usage: python scripts/ncu_summary.py gpurun_out/prof_X.ncu-rep [top_lines]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25


def run(*args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


rows = list(csv.reader(io.StringIO(run("--page", "raw", "--csv"))))
d = dict(zip(rows[0], rows[2] if len(rows) > 2 else rows[1]))
keys = ["gpu__time_duration.sum", "launch__registers_per_thread", "launch__block_size", "launch__grid_size",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "smsp__thread_inst_executed_per_inst_executed.ratio",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "launch__occupancy_limit_registers",
        "launch__occupancy_limit_shared_mem", "sm__maximum_warps_per_active_cycle_pct",
        "launch__shared_mem_per_block_dynamic"]
for k in keys:
    if k in d:
        print(f"{k:70s} {d[k]}")
st = {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): v for k, v in d.items()
      if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")}
tot = sum(float(v.replace(",", "")) for v in st.values() if v.replace(",", "").replace(".", "").isdigit())
print("stall samples:", ", ".join(f"{k}={float(v.replace(',', ''))/tot*100:.1f}%" for k, v in
                                   sorted(st.items(), key=lambda kv: -float(kv[1].replace(',', '')))[:8]))
src = list(csv.reader(io.StringIO(run("--page", "source", "--csv", "--print-source", "cuda,sass"))))
f = None
agg = []
for r in src:
    if len(r) >= 2 and r[0] == "File Path":
        f = r[1].split("/")[-1]
        continue
    if len(r) > 7 and r[0].isdigit():
        try:
            agg.append((int(r[4]), int(r[7]), f, int(r[0]), r[1].strip()[:80]))
        except ValueError:
            pass
ts = sum(a[0] for a in agg) or 1
ti = sum(a[1] for a in agg) or 1
print(f"samples {ts}, warp insts {ti}")
for a in sorted(agg, reverse=True)[:top]:
    print(f"{a[0]/ts*100:5.1f}% {a[1]/ti*100:5.1f}%i {a[2]}:{a[3]} {a[4]}")
