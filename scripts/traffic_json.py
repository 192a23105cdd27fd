"""Fold ncu traffic windows (scripts/measure_traffic.sh CSVs, every kernel of the timed loop) into
profiles/traffic_r02.json: per step launch, dram read + write of the step kernel plus the
dram writes of the flush kernel that follows it (the write-back of the step's dirty L2 lines),
averaged over the window, keyed task+N_envs_precision."""
import csv
import json
import os
import sys

out_path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "traffic_r02.json")
db = json.load(open(out_path)) if os.path.exists(out_path) else {}
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "ns": 1e-9, "usecond": 1e-6,
         "us": 1e-6, "msecond": 1e-3, "ms": 1e-3}
for path, key, algo in zip(sys.argv[1::3], sys.argv[2::3], sys.argv[3::3]):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ki, kn, kv, ku = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    kid = hdr.index("ID")
    per = {}
    for r in rows[1:]:
        per.setdefault(int(r[kid]), {"kernel": r[ki]})[r[kn]] = float(r[kv].replace(",", "")) * scale.get(r[ku], 1)
    seq = [per[i] for i in sorted(per)]
    steps = []
    for i, k in enumerate(seq):
        if "step_kernel" not in k["kernel"]:
            continue
        nxt = seq[i + 1] if i + 1 < len(seq) else None
        wb = nxt["dram__bytes_write.sum"] if nxt is not None and "step_kernel" not in nxt["kernel"] else None
        if wb is None:
            continue
        steps.append((k["dram__bytes_read.sum"], k["dram__bytes_write.sum"], wb, k["gpu__time_duration.sum"]))
    n = len(steps)
    rd = sum(s[0] for s in steps) / n
    wr = sum(s[1] for s in steps) / n
    wb = sum(s[2] for s in steps) / n
    t = sum(s[3] for s in steps) / n
    db[key] = {"bytes_per_launch": rd + wr + wb, "read_per_launch": rd, "write_in_kernel_per_launch": wr,
               "writeback_in_next_flush_per_launch": wb, "launches": n,
               "kernel": next(k["kernel"] for k in seq if "step_kernel" in k["kernel"])[:80],
               "avg_launch_s_under_ncu": t, "algorithmic_bytes_per_launch": float(algo),
               "traffic_over_algorithmic": (rd + wr + wb) / float(algo), "source": os.path.basename(path),
               "how": "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum --cache-control none over every "
                      "kernel of consecutive timed-loop iterations: step reads + writes + the write-back of its "
                      "dirty L2 lines during the following 512 MiB-read flush"}
json.dump(db, open(out_path, "w"), indent=1)
print(json.dumps(db, indent=1))
