"""Fold ncu traffic windows (scripts/measure_traffic.sh CSVs) into profiles/traffic_r02.json:
per-launch dram read+write averaged over the window, keyed task+N_envs_precision."""
import csv
import json
import os
import sys

out_path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "traffic_r02.json")
db = json.load(open(out_path)) if os.path.exists(out_path) else {}
for path, key, algo in zip(sys.argv[1::3], sys.argv[2::3], sys.argv[3::3]):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ki, kn, kv, ku = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    kid = hdr.index("ID")
    per = {}
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "ns": 1e-9, "usecond": 1e-6,
             "us": 1e-6, "msecond": 1e-3, "ms": 1e-3}
    for r in rows[1:]:
        per.setdefault(r[kid], {"kernel": r[ki]})[r[kn]] = float(r[kv].replace(",", "")) * scale.get(r[ku], 1)
    launches = list(per.values())
    rd = sum(x["dram__bytes_read.sum"] for x in launches) / len(launches)
    wr = sum(x["dram__bytes_write.sum"] for x in launches) / len(launches)
    t = sum(x["gpu__time_duration.sum"] for x in launches) / len(launches)
    db[key] = {"bytes_per_launch": rd + wr, "read_per_launch": rd, "write_per_launch": wr,
               "launches": len(launches), "kernel": launches[0]["kernel"][:80], "avg_launch_s_under_ncu": t,
               "algorithmic_bytes_per_launch": float(algo), "traffic_over_algorithmic": (rd + wr) / float(algo),
               "source": os.path.basename(path),
               "how": "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum --cache-control none over 12 "
                      "consecutive step launches of the timed bench loop (L2 flushed by a 512 MiB read between)"}
json.dump(db, open(out_path, "w"), indent=1)
print(json.dumps(db, indent=1))
