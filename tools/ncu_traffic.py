"""Per-kernel DRAM traffic (dram__bytes_read.sum + dram__bytes_write.sum per launch, median over
the captured launches) from ncu --set full reports -> profiles/ncu_traffic.json (bench.py's
roofline.traffic).  usage: python tools/ncu_traffic.py REP [REP ...] [--out OUT]"""
import csv
import json
import re
import statistics
import subprocess
import sys

args = sys.argv[1:]
out = "profiles/ncu_traffic.json"
if "--out" in args:
    out = args[args.index("--out") + 1]
    args = args[:args.index("--out")] + args[args.index("--out") + 2:]
reps = args
per = {}
for rep in reps:
  raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
  rows = list(csv.reader(raw.splitlines()))
  h = rows[0]
  col = {n: i for i, n in enumerate(h)}
  units = rows[1]
  for r in rows[2:]:
    name = re.search(r"k_(\w+?)(<|\()", r[col["Kernel Name"]]).group(1)
    sc = lambda n: 1e6 if "Mbyte" in units[col[n]] else (1e3 if "Kbyte" in units[col[n]] else (1e9 if "Gbyte" in units[col[n]] else 1.0))  # noqa: E731
    rd = float(r[col["dram__bytes_read.sum"]]) * sc("dram__bytes_read.sum")
    wr = float(r[col["dram__bytes_write.sum"]]) * sc("dram__bytes_write.sum")
    us = float(r[col["gpu__time_duration.sum"]]) * (1e-3 if units[col["gpu__time_duration.sum"]] == "nsecond" else 1.0)
    per.setdefault(name, []).append((rd, wr, us))
res = {"_source": f"ncu --set full --clock-control none ({', '.join(reps)}); C5 size (1,061,208 particles, 128^3), "
                  "tools/profile_driver.py --steps 4 --k 2; dram__bytes_read.sum + dram__bytes_write.sum per "
                  "launch, median over the captured launches"}
for k, v in per.items():
    med = sorted(v, key=lambda t: t[0] + t[1])[len(v) // 2]
    res[k] = {"dram_bytes_per_launch": int(med[0] + med[1]), "read_MB": round(med[0] / 1e6, 1),
              "write_MB": round(med[1] / 1e6, 1), "us": round(med[2], 1), "launches_captured": len(v)}
json.dump(res, open(out, "w"), indent=1)
print(json.dumps(res, indent=1))
