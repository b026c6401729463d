#!/bin/bash
# A/B kernel experiments on the GPU box: bench each library build under variants/.
# usage (through gpurun): bash tools/ab.sh NAME.so [NAME2.so ...] [-- bench args]
cd "$(dirname "$0")/.."
libs=()
while [ $# -gt 0 ] && [ "$1" != "--" ]; do libs+=("$1"); shift; done
[ "$1" == "--" ] && shift
for v in "${libs[@]}"; do
  MPM_B200_LIB="$PWD/variants/$v" timeout 400 python bench.py --no-cpu-baseline "$@" > gpurun_out/ab_$v.json 2> gpurun_out/ab_$v.err
  python - "$v" <<'PY'
import json, sys
v = sys.argv[1]
try:
    d = json.load(open(f"gpurun_out/ab_{v}.json"))
except Exception as e:
    print(v, "failed", open(f"gpurun_out/ab_{v}.err").read()[-1500:]); raise SystemExit
r = d["roofline"]
print("%-20s value %.4g ms/step %.1f | %s" % (v, d["value"], d["ms_per_step"], r["kernel_ms"]))
PY
done
