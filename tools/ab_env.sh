#!/bin/bash
# A/B with per-run environment: bash tools/ab_env.sh "ENV=.. LIB.so" "ENV2=.. LIB2.so" -- bench args
cd "$(dirname "$0")/.."; mkdir -p gpurun_out
runs=()
while [ $# -gt 0 ] && [ "$1" != "--" ]; do runs+=("$1"); shift; done
[ "$1" == "--" ] && shift
i=0
for r in "${runs[@]}"; do
  i=$((i+1))
  lib=${r##* }; envs=${r% *}; [ "$envs" == "$r" ] && envs=""
  env $envs MPM_B200_LIB="$PWD/variants/$lib" timeout 400 python bench.py --no-cpu-baseline "$@" > gpurun_out/abe_$i.json 2> gpurun_out/abe_$i.err
  python - "$r" "$i" <<'PY'
import json, sys
r, i = sys.argv[1], sys.argv[2]
try:
    d = json.load(open(f"gpurun_out/abe_{i}.json"))
except Exception as e:
    print(r, "failed", open(f"gpurun_out/abe_{i}.err").read()[-800:]); raise SystemExit
print("%-32s value %.4g ms/step %.1f" % (r, d["value"], d["ms_per_step"]))
PY
done
