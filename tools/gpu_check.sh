#!/bin/bash
# GPU-box check: parity tests + default bench (no cpu baseline); prints a one-line summary.
# usage (through gpurun): bash tools/gpu_check.sh [--no-tests] [bench args...]
cd "$(dirname "$0")/.."
if [ "$1" != "--no-tests" ]; then
  timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
else
  shift
fi
timeout 400 python bench.py --no-cpu-baseline "$@" > gpurun_out/bench.json 2> gpurun_out/bench.err
python - <<'PY'
import json
try:
    d = json.load(open("gpurun_out/bench.json"))
except Exception as e:
    print("bench failed", e); print(open("gpurun_out/bench.err").read()[-2000:]); raise SystemExit
r = d["roofline"]
print("value %.4g ms/step %.1f e2e %.4g | %s frac %.3f | %s" % (d["value"], d["ms_per_step"], d["e2e"]["value"],
      r["kernel"], r["frac"], r["kernel_ms"]))
PY
