#!/bin/bash
# Quick kernel A/B on the GPU box: build each variant (NAME:-DKNOB=V,-DK2=V ... or NAME:git=REV)
# and print the bench's per-kernel ms per C5 iteration (profiling pass) plus the timed value.
# usage (through gpurun): VARIANTS="a: b:-DMPM_X=1 c:prebuilt" bash tools/ab_kernels.sh [bench args]
cd "$(dirname "$0")/.."
python -m paper_1910_00935_b200.build > /dev/null
for v in $VARIANTS; do
  name=${v%%:*}; flags=${v#*:}
  [ "$flags" == "prebuilt" ] && continue  # variants/NAME.so shipped with the snapshot
  python tools/build_variant.py $name ${flags//,/ } > /dev/null 2>&1 || { echo "$name build failed"; continue; }
done
for rep in 1 2; do
for v in $VARIANTS; do
  name=${v%%:*}
  MPM_B200_LIB="$PWD/variants/$name.so" timeout 400 python bench.py --no-cpu-baseline --steps 8 --warmup 3 "$@" > gpurun_out/ab_$name.json 2> gpurun_out/ab_$name.err
  python - "$name" <<'PY'
import json, sys
v = sys.argv[1]
try:
    d = json.load(open(f"gpurun_out/ab_{v}.json"))
except Exception as e:
    print(v, "failed", open(f"gpurun_out/ab_{v}.err").read()[-800:]); raise SystemExit
r = d["roofline"]; k = r["kernel_ms"]
g = lambda n: k.get(n, 0.0)  # noqa: E731
print("%-10s value %.4g ms/it %.1f | p2g %.1f g2p %.1f sc %.1f ga %.1f p2gg %.1f canon %.1f gop %.1f gopg %.1f bin %.1f" % (
    v, d["value"], d["ms_per_step"], g("p2g"), g("g2p"), g("g2p_grad"), g("g2p_grad_gather"), g("p2g_grad"),
    g("canon"), g("grid_op"), g("grid_op_grad"), g("bin")))
PY
done
done
