#!/bin/bash
# Iteration check (through gpurun): GPU suite, C5 bench, launch lists of C5 and C2, optional A/B
# variants (built here from -D knobs: VARIANTS="name:-DKNOB=V name2:-DK=V").
cd "$(dirname "$0")/.."
O=gpurun_out/iter; mkdir -p $O
python -m paper_1910_00935_b200.build > /dev/null
if [ -z "$NO_TESTS" ]; then
  export MPM_PARITY_RECORD=$O/parity_record.jsonl; rm -f $MPM_PARITY_RECORD
  timeout 1500 python -m pytest tests -m gpu -q -x ${PYTEST_ARGS} > $O/pytest_gpu.txt 2>&1; echo "pytest exit $?" >> $O/pytest_gpu.txt
  tail -4 $O/pytest_gpu.txt
fi
timeout 600 python bench.py --no-cpu-baseline ${BENCH_ARGS} > $O/bench.json 2> $O/bench.err
python - <<'PY'
import json
d = json.load(open("gpurun_out/iter/bench.json")); r = d["roofline"]
print("C5 value %.4g ms/step %.1f e2e %.4g | dominant %s %.3f step_frac %.3f" % (d["value"], d["ms_per_step"], d["e2e"]["value"], r["kernel"], r["frac"], r["step_frac"]))
print("kernel ms per iteration:", r["kernel_ms"])
PY
timeout 300 python bench.py --no-cpu-baseline --config c2 > $O/bench_c2.json 2> $O/bench_c2.err
python -c "import json; d=json.load(open('gpurun_out/iter/bench_c2.json')); print('C2 value %.4g ms/iter %.2f' % (d['value'], d['ms_per_step']))"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c5.csv python tools/profile_driver.py --steps 16 --k 2 > /dev/null 2>&1
python tools/launch_summary.py $O/launches_c5.csv 2>/dev/null | head -20
for v in $VARIANTS; do
  name=${v%%:*}; flags=${v#*:}
  python tools/build_variant.py $name ${flags//,/ } > /dev/null 2>&1
  bash tools/ab.sh $name.so
done
