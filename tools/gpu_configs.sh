# Other configs + the f2 optimisation loop on one GPU (through gpurun).
cd "$(dirname "$0")/.."; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3 > gpurun_out/opt_gpu.txt
cat gpurun_out/opt_gpu.txt
for c in c2 c2cl c3 c3cl c3liquid c4 c1a; do
  timeout 600 python bench.py --config $c --steps 5 --warmup 3 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
  python -c "
import json,sys; d=json.load(open('gpurun_out/bench_$c.json')); r=d['roofline']
print('$c', '%.4g'%d['value'], 'e2e %.4g'%d['e2e']['value'], 'ms/step %.2f'%d['ms_per_step'], r['kernel'], 'frac %.3f'%r['frac'], 'cpu %.3g'%(d['cpu_baseline'] or {}).get('value', 0))" || tail -3 gpurun_out/bench_$c.err
done
