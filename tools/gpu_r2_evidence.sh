#!/bin/bash
# SKIP_FULL=1: stop after the launch lists (no ncu --set full captures, no sanitizers).
# ONLY_FULL=1: only the ncu --set full captures and the sanitizers.
# Round-2 evidence run (through gpurun): full GPU suite with the parity record, benches (C5 with
# the bench's k and k = 32, every config), ncu launch list + --set full captures of the step
# kernels, compute-sanitizer logs.  Everything lands in gpurun_out/r2/.
cd "$(dirname "$0")/.."
O=gpurun_out/${EVID:-r2}; mkdir -p $O/configs
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total,driver_version --format=csv > $O/smi.txt
lscpu | grep -E "Model name|^CPU\(s\)" > $O/host.txt
python -m paper_1910_00935_b200.build > /dev/null
if [ -z "$ONLY_FULL" ]; then
export MPM_PARITY_RECORD=$O/parity_record.jsonl; rm -f $MPM_PARITY_RECORD
timeout 1500 python -m pytest tests -m gpu -q -s --durations=30 > $O/pytest_gpu.txt 2>&1; echo "pytest exit $?" >> $O/pytest_gpu.txt
tail -3 $O/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; tail -1 $O/smoke.txt
timeout 900 python bench.py > $O/bench_c5.json 2> $O/bench_c5.err; tail -c 300 $O/bench_c5.json
timeout 900 python bench.py --k-ckpt 32 --no-cpu-baseline > $O/bench_c5_k32.json 2> $O/bench_c5_k32.err; tail -c 200 $O/bench_c5_k32.json
for c in c1a c1b c2 c2cl c3 c3cl c3liquid c4; do
  timeout 600 python bench.py --config $c > $O/configs/bench_$c.json 2> $O/configs/bench_$c.err
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c5.csv python tools/profile_driver.py --steps 16 --k 2 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c2.csv python tools/profile_driver.py --config c2 --steps 64 --k 1 > /dev/null 2>&1
fi
[ -n "$SKIP_FULL" ] && exit 0
X=lts__t_sectors_op_red.sum,lts__t_sectors_op_atom.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed
timeout 1200 ncu --set full --metrics $X --clock-control none --import-source on -k regex:'^k_(p2g|g2p|canon|grid_op|bin_scan|bin_scatter)$' -s 8 -c 8 -o $O/full_fwd -f python tools/profile_driver.py --steps 4 --k 2 > $O/ncu_full.log 2>&1
timeout 1200 ncu --set full --metrics $X --clock-control none --import-source on -k regex:'^k_(p2g_grad|g2p_grad|g2p_grad_gather|grid_op_grad)$' -c 4 -o $O/full_bwd -f python tools/profile_driver.py --steps 4 --k 2 >> $O/ncu_full.log 2>&1
tail -2 $O/ncu_full.log
mkdir -p gpurun_out/sanitize; timeout 2400 bash tools/sanitize.sh > $O/sanitize_summary.txt 2>&1; cp -r gpurun_out/sanitize $O/
cat $O/sanitize_summary.txt
