# Full GPU evidence run (through gpurun): parity tests, default bench (with cpu_baseline),
# ncu launch list of a 16-step C5 fwd+bwd, ncu --set full of the hot kernels.
set -x
cd "$(dirname "$0")/.."; mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/pytest_gpu.txt
cat gpurun_out/pytest_gpu.txt
timeout 600 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err
cat gpurun_out/bench_full.json
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python tools/profile_driver.py --steps 16 --k 2 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'^k_(p2g|g2p|canon|grid_op|bin_scan|bin_scatter)$' -s 8 -c 8 -o gpurun_out/full_fwd -f python tools/profile_driver.py --steps 4 --k 2 > gpurun_out/ncu_full.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'^k_(p2g_grad|g2p_grad|g2p_grad_gather|grid_op_grad)$' -c 4 -o gpurun_out/full_bwd -f python tools/profile_driver.py --steps 4 --k 2 >> gpurun_out/ncu_full.log 2>&1
tail -3 gpurun_out/ncu_full.log
