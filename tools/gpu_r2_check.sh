cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/r2_gpu1_smi.txt
python -m paper_1910_00935_b200.build > /dev/null
rm -f gpurun_out/parity_record.jsonl
timeout 1500 python -m pytest tests -m gpu -q -s -p no:randomly --durations=25 > gpurun_out/r2_pytest_gpu1.txt 2>&1
echo "pytest exit $?" >> gpurun_out/r2_pytest_gpu1.txt
tail -40 gpurun_out/r2_pytest_gpu1.txt
timeout 600 python bench.py > gpurun_out/r2_bench1.json 2> gpurun_out/r2_bench1.err
tail -c 600 gpurun_out/r2_bench1.json
timeout 2400 bash tools/sanitize.sh
