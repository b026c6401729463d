# ncu --set full (with source) of every hot step kernel at C5 size -> gpurun_out/hot.ncu-rep,
# then the per-kernel SASS summaries (executed instructions / stall samples per opcode).
cd "$(dirname "$0")/.."; mkdir -p gpurun_out
python -m paper_1910_00935_b200.build > /dev/null
timeout 1500 ncu --set full --clock-control none --import-source on \
  -k regex:'^k_(p2g|p2g_grad|g2p|g2p_grad|g2p_grad_gather|canon|grid_op|grid_op_grad|bin_scan|bin_scatter)$' \
  -c 40 -o gpurun_out/hot -f python tools/profile_driver.py --steps 3 --k 2 > gpurun_out/ncu_hot.log 2>&1
tail -3 gpurun_out/ncu_hot.log
for k in k_p2g k_p2g_grad k_g2p k_g2p_grad k_g2p_grad_gather k_canon k_grid_op; do
  python tools/ncu_sass_summary.py gpurun_out/hot.ncu-rep "^${k}\$" > gpurun_out/sass_${k}.txt 2>&1
done
python tools/ncu_kernel_table.py gpurun_out/hot.ncu-rep > gpurun_out/hot_table.txt 2>&1
cat gpurun_out/hot_table.txt | cut -c1-250
