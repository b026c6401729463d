# ncu --set full capture of the forward kernels (C5 size) -> gpurun_out/fwd.ncu-rep
cd "$(dirname "$0")/.."; mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'^k_(p2g|g2p|bin_scan|bin_scatter|grid_op)$' -s 6 -c 7 -o gpurun_out/fwd -f python tools/profile_driver.py --steps 4 --k 2 > gpurun_out/ncu_fwd.log 2>&1
tail -3 gpurun_out/ncu_fwd.log
