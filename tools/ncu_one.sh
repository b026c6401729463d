#!/bin/bash
# ncu --set full (with source) of one kernel at C5 size -> gpurun_out/one_$K.ncu-rep + its line / SASS summaries.
# usage (through gpurun): K=k_p2g bash tools/ncu_one.sh
cd "$(dirname "$0")/.."; mkdir -p gpurun_out
python -m paper_1910_00935_b200.build > /dev/null
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^${K}\$" -s 2 -c 2 \
  -o gpurun_out/one_$K -f python tools/profile_driver.py --steps 3 --k 2 > gpurun_out/ncu_one_$K.log 2>&1
tail -2 gpurun_out/ncu_one_$K.log
python tools/ncu_line_summary.py gpurun_out/one_$K.ncu-rep "^${K}\$" 60 > gpurun_out/lines_$K.txt 2>&1
python tools/ncu_sass_summary.py gpurun_out/one_$K.ncu-rep "^${K}\$" > gpurun_out/sass_$K.txt 2>&1
python tools/ncu_kernel_table.py gpurun_out/one_$K.ncu-rep > gpurun_out/table_$K.txt 2>&1
