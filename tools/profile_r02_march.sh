#!/bin/bash
# ncu --set full of the 729^3 marching fused leaf update (one launch)
set -x
mkdir -p gpurun_out
python tools/k3_prof.py 6 0 > gpurun_out/k3p_plain.log 2>&1 || exit 1
name=k3_update_fine_march
timeout 900 ncu --set full --clock-control none --import-source on --kernel-id ::regex:$name:1 \
    -o gpurun_out/prof_r02_729_$name python tools/k3_prof.py 6 0 > gpurun_out/ncu_$name.log 2>&1
ncu -i gpurun_out/prof_r02_729_$name.ncu-rep --page raw --csv > gpurun_out/prof_r02_729_$name.raw.csv
python tools/ncu_hot_lines.py gpurun_out/prof_r02_729_$name.ncu-rep 30 > gpurun_out/prof_r02_729_$name.hot.txt 2>&1
rm -f gpurun_out/prof_r02_729_$name.ncu-rep
python tools/ncu_raw_summary.py gpurun_out/prof_r02_729_$name.raw.csv
head -32 gpurun_out/prof_r02_729_$name.hot.txt
