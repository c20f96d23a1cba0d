#!/bin/bash
set -x
python tools/profile_pack.py 8 || exit 1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_pack_patches -c 1 \
    -o gpurun_out/prof_r02_pack python tools/profile_pack.py 8 > gpurun_out/ncu_pack.log 2>&1
ncu -i gpurun_out/prof_r02_pack.ncu-rep --page raw --csv > gpurun_out/prof_r02_pack.raw.csv
python tools/ncu_hot_lines.py gpurun_out/prof_r02_pack.ncu-rep 40 > gpurun_out/prof_r02_pack.hot.txt 2>&1
rm -f gpurun_out/prof_r02_pack.ncu-rep
python tools/ncu_raw_summary.py gpurun_out/prof_r02_pack.raw.csv
head -30 gpurun_out/prof_r02_pack.hot.txt
