#!/bin/bash
# bench at HEAD + ncu of the 729^3 W=2 residual after the decode work
set -x
python bench.py > gpurun_out/r02h_bench.json 2> gpurun_out/r02h_bench.err; echo bench=$?
tail -c 600 gpurun_out/r02h_bench.err
python tools/k3_prof_w.py 6 2 > /dev/null 2>&1 || exit 1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-id ::regex:k3_residual_tma:1 \
    -o gpurun_out/prof_r02_tma_w2b python tools/k3_prof_w.py 6 2 > gpurun_out/ncu_tma_w2b.log 2>&1
ncu -i gpurun_out/prof_r02_tma_w2b.ncu-rep --page raw --csv > gpurun_out/prof_r02_tma_w2b.raw.csv
python tools/ncu_hot_lines.py gpurun_out/prof_r02_tma_w2b.ncu-rep 40 > gpurun_out/prof_r02_tma_w2b.hot.txt 2>&1
rm -f gpurun_out/prof_r02_tma_w2b.ncu-rep
