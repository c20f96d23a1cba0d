#!/bin/bash
# ncu --set full of the TMA leaf residual at 729^3 (FP64 planes and W = 2
# compressed planes): one launch each, after the plain runs exit 0.
set -x
python tools/k3_prof.py 6 1 > gpurun_out/k3p_plain.log 2>&1 || exit 1
for w in 0 2; do
  timeout 900 ncu --set full --clock-control none --import-source on --kernel-id ::regex:k3_residual_tma:1 \
      -o gpurun_out/prof_r02_tma_w$w python tools/k3_prof_w.py 6 $w > gpurun_out/ncu_tma_w$w.log 2>&1
  ncu -i gpurun_out/prof_r02_tma_w$w.ncu-rep --page raw --csv > gpurun_out/prof_r02_tma_w$w.raw.csv
  ncu -i gpurun_out/prof_r02_tma_w$w.ncu-rep --page source --csv 2>/dev/null | gzip > gpurun_out/prof_r02_tma_w$w.src.csv.gz
  rm -f gpurun_out/prof_r02_tma_w$w.ncu-rep
done
