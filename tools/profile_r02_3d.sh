#!/bin/bash
# ncu --set full of the 729^3 leaf-level cycle kernels (one launch each, picked
# by invocation number: the grid's first cycle launches the leaf residual first,
# u-hat / restriction once per level 6..1, the fused update once; time_kernel
# then launches the leaf kernel again). Run under gpurun from the repo root.
set -x
python tools/k3_prof.py 6 1 0 2 7 > gpurun_out/k3p_plain.log 2>&1 || exit 1
for spec in "k3_residual_z:1" "k3_uhat_st:7" "k3_restrict:7" "k3_update_fine_st:2"; do
  name=${spec%%:*}
  timeout 900 ncu --set full --clock-control none --import-source on --kernel-id ::regex:$spec \
      -o gpurun_out/prof_r02_729_$name python tools/k3_prof.py 6 1 0 2 7 > gpurun_out/ncu_$name.log 2>&1
  ncu -i gpurun_out/prof_r02_729_$name.ncu-rep --page raw --csv > gpurun_out/prof_r02_729_$name.raw.csv
  ncu -i gpurun_out/prof_r02_729_$name.ncu-rep --page source --csv > gpurun_out/prof_r02_729_$name.src.csv 2>/dev/null
  gzip -f gpurun_out/prof_r02_729_$name.src.csv; rm -f gpurun_out/prof_r02_729_$name.ncu-rep
done
ls -la gpurun_out/prof_r02_729_*
