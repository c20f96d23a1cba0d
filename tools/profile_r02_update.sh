#!/bin/bash
# ncu --set full of the 729^3 leaf u-hat and fused update kernels (one launch each)
set -x
python tools/k3_prof.py 6 0 > gpurun_out/k3p_plain.log 2>&1 || exit 1
for spec in "k3_uhat_st:1" "k3_update_fine_st:1"; do
  name=${spec%%:*}
  timeout 900 ncu --set full --clock-control none --import-source on --kernel-id ::regex:$spec \
      -o gpurun_out/prof_r02_729_$name python tools/k3_prof.py 6 0 > gpurun_out/ncu_$name.log 2>&1
  ncu -i gpurun_out/prof_r02_729_$name.ncu-rep --page raw --csv > gpurun_out/prof_r02_729_$name.raw.csv
  python tools/ncu_hot_lines.py gpurun_out/prof_r02_729_$name.ncu-rep 25 > gpurun_out/prof_r02_729_$name.hot.txt 2>&1
  rm -f gpurun_out/prof_r02_729_$name.ncu-rep
done
python tools/ncu_raw_summary.py gpurun_out/prof_r02_729_k3_uhat_st.raw.csv gpurun_out/prof_r02_729_k3_update_fine_st.raw.csv
head -14 gpurun_out/prof_r02_729_k3_update_fine_st.hot.txt
