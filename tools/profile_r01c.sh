#!/bin/bash
# ncu --set full captures of the 3D kernels after the class-plane / z-march /
# exp-recurrence changes (run under gpurun from the repo root); the reports
# are summarised on the box (raw metrics CSV + source hot lines) and only the
# summaries come back (gpurun_out/ is capped at 64 MiB):
#   243^3 p = 8: k_assemble3, k3_residual_z, k3_update_fine, k3_galerkin
#   729^3 p = 2: k_assemble3 (the C5 assembly), k3_residual_z
#   243^3 p = 2, plane_width 2: k3_residual_z on compressed planes
set -x
summ() {
  ncu -i gpurun_out/$1.ncu-rep --page raw --csv > gpurun_out/$1.raw.csv 2>/dev/null
  python tools/ncu_hot_lines.py gpurun_out/$1.ncu-rep 40 > gpurun_out/$1.hot.txt 2>&1
  rm -f gpurun_out/$1.ncu-rep
}
python tools/profile_3d.py 5 8 2 > gpurun_out/p3d_a.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_assemble3|k3_residual_z|k3_update_fine|k3_galerkin" -c 4 \
    -o gpurun_out/prof_r01_3db python tools/profile_3d.py 5 8 2 > gpurun_out/ncu_3db.log 2>&1
echo a=$?; summ prof_r01_3db
python tools/profile_3d.py 6 2 1 > gpurun_out/p3d_b.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_assemble3|k3_residual_z" -c 2 \
    -o gpurun_out/prof_r01_c5 python tools/profile_3d.py 6 2 1 > gpurun_out/ncu_c5.log 2>&1
echo b=$?; summ prof_r01_c5
python tools/profile_3d.py 5 2 1 2 > gpurun_out/p3d_c.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k3_residual_z" -c 1 \
    -o gpurun_out/prof_r01_3dcomp python tools/profile_3d.py 5 2 1 2 > gpurun_out/ncu_3dcomp.log 2>&1
echo c=$?; summ prof_r01_3dcomp
du -sh gpurun_out
