#!/bin/bash
# ncu --set full captures (one launch each) of the 3D kernels after the
# class-plane / z-march / exp-recurrence changes, 243^3, p = 8 (run under
# gpurun from the repo root); reports are summarised on the box (raw metrics
# CSV + source hot lines), only the summaries come back (gpurun_out/ is
# capped at 64 MiB). Then the compressed-plane residual (width 2).
set -x
summ() {
  ncu -i gpurun_out/$1.ncu-rep --page raw --csv > gpurun_out/$1.raw.csv 2>/dev/null
  python tools/ncu_hot_lines.py gpurun_out/$1.ncu-rep 40 > gpurun_out/$1.hot.txt 2>&1
  rm -f gpurun_out/$1.ncu-rep
}
python tools/profile_3d.py 5 8 2 > gpurun_out/p3d_a.log 2>&1 || exit 1
for k in k_assemble3 k3_residual_z k3_update_fine k3_uhat; do
  ncu --set full --clock-control none --import-source on -k regex:"$k" -c 1 \
      -o gpurun_out/prof_r01_3d_$k python tools/profile_3d.py 5 8 2 > gpurun_out/ncu_$k.log 2>&1
  echo $k=$?; summ prof_r01_3d_$k
done
ncu --set full --clock-control none --import-source on -k regex:"k3_galerkin" -s 0 -c 1 \
    -o gpurun_out/prof_r01_3d_k3_galerkin python tools/profile_3d.py 5 8 2 > gpurun_out/ncu_gal.log 2>&1
echo gal=$?; summ prof_r01_3d_k3_galerkin
python tools/profile_3d.py 5 2 1 2 > gpurun_out/p3d_c.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k3_residual_z" -c 1 \
    -o gpurun_out/prof_r01_3dcomp python tools/profile_3d.py 5 2 1 2 > gpurun_out/ncu_3dcomp.log 2>&1
echo c=$?; summ prof_r01_3dcomp
du -sh gpurun_out
