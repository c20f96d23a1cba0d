#!/bin/bash
# ncu --set full captures of the 3D kernels (243^3, p = 8) and of the
# compressed-record residual (6561^2, width 4), for profiles/ (run under gpurun).
set -x
python tools/c3_cycle.py 5 8 2 > gpurun_out/plain_c3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_assemble3|k3_residual|k3_galerkin" -c 3 \
    -o gpurun_out/prof_r01_3d python tools/c3_cycle.py 5 8 2 > gpurun_out/ncu_3d.log 2>&1
echo c3=$?
python tools/profile_comp.py 8 4 > gpurun_out/plain_comp.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_residual_comp" -c 1 \
    -o gpurun_out/prof_r01_comp python tools/profile_comp.py 8 4 > gpurun_out/ncu_comp.log 2>&1
echo comp=$?
