#!/bin/bash
# Profile capture used for profiles/ (run under gpurun from the repo root).
#   1. plain bench run (no profiler) -> gpurun_out/prof_plain.json
#   2. ncu launch list of the same bench command (gpu__time_duration, clocks free)
#   3. ncu --set full of the top kernels: exact assembly (729^2, p=32) and the
#      leaf-level residual / fused update / stream pack on the 6561^2 grid
set -x
python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/prof_plain.json 2> gpurun_out/prof_plain.err && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
echo launches=$?
python tools/profile_step.py exact > gpurun_out/plain_exact.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_fixed_res" -c 2 \
    -o gpurun_out/prof_r01 python tools/profile_step.py exact > gpurun_out/ncu_full.log 2>&1
echo full=$?
python tools/profile_smoother.py 8 1,5 2 > gpurun_out/plain_sm.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_residual|k_pack_patches|k_update_fine" \
    -s 20 -c 3 -o gpurun_out/prof_r01_hbm python tools/profile_smoother.py 8 1,5 2 > gpurun_out/ncu_hbm.log 2>&1
echo hbm=$?
