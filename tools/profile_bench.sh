#!/bin/bash
# Profile capture used for profiles/ (run under gpurun from the repo root).
set -x
python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/prof_plain.json 2> gpurun_out/prof_plain.err && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
echo launches=$?
python tools/profile_step.py exact > gpurun_out/plain_exact.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_fixed|k_coarse_geo|k_residual" -c 6 \
    -o gpurun_out/prof_r01 python tools/profile_step.py exact > gpurun_out/ncu_full.log 2>&1
echo full=$?
