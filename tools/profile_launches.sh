#!/bin/bash
# ncu launch list of the bench command (gpu__time_duration per launch, clocks
# free; cold-cache and serialised, so only the shares are meaningful), after
# the same command has exited 0 without ncu. Run under gpurun from the repo root.
set -x
python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/prof_plain.json 2> gpurun_out/prof_plain.err || exit 1
timeout 2400 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
echo launches=$?
gzip -k gpurun_out/launches_bench.csv; ls -la gpurun_out/launches_bench.csv*
