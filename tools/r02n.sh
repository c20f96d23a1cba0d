#!/bin/bash
set -x
python -m pytest tests -m gpu -x -q > gpurun_out/r02n_gputest.txt 2>&1; echo tests=$? >> gpurun_out/r02n_gputest.txt
tail -3 gpurun_out/r02n_gputest.txt
python -c "import __graft_entry__ as g; g.smoke()"
python bench.py > gpurun_out/r02n_bench.json 2> gpurun_out/r02n_bench.err; echo bench=$?
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r02n_bench_ref.json 2>/dev/null
python tools/profile_comp.py 8 2 > /dev/null 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_residual_comp_st -c 1 \
    -o gpurun_out/prof_r02_comp2d python tools/profile_comp.py 8 2 > gpurun_out/ncu_comp2d.log 2>&1
ncu -i gpurun_out/prof_r02_comp2d.ncu-rep --page raw --csv > gpurun_out/prof_r02_comp2d.raw.csv
rm -f gpurun_out/prof_r02_comp2d.ncu-rep
python tools/ncu_raw_summary.py gpurun_out/prof_r02_comp2d.raw.csv
