#!/bin/bash
# Round-2 evidence pass on one B200 (run under gpurun from the repo root):
# GPU tests, smoke, the bench line, then the ncu launch list of the bench and
# the --set full captures of the 729^3 TMA residual and the 3D assembly.
set -x
python -m pytest tests -m gpu -x -q > gpurun_out/r02_gputest.txt 2>&1; echo tests=$? >> gpurun_out/r02_gputest.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02_smoke.txt 2>&1
python bench.py > gpurun_out/r02_bench.json 2> gpurun_out/r02_bench.err; echo bench=$?
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r02_bench_ref.json 2> gpurun_out/r02_bench_ref.err
bash tools/profile_r02_tma.sh
bash tools/profile_r02_asm3.sh
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fixed_res -c 1 \
    -o gpurun_out/prof_r02_fixed python tools/profile_step.py > gpurun_out/ncu_fixed.log 2>&1
ncu -i gpurun_out/prof_r02_fixed.ncu-rep --page raw --csv > gpurun_out/prof_r02_fixed.raw.csv 2>/dev/null
rm -f gpurun_out/prof_r02_fixed.ncu-rep
bash tools/profile_launches.sh
