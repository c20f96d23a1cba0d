#!/bin/bash
# final evidence pass: GPU suite, smoke, bench (both arms), 3D kernel times
# (the launch list of the bench is tools/profile_launches.sh: ~10 min under ncu, run separately)
set -x
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/r02_final_gputest.txt 2>&1; echo tests=$? >> gpurun_out/r02_final_gputest.txt
tail -4 gpurun_out/r02_final_gputest.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02_final_smoke.txt 2>&1; cat gpurun_out/r02_final_smoke.txt
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r02_final_bench_ref.json 2> gpurun_out/r02_final_bench_ref.err
python bench.py > gpurun_out/r02_final_bench.json 2> gpurun_out/r02_final_bench.err; echo bench=$?
tail -c 300 gpurun_out/r02_final_bench.err
python tools/k3_times.py 5 6 > gpurun_out/r02_final_k3_times.txt 2>&1; cat gpurun_out/r02_final_k3_times.txt
if [ -n "$LZB_EVIDENCE_LAUNCHES" ]; then bash tools/profile_launches.sh > /dev/null 2>&1; ls -la gpurun_out/launches_bench.csv.gz; fi
