#!/bin/bash
set -x
python -m pytest tests -m gpu -x -q > gpurun_out/r02j_gputest.txt 2>&1; echo tests=$? >> gpurun_out/r02j_gputest.txt
tail -4 gpurun_out/r02j_gputest.txt
python -c "import __graft_entry__ as g; g.smoke()"
python bench.py > gpurun_out/r02j_bench.json 2> gpurun_out/r02j_bench.err; echo bench=$?
tail -c 400 gpurun_out/r02j_bench.err
