#!/bin/bash
set -x
python -m pytest tests/test_gpu_grid.py tests/test_gpu_baseline.py tests/test_cpp_shim.py tests/test_vcycle2.py tests/test_dist_cpp.py -m gpu -x -q > gpurun_out/r02e_gputest.txt 2>&1; echo tests=$? >> gpurun_out/r02e_gputest.txt
tail -5 gpurun_out/r02e_gputest.txt
python tools/cycle_probe.py 6 40
LZB_SMALL_MAXN=9 python tools/cycle_probe.py 6 40
LZB_SMALL_MAXN=27 python tools/cycle_probe.py 6 40
LZB_SMALL_MAXN=243 python tools/cycle_probe.py 6 40
python tools/cycle_probe.py 5 40
python tools/cycle_probe.py 8 20
python tools/tts_probe.py 2>&1 | grep pass
LZB_DEVLOOP=1 python tools/tts_probe.py 2>&1 | grep pass
