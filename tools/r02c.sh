#!/bin/bash
set -x
python -m pytest tests/test_gpu_grid.py tests/test_gpu_baseline.py tests/test_cpp_shim.py -m gpu -x -q > gpurun_out/r02c_gputest.txt 2>&1; echo tests=$? >> gpurun_out/r02c_gputest.txt
tail -5 gpurun_out/r02c_gputest.txt
python tools/tts_probe.py > gpurun_out/r02c_tts_devloop.txt 2>&1
LZB_NO_DEVLOOP=1 python tools/tts_probe.py > gpurun_out/r02c_tts_hostloop.txt 2>&1
cat gpurun_out/r02c_tts_devloop.txt gpurun_out/r02c_tts_hostloop.txt
