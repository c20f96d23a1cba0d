#!/bin/bash
# Round-2 second pass on one B200: the conditional-graph probe, the GPU suite,
# the 729^3 leaf residual per plane width, time to solution with the device
# loop (and LZB_NO_DEVLOOP=1 beside it), then the sanitizer passes.
set -x
nvcc -std=c++17 -O2 -gencode arch=compute_100a,code=sm_100a -o /tmp/cond_probe tools/ubench/cond_graph_probe.cu \
    && /tmp/cond_probe > gpurun_out/cond_probe.txt 2>&1
cat gpurun_out/cond_probe.txt
python -m pytest tests -m gpu -x -q > gpurun_out/r02b_gputest.txt 2>&1; echo tests=$? >> gpurun_out/r02b_gputest.txt
tail -5 gpurun_out/r02b_gputest.txt
python tools/c5_planes.py 6 2 0,2,3,4 3 > gpurun_out/r02b_c5_planes.txt 2>&1
cat gpurun_out/r02b_c5_planes.txt
python tools/tts_probe.py > gpurun_out/r02b_tts_devloop.txt 2>&1
LZB_NO_DEVLOOP=1 python tools/tts_probe.py > gpurun_out/r02b_tts_hostloop.txt 2>&1
cat gpurun_out/r02b_tts_devloop.txt gpurun_out/r02b_tts_hostloop.txt
bash tools/sanitize.sh "$@"
