#!/bin/bash
set -x
python -m pytest tests -m gpu -x -q > gpurun_out/r02g_gputest.txt 2>&1; echo tests=$? >> gpurun_out/r02g_gputest.txt
tail -4 gpurun_out/r02g_gputest.txt
LZB_TRACE=1 python tools/tts_eager_trace.py 2>&1 | tail -22
python tools/tts_probe.py 2>&1 | grep "pass 1"
