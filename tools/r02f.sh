#!/bin/bash
set -x
python -m pytest tests -m gpu -x -q > gpurun_out/r02f_gputest.txt 2>&1; echo tests=$? >> gpurun_out/r02f_gputest.txt
tail -5 gpurun_out/r02f_gputest.txt
python tools/cycle_probe.py 6 40
LZB_TRACE=1 python tools/tts_probe.py 2>&1 | grep -v "host step\|graph slot" | tail -12
LZB_DEVLOOP=1 python tools/tts_probe.py 2>&1 | grep "pass 1"
