#!/bin/bash
set -x
LZB_TRACE=1 python tools/tts_probe.py > gpurun_out/r02d_tts_trace.txt 2>&1
tail -120 gpurun_out/r02d_tts_trace.txt | grep -v "host step" | tail -60
for v in 0 1 2 3; do
  echo variant $v
  LZB_ASM3_VARIANT=$v python tools/c3_assembly.py 5 2 2>&1 | cut -c1-120
  LZB_ASM3_VARIANT=$v python tools/c3_assembly.py 6 2 2>&1 | cut -c1-120
done > gpurun_out/r02d_asm3_variants.txt 2>&1
cat gpurun_out/r02d_asm3_variants.txt
