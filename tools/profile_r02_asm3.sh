#!/bin/bash
# ncu --set full of the 3D fixed-p assembly kernel at 243^3, p = 2 and p = 8
# (run under gpurun from the repo root, after the timing pass exits 0).
python tools/c3_assembly.py 5 1 2 4 8 > gpurun_out/c3_asm_times.log 2>&1 || exit 1
python tools/c3_assembly.py 6 2 > gpurun_out/c5_asm_times.log 2>&1 || exit 1
for p in 2 8; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_assemble3" -c 1 \
      -o gpurun_out/prof_r02_asm3_p$p python tools/profile_3d.py 5 $p 0 > gpurun_out/ncu_asm3_p$p.log 2>&1
  ncu -i gpurun_out/prof_r02_asm3_p$p.ncu-rep --page raw --csv > gpurun_out/prof_r02_asm3_p$p.raw.csv 2>/dev/null
  python tools/ncu_hot_lines.py gpurun_out/prof_r02_asm3_p$p.ncu-rep 50 > gpurun_out/prof_r02_asm3_p$p.hot.txt 2>&1
  rm -f gpurun_out/prof_r02_asm3_p$p.ncu-rep
done
