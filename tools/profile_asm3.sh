summ() {
  ncu -i gpurun_out/$1.ncu-rep --page raw --csv > gpurun_out/$1.raw.csv 2>/dev/null
  python tools/ncu_hot_lines.py gpurun_out/$1.ncu-rep 40 > gpurun_out/$1.hot.txt 2>&1
  rm -f gpurun_out/$1.ncu-rep
}
python tools/profile_3d.py 5 2 0 > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_assemble3" -c 1 -o gpurun_out/prof_asm3_p2 python tools/profile_3d.py 5 2 0 > gpurun_out/ncu_asm3.log 2>&1
echo a=$?; summ prof_asm3_p2
