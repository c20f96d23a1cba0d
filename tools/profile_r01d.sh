#!/bin/bash
# ncu --set full captures (one launch each, summarised on the box) of the
# kernels added late in round 1: the separable 3D Galerkin, the adaptive-tree
# assembly and cycle kernels (BASELINE configs[3], lbase 4 / lmax 6).
set -x
summ() {
  ncu -i gpurun_out/$1.ncu-rep --page raw --csv > gpurun_out/$1.raw.csv 2>/dev/null
  python tools/ncu_hot_lines.py gpurun_out/$1.ncu-rep 40 > gpurun_out/$1.hot.txt 2>&1
  rm -f gpurun_out/$1.ncu-rep
}
python tools/profile_3d.py 5 8 1 > /dev/null 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:"k3_galerkin" -c 1 \
    -o gpurun_out/prof_r01_gal python tools/profile_3d.py 5 8 1 > gpurun_out/ncu_gal.log 2>&1
echo gal=$?; summ prof_r01_gal
cat > gpurun_out/c4drv.py <<'PY'
import sys
sys.path.insert(0, ".")
import paper_2005_03606_b200 as lzb
T = lzb.Tree3(4, 6, lzb.field3_sphere())
T.assemble(1)
T.set_shell(0.01)
T.assemble_shell(8)
T.init_cycle(solver="adafac-pi", omega=0.6, max_cycles=100)
for _ in range(2):
    T.step()
PY
python gpurun_out/c4drv.py || exit 1
ncu --set full --clock-control none --import-source on -k regex:"k_assemble3_leaves|k4_residual|k4_update|k4_galerkin" -c 5 \
    -o gpurun_out/prof_r01_c4 python gpurun_out/c4drv.py > gpurun_out/ncu_c4.log 2>&1
echo c4=$?; summ prof_r01_c4
du -sh gpurun_out
