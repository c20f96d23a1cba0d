#!/bin/bash
# the 3D fused leaf update: march kernel (chunk sweep) against the row kernel, then the 3D parity suite
mkdir -p gpurun_out
{
echo "== rows (k3_update_fine_st)"; LZB_UPDATE3_ROWS=1 python tools/k3_times.py 5 6
for pg in 9 27; do echo "== march pg=$pg"; LZB_UPDATE3_PG=$pg python tools/k3_times.py 5 6; done
} > gpurun_out/r02_update3_march_sweep.txt 2>&1
cat gpurun_out/r02_update3_march_sweep.txt
bash tools/profile_r02_march.sh > gpurun_out/march_prof.log 2>&1; tail -48 gpurun_out/march_prof.log | head -36
