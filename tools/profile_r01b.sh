set -x
python tools/profile_smoother.py 8 5 0 > gpurun_out/plain_pack.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_pack_patches" -c 1 \
    -o gpurun_out/prof_pack python tools/profile_smoother.py 8 5 0 > gpurun_out/ncu_pack.log 2>&1
echo pack=$?
python tools/c3_cycle.py 5 8 2 > gpurun_out/plain_c3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k3_residual|k3_update|k3_restrict|k3_uhat|k3_prolong" -c 6 \
    -o gpurun_out/prof_3dcyc python tools/c3_cycle.py 5 8 2 > gpurun_out/ncu_3dcyc.log 2>&1
echo c3=$?
