#!/bin/bash
# compute-sanitizer over the parity configs that exercise concurrency:
# the concurrent anarchic mode (two streams, staging copy, event swap-in), the
# device-side cycle loop, the TMA-staged 3D residual and smoke(). One tool per
# pass; run under gpurun from the repo root. Output: gpurun_out/sanitize_<tool>.txt
SEL='tests/test_gpu_grid.py::test_concurrent_anarchic_converges_to_eager_solution
tests/test_gpu_grid.py::test_geometric_start_concurrent_converges_to_deterministic_solution
tests/test_gpu_grid.py::test_throttled_anarchic_fifo
tests/test_gpu_grid.py::test_run_device_loop_matches_stepping
tests/test_gpu_3d.py::test_grid3_compressed_planes_bit_identical
tests/test_gpu_3d.py::test_cycle3_matches_restatement'
for tool in ${@:-memcheck racecheck synccheck}; do
  timeout 2400 compute-sanitizer --tool $tool --error-exitcode 9 --launch-timeout 0 \
      python -m pytest -x -q -m gpu $SEL > gpurun_out/sanitize_$tool.txt 2>&1
  echo "exit=$?" >> gpurun_out/sanitize_$tool.txt
  tail -4 gpurun_out/sanitize_$tool.txt
done
