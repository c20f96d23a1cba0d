"""V(2,2) cycle time on the 243^3 GRF grid (BASELINE configs[2])."""
import sys
import time
sys.path.insert(0, ".")
import torch  # noqa: E402
import paper_2005_03606_b200 as lzb  # noqa: E402

g3 = lzb.Grid3(5, lzb.field3_grf(lzb.grf_table(1, 64, 0.05, 1.0)), delta_max=1e-8)
g3.assemble_fixed(2)
g3.init_cycle(solver="additive", omega=0.6, seed=42, max_cycles=10 ** 6)
for _ in range(2):
    g3.vcycle(2)
torch.cuda.synchronize()
t = time.perf_counter()
reps = [g3.vcycle(2) for _ in range(10)]
torch.cuda.synchronize()
print("V(2,2) ms", 1e3 * (time.perf_counter() - t) / 10, "normalized", reps[-1]["normalized"])
