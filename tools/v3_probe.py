"""The bench's C3 V(2,2) sequence in isolation: 243^3 (or argv depth), p = 8
operators, 10 V(2,2) cycles; argv[2] = 1 runs the adaFAC-PI solve first as bench.py does."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2005_03606_b200 as lzb  # noqa: E402

depth = int(sys.argv[1]) if len(sys.argv) > 1 else 5
pre = int(sys.argv[2]) if len(sys.argv) > 2 else 0
p = int(sys.argv[3]) if len(sys.argv) > 3 else 8
g3 = lzb.Grid3(depth, lzb.field3_grf(lzb.grf_table(1, 64, 0.05, 1.0)), delta_max=1e-8)
g3.assemble_fixed(p)
if pre:
    g3.init_cycle(solver="adafac-pi", omega=0.6, max_cycles=400, target=1e-10)
    g3.assemble_fixed(p)
    n = 0
    while g3.step()["status"] == 0:
        n += 1
    print("pre-solve cycles", n)
g3.init_cycle(solver="additive", omega=0.6, max_cycles=10 ** 6)
for k in range(10):
    r = g3.vcycle(2)
    print(k, r["residual"], r["normalized"], r["status"], flush=True)
