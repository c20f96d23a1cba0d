"""Driver for ncu captures of the 3D kernels (run it under `ncu -k regex:...`;
the printed times are meaningless under the profiler).

usage: python tools/profile_3d.py [depth] [p] [cycles] [plane_width]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2005_03606_b200 as lzb  # noqa: E402

depth = int(sys.argv[1]) if len(sys.argv) > 1 else 5
p = int(sys.argv[2]) if len(sys.argv) > 2 else 8
cycles = int(sys.argv[3]) if len(sys.argv) > 3 else 2
w = int(sys.argv[4]) if len(sys.argv) > 4 else 0
G = lzb.Grid3(depth, lzb.field3_grf(lzb.grf_table(1, 64, 0.05, 1.0)), delta_max=1e-8, fixed_p3=w, plane_width=w)
G.assemble_fixed(p)
G.init_cycle(solver="adafac-pi", omega=0.6, max_cycles=10 ** 6)
for _ in range(cycles):
    print(G.step()["normalized"])
G.close()
