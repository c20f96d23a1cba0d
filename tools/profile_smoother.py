"""Driver for ncu captures of the leaf-level cycle / stream-pack kernels on a
large 2D grid (run it under `ncu -k regex:...`; the printed times are
meaningless under the profiler).

usage: python tools/profile_smoother.py [depth] [kernel ids, e.g. 1,5] [cycles before]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2005_03606_b200 as lzb  # noqa: E402

depth = int(sys.argv[1]) if len(sys.argv) > 1 else 8
ids = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else [lzb.TK_RESIDUAL, lzb.TK_PACK]
f = lzb.field_sinusoid(0.9, 6.0)
d = lzb.make_desc(depth=depth, field=f, solver="adafac-pi", omega=0.6, rhs_kind="sinprod", max_cycles=100,
                  delta_max=1e-8, integration="fast")
g = lzb.Grid(d, 1)
g.assemble_fixed(4)
for _ in range(int(sys.argv[3]) if len(sys.argv) > 3 else 0):
    g.step()
for tk in ids:
    print(tk, g.time_kernel(tk, 1))
g.close()
