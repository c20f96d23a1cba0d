"""ncu driver: the compressed-record residual at one plane width on a large grid.

usage: python tools/profile_comp.py depth width
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2005_03606_b200 as lzb  # noqa: E402

depth, w = int(sys.argv[1]), int(sys.argv[2])
d = lzb.make_desc(depth=depth, field=lzb.field_sinusoid(0.9, 6.0), solver="adafac-pi", omega=0.6,
                  rhs_kind="sinprod", max_cycles=100, delta_max=1e-8, integration="fast", fixed_p3=w, plane_width=w)
g = lzb.Grid(d, 1)
g.assemble_fixed(4)
print(g.time_kernel(lzb.TK_RESIDUAL, 1))
