"""5 cycles on a 3^depth grid (after a p=4 fixed assembly) for ncu launch lists.

usage: python tools/profile_cycle.py [solver] [depth]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2005_03606_b200 as lzb  # noqa: E402

f = lzb.field_sinusoid(0.9, 6.0)
d = lzb.make_desc(depth=int(sys.argv[2]) if len(sys.argv) > 2 else 6, field=f, solver=sys.argv[1] if len(sys.argv) > 1 else "additive", omega=0.6,
                  rhs_kind="sinprod", max_cycles=100)
g = lzb.Grid(d, 1)
g.assemble_fixed(4)
for _ in range(5):
    g.step()
print("done")
