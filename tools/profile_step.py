"""Small driver for ncu captures: one 729^2 assembly pass per integration
path at p=32, then a few multigrid cycles."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2005_03606_b200 as lzb  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "both"
f = lzb.field_sinusoid(0.9, 6.0)
for mode in (["exact", "fast"] if which == "both" else [which]):
    d = lzb.make_desc(depth=6, field=f, solver="additive", omega=0.6, assembly="adaptive",
                      rhs_kind="sinprod", integration=mode, max_cycles=100)
    g = lzb.Grid(d, 42)
    g.assemble_fixed(32)
    g.assemble_fixed(32)
    for _ in range(3):
        g.step()
print("done")
