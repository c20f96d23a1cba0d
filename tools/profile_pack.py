"""One LZMG stream pack of the 6561^2 grid (p = 4 assembly): for an ncu capture of k_pack_patches."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2005_03606_b200 as lzb  # noqa: E402

depth = int(sys.argv[1]) if len(sys.argv) > 1 else 8
d = lzb.make_desc(depth=depth, field=lzb.field_sinusoid(0.9, 6.0), solver="adafac-pi", omega=0.6, rhs_kind="sinprod",
                  max_cycles=100, delta_max=1e-8, integration="fast")
g = lzb.Grid(d, 1)
g.assemble_fixed(4)
g.step()
print("pack ms", g.time_kernel(lzb.TK_PACK, 2))
