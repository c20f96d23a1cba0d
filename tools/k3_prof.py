"""One 729^3 (or 243^3) grid, one cycle, then one launch each of the leaf
u-hat and the fused update (for an ncu capture of those kernels)."""
import sys

sys.path.insert(0, ".")
import paper_2005_03606_b200 as lzb  # noqa: E402

depth = int(sys.argv[1]) if len(sys.argv) > 1 else 6
g = lzb.Grid3(depth, lzb.field3_grf(lzb.grf_table(1, 64, 0.05, 1.0)), delta_max=1e-8)
g.assemble_fixed(2)
g.init_cycle(solver="adafac-pi", omega=0.6, max_cycles=10 ** 6)
g.step()
for tk in [int(a) for a in (sys.argv[2:] or [lzb.TK_UHAT, lzb.TK_BACK, lzb.TK_RESTRICT])]:
    g.time_kernel(tk, 1)
print("ok")
