"""A 3D grid with leaf planes of width W (0 = FP64), one cycle (its first
kernel launches include the leaf residual): for a targeted ncu capture."""
import sys

sys.path.insert(0, ".")
import paper_2005_03606_b200 as lzb  # noqa: E402

depth, W = int(sys.argv[1]), int(sys.argv[2])
g = lzb.Grid3(depth, lzb.field3_grf(lzb.grf_table(1, 64, 0.05, 1.0)), delta_max=1e-8, fixed_p3=W, plane_width=W)
g.assemble_fixed(2)
g.init_cycle(solver="adafac-pi", omega=0.6, max_cycles=10 ** 6)
g.step()
print("ok")
