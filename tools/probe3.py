import os, sys
sys.path.insert(0, '.')
import paper_2005_03606_b200 as lzb
depth = int(sys.argv[1]); W = int(sys.argv[2])
g = lzb.Grid3(depth, lzb.field3_grf(lzb.grf_table(1, 16, 0.05, 1.0)), delta_max=1e-8, fixed_p3=W, plane_width=W)
g.assemble_fixed(2)
g.init_cycle(solver="adafac-pi", omega=0.6, max_cycles=100)
try:
    r = g.step()
    print(depth, W, os.environ.get("LZB_NO_TMA"), "ok", r["residual"])
except Exception as e:
    print(depth, W, os.environ.get("LZB_NO_TMA"), "ERR", e)
