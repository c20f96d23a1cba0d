"""Debug probe: lzb_grid_vcycle vs the restatement, ops refreshed per cycle."""
import sys
sys.path.insert(0, ".")
import numpy as np
import paper_2005_03606_b200 as lzb
from oracle.port2v import VCycle2

depth, nu = 3, 1
d = lzb.make_desc(depth=depth, field=lzb.checkerboard(7, 8), solver="additive", omega=0.6, rhs_kind="sinprod",
                  max_cycles=100)
G = lzb.Grid(d, 42)
G.assemble_fixed(3)
u0 = G.vertices(depth, lzb.T.V_U).copy()
prev = None
ref = None
for k in range(5):
    a = G.vcycle(nu)
    ops = [G.cells(l)["ops"].copy() for l in range(depth + 1)]
    p1 = [G.cells(l)["p1"].copy() for l in range(depth + 1)]
    if prev is not None:
        print("cycle", k, "ops changed per level", [float(np.abs(x - y).max()) for x, y in zip(ops, prev)],
              "p1 bottom count", [int((q == 0).sum()) for q in p1])
    prev = ops
    if ref is None:
        fl = G.vertices(depth, lzb.T.V_FL)
        P = [np.array([[G.transfer(l, cx, cy) for cx in range(3 ** l)] for cy in range(3 ** l)]) for l in range(depth)]
        ref = VCycle2(ops, P, fl, u0, omega=0.6, max_cycles=100)
    b = ref.vstep(nu)
    print(k, a["residual"], b["residual"], a["status"], b["status"])
    for l in range(depth + 1):
        print("   lvl", l, "u diff", float(np.abs(G.vertices(l, lzb.T.V_U) - ref.u[l]).max()),
              "fl diff", float(np.abs(G.vertices(l, lzb.T.V_FL) - ref.fl[l]).max()))
