"""Per-kernel HBM roofline of the cycle and stream-pack kernels on large 2D grids.

usage: python tools/smoother_roofline.py [depth ...]   (default 7 8)
Bytes / timing: paper_2005_03606_b200.measure.
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2005_03606_b200 as lzb  # noqa: E402
from paper_2005_03606_b200 import measure  # noqa: E402


def run(depth, peak):
    f = lzb.field_sinusoid(0.9, 6.0)
    d = lzb.make_desc(depth=depth, field=f, solver="adafac-pi", omega=0.6, rhs_kind="sinprod", max_cycles=100,
                      delta_max=1e-8, integration="fast")
    g = lzb.Grid(d, 1)
    g.assemble_fixed(4)
    for _ in range(2):
        g.step()
    tab = measure.hbm_kernel_table(g, depth, peak)
    for tk, name in ((lzb.TK_FRONT, "front_graph"), (lzb.TK_BACK, "back_graph")):
        tab[name] = {"ms": g.time_kernel(tk, 5)}
    g.close()
    rnd = {k: ({kk: (round(vv, 4) if isinstance(vv, float) else vv) for kk, vv in v.items()}
               if isinstance(v, dict) else v) for k, v in tab.items()}
    return {"depth": depth, "N": 3 ** depth, "kernels": rnd}


if __name__ == "__main__":
    depths = [int(a) for a in sys.argv[1:]] or [7, 8]
    peak = 6468.6
    try:
        mp = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                         "MEASURED_PEAKS.json")))
        peak = float(mp.get("hbm_gbs", peak))
    except Exception:
        pass
    for dpt in depths:
        print(json.dumps(run(dpt, peak)))
