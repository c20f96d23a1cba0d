"""Per-kernel HBM roofline of the cycle and stream-pack kernels on large 2D grids.

usage: python tools/smoother_roofline.py [depth ...]   (default 7 8)
Algorithmic bytes per launch are the DESIGN.md §4 figures (unique bytes a
perfect-cache kernel must move); times are lzb_grid_time_kernel (CUDA events
on the solve stream, back-to-back launches of one kernel).
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2005_03606_b200 as lzb  # noqa: E402


def algorithmic_bytes(depth, image_bytes, stats):
    N = 3 ** depth
    nc, nv = N * N, (N + 1) ** 2
    Nc = N // 3
    nvc = (Nc + 1) ** 2
    return {
        lzb.TK_UHAT: nv * 16 + nvc * 8,
        lzb.TK_RESIDUAL: nv * 48 + nc * (128 + 4),
        lzb.TK_RESTRICT: nv * 8 + nvc * 8,
        lzb.TK_JACOBI: nv * 32,
        lzb.TK_PROLONG: nv * 16 + nvc * 16,
        # per record: p1 + p3 + p2 + offset (14 B), the stored operator when
        # it has a payload, and the image bytes written
        lzb.TK_PACK: stats["cells_total"] * 14 + stats["payload_cells"] * 128 + image_bytes,
    }


def run(depth, peak):
    f = lzb.field_sinusoid(0.9, 6.0)
    d = lzb.make_desc(depth=depth, field=f, solver="adafac-pi", omega=0.6, rhs_kind="sinprod", max_cycles=100,
                      delta_max=1e-8, integration="fast")
    g = lzb.Grid(d, 1)
    g.assemble_fixed(4)
    for _ in range(2):
        g.step()
    st = g.stats()
    total_cells = sum(9 ** l for l in range(depth + 1))
    payload = st.fine_cells - st.p3_histogram[0]
    img = g.stream_image_size()
    ab = algorithmic_bytes(depth, img, {"cells_total": total_cells, "payload_cells": payload})
    names = {lzb.TK_UHAT: "k_uhat", lzb.TK_RESIDUAL: "k_residual", lzb.TK_RESTRICT: "k_restrict",
             lzb.TK_JACOBI: "k_jacobi", lzb.TK_PROLONG: "k_prolong", lzb.TK_PACK: "k_pack_groups"}
    out = {"depth": depth, "N": 3 ** depth, "image_bytes": img, "kernels": {}}
    for tk, name in names.items():
        ms = g.time_kernel(tk, 10)
        gbs = ab[tk] / (ms * 1e-3) / 1e9
        out["kernels"][name] = {"ms": round(ms, 4), "bytes": ab[tk], "GB/s": round(gbs, 1),
                                "frac": round(gbs / peak, 3)}
    for tk, name in ((lzb.TK_FRONT, "front_graph"), (lzb.TK_BACK, "back_graph")):
        out["kernels"][name] = {"ms": round(g.time_kernel(tk, 5), 4)}
    g.close()
    return out


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
