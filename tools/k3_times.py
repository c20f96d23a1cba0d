"""Per-kernel device times of the 3D leaf-level cycle kernels (CUDA events,
lzb_grid3_time_kernel) at 243^3 / 729^3 with their algorithmic HBM bytes."""
import json
import sys

sys.path.insert(0, ".")
import paper_2005_03606_b200 as lzb  # noqa: E402

peak = json.load(open("MEASURED_PEAKS.json")).get("hbm_gbs", 6446.6) if __import__("os").path.exists(
    "MEASURED_PEAKS.json") else 6446.6
for depth in [int(a) for a in (sys.argv[1:] or ["5", "6"])]:
    g = lzb.Grid3(depth, lzb.field3_grf(lzb.grf_table(1, 64, 0.05, 1.0)), delta_max=1e-8)
    g.assemble_fixed(2)
    g.init_cycle(solver="adafac-pi", omega=0.6, max_cycles=10 ** 6)
    g.step()
    N = 3 ** depth
    nv, nc, nvc = (N + 1) ** 3, N ** 3, (N // 3 + 1) ** 3
    rows = {"uhat": (lzb.TK_UHAT, 16 * nv), "residual": (lzb.TK_RESIDUAL, 40 * nv + 216 * nc),
            "restrict": (lzb.TK_RESTRICT, 8 * nv + 8 * nvc), "back(pre+update)": (lzb.TK_BACK, 32 * nv + 48 * nvc)}
    out = {}
    for name, (tk, b) in rows.items():
        ms = g.time_kernel(tk, 5)
        out[name] = {"ms": round(ms, 4), "GB/s": round(b / ms / 1e6, 1), "frac": round(b / ms / 1e6 / peak, 3)}
    print(json.dumps({"depth": depth, "kernels": out}))
    g.close()
