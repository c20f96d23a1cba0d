"""3D smoother on compressed class planes (BASELINE configs[4]): per plane
width W (0 = FP64 class planes), the leaf residual kernel time, its HBM
bytes, and the adaFAC-PI cycle rate.

usage: python tools/c5_planes.py [depth] [p] [widths, e.g. 0,2,4,8] [cycles]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2005_03606_b200 as lzb  # noqa: E402

depth = int(sys.argv[1]) if len(sys.argv) > 1 else 5
p = int(sys.argv[2]) if len(sys.argv) > 2 else 2
widths = [int(x) for x in sys.argv[3].split(",")] if len(sys.argv) > 3 else [0, 2, 3, 4, 5, 6, 7, 8]
cycles = int(sys.argv[4]) if len(sys.argv) > 4 else 3
ctx = lzb.default_context()
stream = torch.cuda.ExternalStream(ctx.solve_stream)
f = lzb.field3_grf(lzb.grf_table(1, 64, 0.05, 1.0))
N = 3 ** depth
out = []
for w in widths:
    G = lzb.Grid3(depth, f, delta_max=1e-8, fixed_p3=w, plane_width=w, ctx=ctx)
    G.assemble_fixed(p)
    G.init_cycle(solver="adafac-pi", omega=0.6, max_cycles=10 ** 6)
    G.step()
    tk = {k: G.time_kernel(i, 5) for k, i in (("uhat", lzb.TK_UHAT), ("residual", lzb.TK_RESIDUAL),
                                              ("restrict", lzb.TK_RESTRICT), ("jacobi", lzb.TK_JACOBI),
                                              ("prolong", lzb.TK_PROLONG))}
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    reps = [G.step() for _ in range(cycles)]
    b.record(stream)
    b.synchronize()
    ms = a.elapsed_time(b) / cycles
    nv = (N + 1) ** 3
    res_bytes = nv * 40 + N ** 3 * G.leaf_bytes_per_cell()  # the TMA residual: no diagonal write
    out.append({"plane_width": w, "leaf_bytes_per_cell": G.leaf_bytes_per_cell(), "kernel_ms": tk,
                "residual_GBs": res_bytes / tk["residual"] / 1e6, "ms_per_cycle": ms,
                "dof_updates_per_s": (N - 1) ** 3 / (ms * 1e-3), "normalized": reps[-1]["normalized"]})
    print(json.dumps(out[-1]), flush=True)
    G.close()
    del G
    torch.cuda.empty_cache()
