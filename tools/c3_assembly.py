"""C3 assembly throughput (BASELINE configs[2]): 243^3 cells, eps = exp(GRF)
(64^3 Fourier modes, ell = 0.05, sigma^2 = 1), p = 1..8 per axis; one step =
integrate + code + store every leaf record.

usage: python tools/c3_assembly.py [depth] [p ...]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2005_03606_b200 as lzb  # noqa: E402

depth = int(sys.argv[1]) if len(sys.argv) > 1 else 5
ps = [int(a) for a in sys.argv[2:]] or list(range(1, 9))
ctx = lzb.default_context()
stream = torch.cuda.ExternalStream(ctx.solve_stream)
g = lzb.grf_table(1, 64, 0.05, 1.0)
G = lzb.Grid3(depth, lzb.field3_grf(g), delta_max=1e-8, ctx=ctx)
nc = (3 ** depth) ** 3
for p in ps:
    G.assemble_fixed(p)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 3
    a.record(stream)
    for _ in range(reps):
        G.assemble_fixed(p)
    b.record(stream)
    b.synchronize()
    ms = a.elapsed_time(b) / reps
    st = G.stats()
    print(json.dumps({"p": p, "ms": ms, "sub_samples_per_s": nc * p ** 3 / (ms * 1e-3),
                      "cells_per_s": nc / (ms * 1e-3), "bytes_per_cell": st.fine_stored_bytes / nc,
                      "p3_hist": list(st.p3_histogram)}))
