"""Device time of the fixed-p assembly step of bench.py (BASELINE configs[1]:
729^2, sinusoid eps, p = 32), EXACT and FAST, CUDA events on the solve stream.

usage: python tools/asm_probe.py [reps]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2005_03606_b200 as lzb  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
ctx = lzb.default_context()
stream = torch.cuda.ExternalStream(ctx.solve_stream)
for integ in ("exact", "fast"):
    d = lzb.make_desc(depth=6, field=lzb.field_sinusoid(0.9, 6.0), solver="additive", omega=0.6,
                      delta_max=1e-8, integration=integ)
    g = lzb.Grid(d, 1)
    for _ in range(3):
        g.assemble_fixed(32)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for _ in range(reps):
        g.assemble_fixed(32)
    b.record(stream)
    b.synchronize()
    ms = a.elapsed_time(b) / reps
    print(f"{integ}: {ms:.4f} ms per step, {531441 * 1024 / (ms * 1e-3) / 1e9:.1f} G sub-samples/s")
