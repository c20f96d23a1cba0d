"""Per-call time of the e2e path of bench.py (BASELINE configs[1], p = 32:
assemble_fixed + stream_image into pinned host memory), host wall clock and
CUDA events on the solve stream, with and without the L2 flush between calls.

usage: python tools/e2e_probe.py [reps]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2005_03606_b200 as lzb  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
ctx = lzb.default_context()
stream = torch.cuda.ExternalStream(ctx.solve_stream)
f = lzb.field_sinusoid(0.9, 6.0)
d = lzb.make_desc(depth=6, field=f, solver="adafac-pi", omega=0.6, max_cycles=100, delta_max=1e-8)
g = lzb.Grid(d, 1)
g.assemble_fixed(32)
img = g.stream_image()
host = torch.empty(len(img) + (1 << 20), dtype=torch.uint8, pin_memory=True).numpy()
flush = torch.empty(1 << 25, dtype=torch.float64, device="cuda")
for label, fn in (("assemble", lambda: g.assemble_fixed(32)), ("image", lambda: g.stream_image(host)),
                  ("both", lambda: (g.assemble_fixed(32), g.stream_image(host)))):
    for fl in (False, True):
        for i in range(reps):
            if fl:
                with torch.cuda.stream(stream):
                    flush.fill_(1.0)
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            t = time.perf_counter()
            a.record(stream)
            fn()
            b.record(stream)
            b.synchronize()
            print(label, "flush" if fl else "warm", i, f"wall {1e3 * (time.perf_counter() - t):.3f} ms",
                  f"events {a.elapsed_time(b):.3f} ms", flush=True)
