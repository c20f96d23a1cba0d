"""The e2e path of bench.py (BASELINE configs[1], p = 32: assembly + the LZMG
image into pinned host memory, after a few cycles so the refined records carry
payloads as in bench.py): the sequential calls against the pipelined
lzb_grid_assemble_stream (with its per-band device timeline), CUDA events on
the solve stream.

usage: python tools/e2e_probe.py [reps] [cycles before]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2005_03606_b200 as lzb  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
cyc = int(sys.argv[2]) if len(sys.argv) > 2 else 5
ctx = lzb.default_context()
stream = torch.cuda.ExternalStream(ctx.solve_stream)
d = lzb.make_desc(depth=6, field=lzb.field_sinusoid(0.9, 6.0), solver="adafac-pi", omega=0.6, max_cycles=100,
                  delta_max=1e-8)
g = lzb.Grid(d, 1)
g.assemble_fixed(32)
for _ in range(cyc):
    g.step()
img = g.stream_image()
print("image bytes", len(img))
host = torch.empty(len(img) + (1 << 20), dtype=torch.uint8, pin_memory=True).numpy()
tl = np.zeros(9, np.float32)
for label, fn in (("sequential", lambda: (g.assemble_fixed(32), g.stream_image(host))),
                  ("pipelined", lambda: g.assemble_stream(32, host, tl))):
    for i in range(reps):
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        fn()
        b.record(stream)
        b.synchronize()
        print(label, i, f"{a.elapsed_time(b):.3f} ms", flush=True)
print("band assembly ends", np.round(tl[:3], 3), "pack ends", np.round(tl[3:6], 3), "copy ends", np.round(tl[6:], 3))
