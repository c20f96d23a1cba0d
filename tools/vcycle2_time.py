"""Device time per 2D V(1,1) cycle (BASELINE configs[0..1]): 243^2 checkerboard and 729^2 sinusoid.
LZB_PLAIN_VSMALL=1: the per-level launches on the small levels too."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2005_03606_b200 as lzb  # noqa: E402

ctx = lzb.default_context()
stream = torch.cuda.ExternalStream(ctx.solve_stream)
for depth, field, p in ((5, lzb.checkerboard(1, 8), 16), (6, lzb.field_sinusoid(0.9, 6.0), 32)):
    g = lzb.Grid(lzb.make_desc(depth=depth, field=field, solver="additive", omega=0.6, rhs_kind="sinprod",
                               max_cycles=10 ** 6), 42, ctx)
    g.assemble_fixed(p)
    for _ in range(3):
        g.vcycle(1)
    l0 = lzb.launch_count()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for _ in range(20):
        r = g.vcycle(1)
    b.record(stream)
    b.synchronize()
    print(f"depth {depth}: {a.elapsed_time(b) / 20 * 1e3:.1f} us per V(1,1) cycle, "
          f"{(lzb.launch_count() - l0) / 20:.0f} launches, normalized {r['normalized']:.3e}")
    g.close()
