"""Assembly-pass time vs n (fixed cost = intercept) for both integration paths."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2005_03606_b200 as lzb  # noqa: E402

ctx = lzb.default_context()
stream = torch.cuda.ExternalStream(ctx.solve_stream)
f = lzb.field_sinusoid(0.9, 6.0)
for mode in ("exact", "fast"):
    d = lzb.make_desc(depth=6, field=f, integration=mode)
    g = lzb.Grid(d, 1)
    row = []
    for n in (1, 2, 4, 8, 16, 32, 64):
        g.assemble_fixed(n)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(5):
            g.assemble_fixed(n)
        b.record(stream)
        b.synchronize()
        ms = a.elapsed_time(b) / 5
        row.append(f"n={n}:{ms:.3f}ms({531441 * n * n / ms / 1e9:.0f}G/s)")
    print(mode, " ".join(row))
# cycle breakdown
d = lzb.make_desc(depth=6, field=f, solver="additive", omega=0.6, rhs_kind="sinprod", max_cycles=100)
g = lzb.Grid(d, 1)
g.assemble_fixed(4)
for name, which in (("assembly_pass", 0), ("residual_pass", 1), ("update", 2), ("prolong", 3), ("inject", 4)):
    g.pass_(which)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for _ in range(5):
        g.pass_(which)
    b.record(stream)
    b.synchronize()
    print(name, f"{a.elapsed_time(b) / 5:.3f} ms")
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
g.step()
a.record(stream)
for _ in range(5):
    g.step()
b.record(stream)
b.synchronize()
print("step", f"{a.elapsed_time(b) / 5:.3f} ms")
