"""Device time per cycle of the 729^2 grid (BASELINE configs[1] smoother:
adaFAC-PI, omega 0.6, p = 32 operators), CUDA events on the solve stream.
LZB_NO_PDL=1 / LZB_NO_GRAPHS=1 switch off programmatic dependent launch / the
CUDA graphs for comparison; LZB_SMALL_MAXN=9 keeps only levels up to 9^2 in the
cluster kernels (the round-1 fusion).

usage: python tools/cycle_probe.py [depth] [cycles]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2005_03606_b200 as lzb  # noqa: E402

depth = int(sys.argv[1]) if len(sys.argv) > 1 else 6
cycles = int(sys.argv[2]) if len(sys.argv) > 2 else 20
ctx = lzb.default_context()
stream = torch.cuda.ExternalStream(ctx.solve_stream)
d = lzb.make_desc(depth=depth, field=lzb.field_sinusoid(0.9, 6.0), solver="adafac-pi", omega=0.6,
                  rhs_kind="sinprod", max_cycles=10 ** 6, delta_max=1e-8)
g = lzb.Grid(d, 1)
g.assemble_fixed(32)
for _ in range(12):  # the Galerkin hierarchy settles one level per cycle; then the settled cycles
    g.step()
l0 = lzb.launch_count()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record(stream)
for _ in range(cycles):
    r = g.step()
b.record(stream)
b.synchronize()
print(f"depth {depth}: {a.elapsed_time(b) / cycles * 1e3:.1f} us per cycle, {(lzb.launch_count() - l0) / cycles:.0f} "
      f"launches per cycle, normalized {r['normalized']:.3e}")
