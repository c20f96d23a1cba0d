"""C3 cycles (BASELINE configs[2]): 243^3, eps = exp(GRF), p = 8 assembly,
then adaFAC-PI cycles; per-cycle time and fine DoF-updates/s.

usage: python tools/c3_cycle.py [depth] [p] [cycles]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2005_03606_b200 as lzb  # noqa: E402

depth = int(sys.argv[1]) if len(sys.argv) > 1 else 5
p = int(sys.argv[2]) if len(sys.argv) > 2 else 8
cycles = int(sys.argv[3]) if len(sys.argv) > 3 else 10
ctx = lzb.default_context()
stream = torch.cuda.ExternalStream(ctx.solve_stream)
G = lzb.Grid3(depth, lzb.field3_grf(lzb.grf_table(1, 64, 0.05, 1.0)), ctx=ctx)
G.assemble_fixed(p)
G.init_cycle(solver="adafac-pi", omega=0.6, max_cycles=10 ** 6)
G.step()  # coarse operators + first cycle
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record(stream)
reps = [G.step() for _ in range(cycles)]
b.record(stream)
b.synchronize()
ms = a.elapsed_time(b) / cycles
N = 3 ** depth
print(json.dumps({"depth": depth, "p": p, "cycles": cycles, "ms_per_cycle": ms,
                  "dof_updates_per_s": (N - 1) ** 3 / (ms * 1e-3),
                  "normalized": [r["normalized"] for r in reps]}))
