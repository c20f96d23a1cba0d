"""LZB_TRACE=1 breakdown of the eager ladder (eager_setup) of BASELINE configs[1]."""
import os
import sys
import time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2005_03606_b200 as lzb  # noqa: E402
f = lzb.field_sinusoid(0.9, 6.0)
for rnd in range(2):
    d = lzb.make_desc(depth=6, field=f, delta_max=1e-8, solver="adafac-pi", omega=0.6, assembly="eager",
                      rhs_kind="sinprod", schedule="double", n_max=32, termination_c=0.0, target=1e-10,
                      max_cycles=3, concurrent=False, integration="exact")
    g = lzb.Grid(d, 42)
    t0 = time.perf_counter()
    g.run(cap=10)
    print(f"pass {rnd}: {1e3 * (time.perf_counter() - t0):.2f} ms", flush=True)
    g.close()
