"""Time-to-solution probe on BASELINE configs[1] (729^2 sinusoid, adaFAC-PI to
1e-10) with bench.py's settings: eager (p = 32 assembled first) vs the delayed
ladder 1 -> 32 from the geometric stencil, deterministic and concurrent.
LZB_NO_DEVLOOP=1 keeps the host cycle loop (one norm round trip per cycle)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2005_03606_b200 as lzb  # noqa: E402

f = lzb.field_sinusoid(0.9, 6.0)
for rnd in range(2):  # second pass: modules warm
    for mode, conc, geo in (("eager", False, False), ("anarchic", False, True), ("anarchic", True, True)):
        d = lzb.make_desc(depth=6, field=f, delta_max=1e-8, solver="adafac-pi", omega=0.6, assembly=mode,
                          rhs_kind="sinprod", schedule="double", n_max=32, termination_c=0.0, target=1e-10,
                          max_cycles=2000, concurrent=conc, integration="exact", start_geometric=geo)
        g = lzb.Grid(d, 42)
        l0 = lzb.launch_count()
        t0 = time.perf_counter()
        reps = g.run(cap=2100)
        dt = time.perf_counter() - t0
        r = reps[-1]
        print(f"pass {rnd} {mode:8s} conc={conc!s:5s} cycles={len(reps):4d} status={r['status']} "
              f"norm={r['normalized']:.3e} max_n={r['max_n']} t={1e3 * dt:.2f} ms "
              f"launches={lzb.launch_count() - l0} last-cycle wall={1e6 * r['wall_seconds']:.1f} us", flush=True)
        g.close()
