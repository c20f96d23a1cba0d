"""Time-to-solution probe on the 729^2 config-2 problem: eager (assemble first)
vs delayed/concurrent (anarchic on the side stream)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2005_03606_b200 as lzb  # noqa: E402

f = lzb.field_sinusoid(0.9, 6.0)
for solver, omega in (("adafac-pi", 0.6), ("adafac-pi", 0.6)):  # second pass: modules and graphs warm
    for mode, conc in (("eager", False), ("anarchic", True), ("anarchic", False)):
        d = lzb.make_desc(depth=6, field=f, solver=solver, omega=omega, rhs_kind="sinprod", assembly=mode,
                          schedule="double", n_max=32, max_cycles=3000, concurrent=conc, integration="exact")
        g = lzb.Grid(d, 42)
        t0 = time.perf_counter()
        reps = g.run(cap=4000)
        dt = time.perf_counter() - t0
        r = reps[-1]
        print(f"{solver:10s} w={omega} {mode:8s} conc={conc!s:5s} cycles={len(reps):5d} status={r['status']} "
              f"norm={r['normalized']:.2e} max_n={r['max_n']} avg_n={r['avg_n']:.2f} t={dt:.3f}s "
              f"factor={r['factor_totals']:.2f}", flush=True)
