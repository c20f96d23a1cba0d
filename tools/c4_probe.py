"""Where the C4 delayed solve's time goes (BASELINE configs[3]: sphere tree,
re-refinement + shell re-assembly every 5 cycles): wall time per call."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2005_03606_b200 as lzb  # noqa: E402

t0 = time.perf_counter()
t4 = lzb.Tree3(4, 6, lzb.field3_sphere(), delta_max=1e-8)
print(f"create {time.perf_counter() - t0:.3f} s, leaves {t4.n_leaves}", flush=True)


def timed(name, fn):
    a = time.perf_counter()
    r = fn()
    print(f"  {name}: {1e3 * (time.perf_counter() - a):.1f} ms", flush=True)
    return r


timed("assemble(1)", lambda: t4.assemble(1))
timed("init_cycle", lambda: t4.init_cycle(solver="adafac-pi", omega=0.6, max_cycles=10 ** 6))
ladder = [2, 4, 8, 16]
T0 = time.perf_counter()
for k in range(25):
    if k % 5 == 0 and 0 < k // 5 <= len(ladder):
        e = k // 5
        timed(f"refine to {0.25 + 0.01 * e:.2f}", lambda: t4.refine(0.25 + 0.01 * e, ladder[e - 1]))
        timed("set_shell", lambda: t4.set_shell(0.01))
        timed(f"assemble_shell({ladder[e - 1]})", lambda: t4.assemble_shell(ladder[e - 1]))
        timed("refresh_ops", lambda: t4.refresh_ops())
    a = time.perf_counter()
    r = t4.step()
    if k % 5 == 1:
        print(f"  step {k}: {1e3 * (time.perf_counter() - a):.1f} ms, normalized {r['normalized']:.3e}", flush=True)
print(f"solve {time.perf_counter() - T0:.3f} s")
