"""The 729^3 fused leaf update timed over 1..100 back-to-back launches, with the SM clock sampled (burst vs sustained)."""
import subprocess
import sys
import threading
import time

sys.path.insert(0, ".")
import paper_2005_03606_b200 as lzb  # noqa: E402

g = lzb.Grid3(6, lzb.field3_grf(lzb.grf_table(1, 64, 0.05, 1.0)), delta_max=1e-8)
g.assemble_fixed(2)
g.init_cycle(solver="adafac-pi", omega=0.6, max_cycles=10 ** 6)
g.step()
clk = []
stop = False


def sample():
    import pynvml
    pynvml.nvmlInit()
    h = pynvml.nvmlDeviceGetHandleByIndex(0)
    while not stop:
        clk.append((pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM), pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_MEM),
                    pynvml.nvmlDeviceGetPowerUsage(h) // 1000))
        time.sleep(0.02)


t = threading.Thread(target=sample)
t.start()
for tk, name in ((lzb.TK_BACK, "back"), (lzb.TK_UHAT, "uhat"), (lzb.TK_RESIDUAL, "residual")):
    for reps in (1, 1, 2, 5, 20, 100):
        time.sleep(0.5)
        n0 = len(clk)
        ms = g.time_kernel(tk, reps)
        c = clk[n0:] or clk[-1:]
        print(name, "reps", reps, "ms", round(ms, 4), "clocks(sm,mem,W) min", min(c), "max", max(c), flush=True)
stop = True
t.join()
