"""Summarise an ncu launch list (gpu__time_duration per launch, from
tools/profile_launches.sh) into profiles/<tag>_launches.{md,csv}.

usage: python tools/summarize_launches.py <tag> <launches.csv> [command]
"""
import collections
import csv
import os
import sys

tag, path = sys.argv[1], sys.argv[2]
cmd = sys.argv[3] if len(sys.argv) > 3 else "python bench.py --steps 3 --warmup 3 --no-cpu-baseline"
out_dir = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles")
rows = list(csv.reader(open(path)))
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h, data = rows[hi], rows[hi + 1:]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "second": 1e6, "s": 1e6}
tot = collections.defaultdict(lambda: [0, 0.0])
seq = []
for r in data:
    if len(r) <= vi:
        continue
    name = r[ki].split("(")[0]
    for junk in ("void ", "lzb::<unnamed>::", "(anonymous namespace)::", "unnamed>::", "lzb::"):
        name = name.replace(junk, "")
    name = name[:60] if name.startswith("cub") else name.split("<")[0].strip()
    v = float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
    tot[name][0] += 1
    tot[name][1] += v
    seq.append((name, v))
grand = sum(t for _, t in tot.values())
lines = [f"# {tag}: ncu launch list of `{cmd}` (gpu__time_duration, --clock-control none; cold-cache, "
         "serialised: shares only)", "",
         f"source: `{os.path.basename(path)}` ({len(seq)} launches, {grand / 1e3:.1f} ms total)", "",
         "| kernel | launches | total ms | share | avg us |", "|---|---|---|---|---|"]
for name, (n, t) in sorted(tot.items(), key=lambda x: -x[1][1])[:50]:
    lines.append(f"| `{name}` | {n} | {t / 1e3:.2f} | {100 * t / grand:.1f}% | {t / n:.1f} |")
open(os.path.join(out_dir, f"{tag}_launches.md"), "w").write("\n".join(lines) + "\n")
with open(os.path.join(out_dir, f"{tag}_launches.csv"), "w") as f:
    f.write("kernel,duration_us\n")
    for name, v in seq:
        f.write(f"{name},{v:.3f}\n")
print("\n".join(lines[:25]))
