"""Summarise an ncu launch list + a `--set full` report into profiles/<tag>_*.

usage: python tools/summarize_profiles.py <tag> <launches.csv | -> <full.ncu-rep | raw.csv>
(raw.csv: `ncu -i <rep> --page raw --csv`, written on the GPU box when the
report itself is too large to bring back)
Also merges the per-launch DRAM traffic of every captured kernel into
profiles/traffic.json (read by bench.py for roofline.traffic).
"""
import collections
import json
import csv
import io
import os
import subprocess
import sys

tag, launches, rep = sys.argv[1], sys.argv[2], sys.argv[3]
# optional: a suffix for the traffic.json keys (e.g. "@729^3" for a per-config capture)
key_suffix = sys.argv[4] if len(sys.argv) > 4 else ""
out_dir = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles")
rows = list(csv.reader(open(launches))) if launches != "-" else [["Kernel Name", "Metric Value", "Metric Unit"]]
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h, data = rows[hi], rows[hi + 1:]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
tot = collections.defaultdict(lambda: [0, 0.0])
seq = []
for r in data:
    if len(r) <= vi:
        continue
    name = r[ki].split("(")[0].replace("lzb::<unnamed>::", "").replace("(anonymous namespace)::", "")
    v = float(r[vi].replace(",", ""))
    v = v * {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "second": 1e6, "s": 1e6}.get(r[ui], 1.0)
    tot[name][0] += 1
    tot[name][1] += v
    seq.append((name, v))
grand = sum(t for _, t in tot.values())
lines = [f"# {tag}: ncu launch list (gpu__time_duration, --clock-control none; cold-cache, serialised)", "",
         f"source: `{os.path.basename(launches)}` ({len(seq)} launches, {grand:.1f} us total)", "",
         "| kernel | launches | total us | share | avg us |", "|---|---|---|---|---|"]
for name, (n, t) in sorted(tot.items(), key=lambda x: -x[1][1]):
    lines.append(f"| `{name}` | {n} | {t:.1f} | {100 * t / grand:.1f}% | {t / n:.1f} |")
if launches != "-":
    open(os.path.join(out_dir, f"{tag}_launches.md"), "w").write("\n".join(lines) + "\n")
    with open(os.path.join(out_dir, f"{tag}_launches.csv"), "w") as f:
        f.write("kernel,duration_us\n")
        for name, v in seq:
            f.write(f"{name},{v:.3f}\n")

raw = (open(rep).read() if rep.endswith(".csv") else
       subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout)
rr = list(csv.reader(io.StringIO(raw)))
hdr, units, vals = rr[0], rr[1], rr[2:]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__throughput.avg.pct_of_peak_sustained_active", "lts__t_bytes.sum"]
col = {w: hdr.index(w) for w in want if w in hdr}
kn = hdr.index("Kernel Name")
lines = [f"# {tag}: ncu --set full (selected metrics per captured launch)", "",
         f"source: `{os.path.basename(rep)}`", "",
         "| kernel | " + " | ".join(w.split(".")[0] + ("" if "pct" not in w else " %") for w in col) + " |",
         "|---|" + "---|" * len(col)]
for v in vals:
    name = v[kn].split("(")[0].replace("lzb::<unnamed>::", "").replace("(anonymous namespace)::", "")
    name = name.replace("void ", "").replace("unnamed>::", "").split("<")[0]
    cells = []
    for w, i in col.items():
        u = units[i]
        cells.append(f"{v[i]} {u}".strip())
    lines.append(f"| `{name}` | " + " | ".join(cells) + " |")
open(os.path.join(out_dir, f"{tag}_ncu_full.md"), "w").write("\n".join(lines) + "\n")
print("\n".join(lines))

# per-launch DRAM traffic (bytes) of each captured kernel, last capture wins
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
tpath = os.path.join(out_dir, "traffic.json")
traffic = json.load(open(tpath)) if os.path.exists(tpath) else {}
ir, iw = hdr.index("dram__bytes_read.sum"), hdr.index("dram__bytes_write.sum")
for v in vals:
    name = v[kn].split("(")[0].replace("void ", "").replace("lzb::<unnamed>::", "")
    name = name.replace("(anonymous namespace)::", "").replace("unnamed>::", "").split("<")[0].strip()
    b = float(v[ir].replace(",", "")) * scale.get(units[ir], 1) + float(v[iw].replace(",", "")) * scale.get(units[iw], 1)
    entry = {"dram_bytes_per_launch": b, "report": os.path.basename(rep), "tag": tag}
    for key, metric in (("fp64_pipe_active_pct", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
                        ("dram_throughput_pct", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
                        ("issue_active_pct", "smsp__issue_active.avg.pct_of_peak_sustained_active"),
                        ("duration_us", "gpu__time_duration.sum")):
        if metric in hdr:
            try:
                x = float(v[hdr.index(metric)].replace(",", ""))
                if key == "duration_us":
                    x *= {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "second": 1e6}.get(units[hdr.index(metric)], 1.0)
                entry[key] = x
            except ValueError:
                pass
    traffic[name + key_suffix] = entry
json.dump(traffic, open(tpath, "w"), indent=1, sort_keys=True)
