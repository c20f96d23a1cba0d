"""Key metrics + top stall reasons of `ncu --page raw --csv` exports."""
import csv
import sys

WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "l1tex__throughput.avg.pct_of_peak_sustained_active", "lts__t_bytes.sum", "launch__grid_size",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "launch__occupancy_limit_registers",
        "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct"]
for path in sys.argv[1:]:
    rows = list(csv.reader(open(path)))
    hdr, units, vals = rows[0], rows[1], rows[2:]
    for v in vals:
        print(path.split("/")[-1], v[hdr.index("Kernel Name")][:60])
        for w in WANT:
            if w in hdr:
                print(f"  {w} = {v[hdr.index(w)]} {units[hdr.index(w)]}")
        st = [i for i, h in enumerate(hdr) if h.startswith("smsp__pcsamp_warps_issue_stalled") and not h.endswith("not_issued")]
        pairs = sorted(((float(v[i].replace(",", "") or 0), hdr[i].replace("smsp__pcsamp_warps_issue_stalled_", ""))
                        for i in st if v[i] not in ("", "n/a")), reverse=True)[:6]
        print("  stalls:", pairs)
