"""One ncu --set full raw CSV (`ncu -i X.ncu-rep --page raw --csv`) -> the fields kept in
profiles/r01_ncu_kernels_summary.json. Usage: ncu_kernel_summary.py TAG RAW_CSV [TAG RAW_CSV ...]
(merged into the JSON under each TAG)."""
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "profiles", "r01_ncu_kernels_summary.json")
want = {"gpu__time_duration.sum": "duration_us", "dram__bytes_read.sum": "dram_read_bytes",
        "dram__bytes_write.sum": "dram_write_bytes", "launch__grid_size": "grid", "launch__block_size": "block",
        "launch__registers_per_thread": "registers",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed": "memory_throughput_pct",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed": "dram_throughput_pct",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_throughput_pct",
        "sm__warps_active.avg.pct_of_peak_sustained_active": "achieved_occupancy_pct"}
scale = {"Mbyte": 1e6, "Gbyte": 1e9, "Kbyte": 1e3, "byte": 1.0, "ms": 1e3, "us": 1.0, "ns": 1e-3}
out = json.load(open(OUT)) if os.path.exists(OUT) else {}
args = sys.argv[1:]
for tag, f in zip(args[::2], args[1::2]):
    rows = list(csv.reader(open(f)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    d = {"kernel": vals[hdr.index("Kernel Name")]}
    stalls = {}
    for i, h in enumerate(hdr):
        try:
            v = float(vals[i].replace(",", ""))
        except ValueError:
            continue
        if h in want:
            if want[h].endswith("bytes") or want[h] == "duration_us":
                v *= scale.get(units[i], 1.0)
            d[want[h]] = v
        if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("_not_issued"):
            stalls[h[len("smsp__pcsamp_warps_issue_stalled_"):]] = v
    tot = sum(stalls.values()) or 1.0
    d["top_stalls_pct"] = {k: round(100 * v / tot, 1) for k, v in sorted(stalls.items(), key=lambda kv: -kv[1])[:5]}
    out[tag] = d
json.dump(out, open(OUT, "w"), indent=1)
print(json.dumps({t: out[t] for t in args[::2]}, indent=1))
