"""Summarise the ncu --set full raw CSVs of the pass kernels (tools/ncu_round.sh)
into profiles/r01_ncu_pass_summary.json and profiles/traffic.json."""
import csv
import glob
import json
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
want = {"gpu__time_duration.sum": "duration_us", "dram__bytes_read.sum": "dram_read_bytes",
        "dram__bytes_write.sum": "dram_write_bytes", "launch__grid_size": "grid",
        "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active": "tensor_pipe_active_pct",
        "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_elapsed": "tensor_pipe_elapsed_pct"}
scale = {"Mbyte": 1e6, "Gbyte": 1e9, "Kbyte": 1e3, "byte": 1.0, "ms": 1e3, "us": 1.0, "ns": 1e-3}
out = {}
for f in sorted(glob.glob(os.path.join(ROOT, "gpurun_out", "ncu_pass_*_raw.csv"))):
    tag = re.sub(r"^ncu_pass_|_raw\.csv$", "", os.path.basename(f))
    rows = list(csv.reader(open(f)))
    if len(rows) < 3:
        continue
    hdr, units, vals = rows[0], rows[1], rows[2]
    d = {"kernel": vals[hdr.index("Kernel Name")]}
    for i, h in enumerate(hdr):
        if h in want:
            v = float(vals[i].replace(",", ""))
            if want[h].endswith("bytes") or want[h] == "duration_us":
                v *= scale.get(units[i], 1.0)
            d[want[h]] = v
    out[tag] = d
json.dump(out, open(os.path.join(ROOT, "profiles", "r01_ncu_pass_summary.json"), "w"), indent=1)
traffic = {t.split("_ta")[0]: {"pass_nn_dram_bytes": v["dram_read_bytes"] + v["dram_write_bytes"],
                               "source": f"ncu --set full, {v['kernel'].split('(')[0]}, gpurun_out/ncu_pass_{t}_raw.csv"}
           for t, v in out.items() if t.endswith("ta0")}
json.dump(traffic, open(os.path.join(ROOT, "profiles", "traffic.json"), "w"), indent=1)
print(json.dumps(out, indent=1))
