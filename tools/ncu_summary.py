"""Summarise an ncu --set full report (raw page CSV on stdin) into profiles/*.json."""
import csv
import json
import sys

rows = list(csv.reader(sys.stdin))
h = rows[0]
units = rows[1]
mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}
out = {}
for r in rows[2:]:
    d = dict(zip(h, r))
    name = d["Kernel Name"].split("(")[0].replace("void ", "")

    def f(k):
        try:
            return float(d[k].replace(",", "")) * mult.get(units[h.index(k)], 1)
        except (KeyError, ValueError):
            return None

    out[name] = {k2: f(k) for k2, k in {
        "dram_read_bytes": "dram__bytes_read.sum", "dram_write_bytes": "dram__bytes_write.sum",
        "duration": "gpu__time_duration.sum", "dram_throughput_pct": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm_throughput_pct": "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
        "registers_per_thread": "launch__registers_per_thread",
        "issue_active_pct": "sm__inst_issued.avg.pct_of_peak_sustained_active",
        "fp64_pipe_active_pct": "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "l1_hit_pct": "l1tex__t_sector_hit_rate.pct", "l2_hit_pct": "lts__t_sector_hit_rate.pct"}.items()}
    out[name]["duration_unit"] = units[h.index("gpu__time_duration.sum")] if "gpu__time_duration.sum" in h else None
json.dump(out, open(sys.argv[1], "w"), indent=1)
traffic = {}
for k, v in out.items():
    fam = None
    for key, nm in (("k_batch_fwd", "batch_fwd"), ("k_batch_bwd", "batch_bwd"), ("k_plane_fwd", "plane_fwd"),
                    ("k_plane_bwd", "plane_bwd")):
        if key in k:
            fam = nm
    if fam and v["dram_read_bytes"] is not None:
        traffic[fam] = v["dram_read_bytes"] + v["dram_write_bytes"]
if len(sys.argv) > 2:
    json.dump(traffic, open(sys.argv[2], "w"), indent=1)
for k, v in out.items():
    print(k, {a: (round(b, 3) if isinstance(b, float) else b) for a, b in v.items()})
print("traffic per launch:", traffic)
