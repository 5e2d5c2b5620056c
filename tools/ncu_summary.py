"""Summarise ncu reports into JSON (dev tool; runs where the .ncu-rep files are):
key throughput metrics with DRAM bytes normalised to bytes, and the top stall reasons.
  python tools/ncu_summary.py out.json rep1.ncu-rep [rep2.ncu-rep ...]"""
import csv
import json
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "sm__cycles_elapsed.avg", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct", "dram__bytes_read.sum",
        "dram__bytes_write.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__occupancy_limit_shared_mem", "launch__occupancy_limit_registers"]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "nsecond": 1e-6, "usecond": 1e-3,
         "msecond": 1.0, "second": 1e3}

out = {}
for rep in sys.argv[2:]:
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(raw.splitlines()))
    h, units, v = r[0], r[1], r[2]
    d = {}
    for i, k in enumerate(h):
        if k in KEYS or k == "Kernel Name":
            val = v[i]
            try:
                x = float(val.replace(",", ""))
                u = units[i]
                if k.startswith("dram__bytes"):
                    x *= SCALE.get(u, 1)
                elif k == "gpu__time_duration.sum":
                    x *= SCALE.get(u, 1)   # -> ms
                val = x
            except ValueError:
                pass
            d[k] = val
    st = {}
    for i, k in enumerate(h):
        if k.startswith("smsp__average_warp_latency_issue_stalled") and k.endswith("ratio"):
            try:
                st[k.replace("smsp__average_warp_latency_issue_stalled_", "").replace("_per_warp_active.ratio", "")] = float(v[i])
            except ValueError:
                pass
    d["top_stalls"] = dict(sorted(st.items(), key=lambda x: -x[1])[:8])
    d["dram_bytes_total"] = d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0)
    out[rep.split("/")[-1].replace(".ncu-rep", "")] = d
json.dump(out, open(sys.argv[1], "w"), indent=1)
print(json.dumps(out, indent=1)[:3000])
