"""Summarise an ncu report: key throughput metrics + top SASS opcodes/stalls."""
import csv, collections, subprocess, sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(raw.splitlines()))
h, v = r[0], r[2] if len(r) > 2 else r[1]
d = dict(zip(h, v))
keys = ["Kernel Name", "gpu__time_duration.sum", "sm__cycles_elapsed.avg", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__t_bytes.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread"]
for k in keys:
    print(f"{k:75s} {d.get(k)}")
st = {k: float(v) for k, v in d.items() if k.startswith("smsp__average_warp_latency_issue_stalled") and k.endswith("ratio") and v}
for k, val in sorted(st.items(), key=lambda x: -x[1])[:10]:
    print(f"  stall {k.replace('smsp__average_warp_latency_issue_stalled_',''):50s} {val:.3f}")
