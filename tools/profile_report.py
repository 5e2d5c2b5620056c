"""Write a markdown summary of ncu reports into profiles/ (kernel metrics that
back the bench roofline and the DESIGN.md claims).

  python tools/profile_report.py OUT.md REPORT.ncu-rep [...]
"""
import csv
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration (ms)"),
    ("sm__cycles_elapsed.avg", "SM cycles"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor pipe active % (elapsed)"),
    ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "XU (MUFU) pipe %"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe %"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 throughput %"),
    ("dram__bytes_read.sum", "DRAM read (MB)"),
    ("dram__bytes_write.sum", "DRAM write (MB)"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
]


def summary(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hdr, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        out.append((d.get("Kernel Name", "?"), [(lab, d.get(k, ""), u.get(k, "")) for k, lab in KEYS]))
    return out


def main():
    out, reps = sys.argv[1], sys.argv[2:]
    lines = []
    for rep in reps:
        for name, vals in summary(rep):
            lines.append(f"### `{name[:110]}`\n\nsource: `{rep}`\n")
            lines.append("| metric | value | unit |\n|---|---|---|")
            for lab, v, u in vals:
                lines.append(f"| {lab} | {v} | {u} |")
            lines.append("")
    with open(out, "a") as f:
        f.write("\n".join(lines) + "\n")


if __name__ == "__main__":
    main()
