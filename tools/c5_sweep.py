"""C5 sweep (BASELINE configs[4]) on one GPU: LSTM/GRU x M in {32,128,512,1024} x
Q in {10,50,100} at one GPU's share (2M rows), every H-builder path the shape
admits (--force-path 1 FP32-FMA, 2 tcgen05), one bench.py subprocess per point.
Prints one JSON line per point; dev tool (GPU box).
  python tools/c5_sweep.py [--steps 3] [--archs lstm,gru] [--ms 32,128,512,1024] [--qs 10,50,100]"""
import argparse
import json
import subprocess
import sys

ap = argparse.ArgumentParser()
ap.add_argument("--steps", type=int, default=3)
ap.add_argument("--archs", default="lstm,gru")
ap.add_argument("--ms", default="32,128,512,1024")
ap.add_argument("--qs", default="10,50,100")
ap.add_argument("--fma-max-m", type=int, default=128, help="largest M timed on the FP32-FMA path")
a = ap.parse_args()
for arch in a.archs.split(","):
    for M in map(int, a.ms.split(",")):
        for Q in map(int, a.qs.split(",")):
            paths = ([1] if M <= a.fma_max_m else []) + ([2] if M >= 128 else [])
            for fp in paths:
                cmd = [sys.executable, "bench.py", "--config", f"C5{arch}{M}q{Q}", "--force-path", str(fp),
                       "--steps", str(a.steps), "--warmup", "2", "--no-cpu-baseline", "--no-e2e"]
                r = subprocess.run(cmd, capture_output=True, text=True)
                try:
                    d = json.loads(r.stdout.strip().splitlines()[-1])
                    ph = d["config"]["phases_ms"]
                    out = {"arch": arch, "M": M, "Q": Q, "force_path": fp, "path": d["config"]["path"],
                           "samples_per_s": d["value"], "build_ms": ph["build_H"], "solve_ms": ph["solve"],
                           "frac_build": d["roofline"]["phases"]["build_H"]["frac_burst"],
                           "frac_solve": d["roofline"]["phases"]["solve"]["frac_burst"],
                           "frac_overall": d["roofline"]["phases"]["overall"]["frac_burst"],
                           "bound": d["roofline"]["phases"]["build_H"]["bound"], "sm_mhz": d["clocks"]["sm_mhz"]}
                except Exception:
                    out = {"arch": arch, "M": M, "Q": Q, "force_path": fp, "error": (r.stderr or r.stdout)[-300:]}
                print(json.dumps(out), flush=True)
