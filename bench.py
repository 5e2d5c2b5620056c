#!/usr/bin/env python
"""bench.py -- ELM-RNN training throughput (H build + QR solve) on B200.

One "step" = one pass of the whole hot path over the workload: build H(Q)
(Alg. 1 line 2) and solve beta by fp64 Householder TSQR (S4.2,
P:327-328); for N > 1 GPUs rows are sharded, each rank factors its block,
the packed R factors are all-gathered over NCCL, rank 0 merges and solves,
and beta is broadcast.  Default workload: BASELINE.json configs[3] (C4, LSTM
N = 4M, Q = 50, M = 256), the one the headline metric is quoted on.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C4] [--impl reference]

Prints ONE JSON line on rank 0 (contract in DESIGN.md "Measurement").
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from synth import series as sy  # noqa: E402

METRIC = "ELM-RNN train samples/s (H build+QR solve)"
UNIT = "samples/s"

WORKLOAD_NAMES = {
    "C1": "C1 Elman N=1000 Q=10 M=20 d=1, Mackey-Glass",
    "C2j": "C2 Jordan (teacher forced) N=100k Q=20 M=64 d=1, AR(5)",
    "C2n": "C2 NARMAX (teacher forced) N=100k Q=20 M=64 d=1, AR(5)",
    "C3fc": "C3 fully connected (Q lags) N=1M Q=30 M=128 d=4, sinusoid mixture",
    "C3gru": "C3 GRU N=1M Q=30 M=128 d=4, sinusoid mixture",
    "C4": "C4 LSTM N=4M Q=50 M=256 d=1, Mackey-Glass + noise",
    "C3lstm_diag": "C3 shape, LSTM with diagonal U (paper-literal per-cell) N=1M Q=30 M=128 d=4",
    "C3gru_diag": "C3 shape, GRU with diagonal U (paper-literal per-cell) N=1M Q=30 M=128 d=4",
    "C3fc_eq8": "C3 shape, fully connected by the letter of Eq. 8 (per-cell) N=1M Q=30 M=128 d=4",
    "C2n_ef": "C2 NARMAX with error feedback (two passes: e = y - yhat(beta0), rebuild, re-solve) N=100k Q=20 M=64",
    "C5lstm1024": "C5 LSTM M=1024 Q=10 d=1, one GPU's share (N=2M of 16M), Mackey-Glass + noise",
    "C5gru1024": "C5 GRU M=1024 Q=10 d=1, one GPU's share (N=2M of 16M), Mackey-Glass + noise",
}
for _k, _c in sy.CONFIGS.items():
    if _k not in WORKLOAD_NAMES:
        WORKLOAD_NAMES[_k] = (f"C5 {_c['arch'].upper()} M={_c['M']} Q={_c['Q']} d=1, one GPU's share "
                              f"(N=2M of 16M), Mackey-Glass + noise")


def algorithmic_flops_per_sample(arch: str, S: int, M: int, Q: int) -> float:
    """Minimal exact work for H(Q), FMA = 2."""
    if arch in ("elman", "fc_eq8"):   # Eq. 8 after the per-lag column sums (init) is Eq. 5
        return 2 * S * M * Q + M * Q * (Q - 1)
    if arch == "lstm_diag":
        return Q * M * (8 * S + 8 + 6)
    if arch == "gru_diag":
        return Q * M * (6 * S + 6 + 5)
    if arch in ("jordan", "narmax"):
        return 2 * S * M + 2 * M * (Q - 1)
    if arch == "fc":
        return 2 * S * M * Q + M * M * Q * (Q - 1)
    if arch == "gru":
        return Q * (6 * S * M + 6 * M * M + 5 * M)
    return Q * (8 * S * M + 8 * M * M + 6 * M)


def algorithmic_bytes_per_sample(arch: str, S: int, M: int, Q: int) -> float:
    """HBM bytes of the build kernel: X window in, H(Q) row out (fp32)."""
    return 4 * Q * S + 4 * M


def qr_flops(M: int, N: int, nrhs: int = 1) -> float:
    """fp64 Householder TSQR of [H | Y]: 2 (M+P)^2 flop per row."""
    return 2.0 * N * (M + nrhs) ** 2


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d, "measured"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "sm_max_mhz": 1965.0}, \
        "fallback"


# ------------------------------------------------------------------- clocks
class ClockSampler:
    """Samples SM clock and throttle reasons of this rank's GPU via NVML."""
    REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown", 0x2: "applications_clocks_setting"}

    def __init__(self, device: int):
        self.samples, self.reasons, self.max_mhz, self.ok = [], 0, None, False
        try:
            import pynvml
            pynvml.nvmlInit()
            p = torch.cuda.get_device_properties(device)
            bus = f"{p.pci_domain_id:08X}:{p.pci_bus_id:02X}:{p.pci_device_id:02X}.0"
            try:
                self.h = pynvml.nvmlDeviceGetHandleByPciBusId(bus)
            except Exception:
                self.h = pynvml.nvmlDeviceGetHandleByIndex(device)
            self.nv = pynvml
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            pass
        self._stop = threading.Event()

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                self.reasons |= self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            except Exception:
                pass
            time.sleep(0.05)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.ok:
            self.t.join()

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unavailable"]}
        return {"sm_mhz": float(statistics.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(v for k, v in self.REASONS.items() if self.reasons & k)}


# ------------------------------------------------------------------- data
def make_inputs(cfg: str, N_total: int, rank: int, world: int):
    """Rank-local rows [lo, hi) of the workload (same seeded series on every rank)."""
    c = sy.CONFIGS[cfg]
    lo = N_total * rank // world
    hi = N_total * (rank + 1) // world
    s = sy.series(c["series"], N_total + c["Q"], noise=c["noise"])
    X, Y, Yfb = sy.windows(s[lo: hi + c["Q"]], hi - lo, c["Q"])
    return X, Y, Yfb


# ------------------------------------------------------------------- cpu baseline (oracle)
def cpu_oracle_rate(cfg: str, n_sub: int, X, Y, threads: int, weight_grid: int = 0):
    """Time the fp64 oracle (as it stands) on n_sub rows: H build + QR."""
    from oracle import oracle as orc
    c = sy.CONFIGS[cfg]
    net = orc.Net(c["arch"], S=c["S"], M=c["M"], Q=c["Q"], weight_grid=weight_grid)
    blocks = orc.gen_weights(net, 1)
    t0 = time.perf_counter()
    if c.get("mode") == "ef":
        orc.train_narmax_ef(net, blocks, X[:n_sub], Y[:n_sub], None, threads=threads)
    else:
        H = orc.build_H(net, blocks, X[:n_sub], threads=threads)
        orc.lstsq(H, Y[:n_sub])
    dt = time.perf_counter() - t0
    return n_sub / dt, dt


def oracle_sample_rows(cfg: str) -> int:
    c = sy.CONFIGS[cfg]
    f = algorithmic_flops_per_sample(c["arch"], c["S"], c["M"], c["Q"]) + 2 * (c["M"] + 1) ** 2
    # ~2 GFLOP/s per core of plain fp64 loops, all cores, aim at ~10 s
    rows = int(10.0 * 2.0e9 * max(1, os.cpu_count() or 1) / max(f, 1.0))
    return int(min(c["N"], max(2 * (c["M"] + 1), min(rows, 200_000))))


def run_reference(args, rank: int, world: int):
    """--impl reference: the oracle timed on host cores, rank 0 only."""
    if rank != 0:
        return
    cfg = args.config
    c = sy.CONFIGS[cfg]
    n = oracle_sample_rows(cfg) if args.n is None else min(args.n, oracle_sample_rows(cfg))
    n = max(n // 4, 2 * (c["M"] + 1))          # each step a bounded sample
    X, Y, _ = make_inputs(cfg, n, 0, 1)
    threads = os.cpu_count() or 1
    for _ in range(args.warmup):
        cpu_oracle_rate(cfg, n, X, Y, threads, args.weight_grid)
    times = [cpu_oracle_rate(cfg, n, X, Y, threads, args.weight_grid)[1] for _ in range(args.steps)]
    tot = sum(times)
    value = n * args.steps / tot
    sample = (f"{n} windows of {WORKLOAD_NAMES[cfg]} per step: fp64 oracle H build ({threads} threads, "
              f"OpenMP row split) + unblocked fp64 Householder QR (1 thread)")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": WORKLOAD_NAMES[cfg], "rows_per_step": n},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "oracle", "sample": sample,
                             "cpu_model": cpu_model()},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------- our arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C4", choices=sorted(sy.CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--n", type=int, default=None, help="override total rows (testing only)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--profile", action="store_true", help="short run for ncu (no baselines)")
    ap.add_argument("--force-path", type=int, default=0)
    ap.add_argument("--weight-grid", type=int, default=0, choices=[0, 1],
                    help="1: recurrent weights on the fp16 grid (SURVEY 8(c) '2xFP16 A-split'; 2-pass MMA)")
    ap.add_argument("--graph", choices=["auto", "on", "off"], default="auto",
                    help="replay the step as a CUDA graph (auto: configs whose step is launch-latency bound)")
    args = ap.parse_args()

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    import torch.distributed as dist
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    from paper_1911_13252_b200 import ELMRNN
    from paper_1911_13252_b200 import parallel as par

    cfg = args.config
    c = sy.CONFIGS[cfg]
    N_total = c["N"] if args.n is None else args.n
    X, Y, Yfb = make_inputs(cfg, N_total, rank, world)
    N_local = X.shape[0]
    Xh = torch.from_numpy(X).pin_memory()
    Yh = torch.from_numpy(Y).pin_memory()
    Xd = Xh.cuda()
    Yd = Yh.cuda()
    Hd = torch.empty((N_local, c["M"]), dtype=torch.float32, device="cuda")
    beta = torch.empty(c["M"], dtype=torch.float64, device="cuda")
    model = ELMRNN(c["arch"], c["S"], c["M"], c["Q"], seed=1, force_path=args.force_path,
                   weight_grid=args.weight_grid)
    stream = torch.cuda.current_stream()
    two_pass = c.get("mode") == "ef"
    if two_pass and world > 1:
        raise SystemExit("C2n_ef: the error windows cross shard boundaries; single GPU only")
    Ef = torch.empty((N_local, c["Q"]), dtype=torch.float32, device="cuda") if two_pass else None

    def step(ev_b0=None, ev_b1=None):
        if ev_b0 is not None:
            ev_b0.record(stream)
        model.build_H(Xd, None, Hd)
        if ev_b1 is not None:
            ev_b1.record(stream)
        if world == 1:
            model.solve_beta(Hd, Yd, beta, info=False)
        else:
            par.solve_sharded(model, Hd, Yd, N_total, beta)
        if two_pass:   # e = y - yhat(beta0), rebuild H with e, re-solve
            model.error_windows(Hd, Yd, beta, Ef)
            model.build_H(Xd, None, Hd, Ef=Ef)
            model.solve_beta(Hd, Yd, beta, info=False)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(max(args.warmup, 1 if args.profile else 3)):
        step()
    barrier()

    # ---- device-timed region (inputs resident in HBM; X and H exceed L2)
    K = args.steps
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    l0 = model.launch_count
    with ClockSampler(local) as clk:
        barrier()
        e0.record(stream)
        for k in range(K):
            step(*evs[k])
        e1.record(stream)
        barrier()
    launches = model.launch_count - l0
    ms = e0.elapsed_time(e1)
    build_ms = sum(a.elapsed_time(b) for a, b in evs) / K
    if world > 1:
        t = torch.tensor([ms, build_ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms, build_ms = float(t[0]), float(t[1])
    ms_step = ms / K
    ms_step_eager = ms_step

    # ---- small configs: inputs fit in L2 and the step is launch-latency bound.
    # Replay the step as one CUDA graph and flush L2 (write a
    # 256 MB buffer) between timed steps; each step is bracketed by its own events.
    small = (X.nbytes + N_local * c["M"] * 4) < 2 * 126 * 2**20
    use_graph = world == 1 and (args.graph == "on" or (args.graph == "auto" and small))
    graph = None
    if use_graph:
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            step()
        for _ in range(max(args.warmup, 3)):
            graph.replay()
        barrier()
    if small and world == 1:
        flush = torch.empty(256 * 2**20 // 4, dtype=torch.float32, device="cuda")
        pairs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
        with ClockSampler(local) as clk:
            barrier()
            for k in range(K):
                flush.fill_(float(k))
                pairs[k][0].record(stream)
                graph.replay() if graph is not None else step()
                pairs[k][1].record(stream)
            barrier()
        ms_step = sum(a.elapsed_time(b) for a, b in pairs) / K
    value = N_total / (ms_step / 1e3)

    # ---- end to end through the public API: host X/Y in, beta + rmse out
    e2e = None
    if not args.no_e2e and not args.profile:
        beta_h = torch.empty(c["M"], dtype=torch.float64).pin_memory()
        barrier()
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        cs = torch.cuda.Stream()
        # chunked copy/build overlap pays only when the copy is long; inputs under
        # 4 MiB (C1) take one copy and one launch
        e2e_chunks = 4 if Xh.numel() * 4 > 4 * 2**20 else 1

        def e2e_step():
            # public API from pinned host inputs: the X copy is chunked and
            # overlapped with the build (ELMRNN.build_H_from_host), Y rides along
            Yd.copy_(Yh, non_blocking=True)
            model.build_H_from_host(Xh, Xd, Hd, chunks=e2e_chunks, copy_stream=cs)
            if world == 1:
                model.solve_beta(Hd, Yd, beta, info=False)
            else:
                par.solve_sharded(model, Hd, Yd, N_total, beta)
            if two_pass:
                model.error_windows(Hd, Yd, beta, Ef)
                model.build_H(Xd, None, Hd, Ef=Ef)
                model.solve_beta(Hd, Yd, beta, info=False)
            beta_h.copy_(beta, non_blocking=True)
            stream.synchronize()

        e2e_step()   # untimed warm-up of the e2e path (side stream, events)
        barrier()
        t0.record(stream)
        for _ in range(K):
            e2e_step()
        t1.record(stream)
        barrier()
        ems = t0.elapsed_time(t1)
        if world > 1:
            t = torch.tensor([ems], dtype=torch.float64, device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ems = float(t[0])
        e2e = {"value": N_total / (ems / K / 1e3), "unit": UNIT,
               "h2d_bytes_per_step": int(Xh.numel() * 4 + Yh.numel() * 4),
               "d2h_bytes_per_step": int(beta_h.numel() * 8)}

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    peaks, src = load_peaks()
    flops = algorithmic_flops_per_sample(c["arch"], c["S"], c["M"], c["Q"]) * N_local
    path = model.path
    if c["arch"] in ("jordan", "narmax", "elman", "fc_eq8"):
        bound, unit = "hbm", "GB/s"
        achieved = algorithmic_bytes_per_sample(c["arch"], c["S"], c["M"], c["Q"]) * N_local / (build_ms / 1e3) / 1e9
        peak = peaks["hbm_gbs"]
        peak_note = f"{src} HBM copy bandwidth"
    elif path == 2:
        bound, unit = "tensor", "TFLOP/s"
        achieved = flops / (build_ms / 1e3) / 1e12
        passes = 2 if args.weight_grid == 1 else 3
        peak = peaks["bf16_tflops"] / passes
        peak_note = (f"{src} bf16 dense burst / {passes} ({passes}-pass fp16 split emulating fp32"
                     + (", fp16-grid weights)" if passes == 2 else ")"))
    else:
        bound, unit = "alu", "TFLOP/s"
        achieved = flops / (build_ms / 1e3) / 1e12
        peak = 148 * 128 * 2 * peaks.get("sm_max_mhz", 1965.0) * 1e6 / 1e12
        peak_note = "derived FP32 FFMA: 148 SMs x 128 lanes x 2 flop x sm_max_mhz"
    traffic = qr_traffic = None
    tf = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tf):
        tj = json.load(open(tf))
        traffic = tj.get(f"{cfg}:path{path}")
        qr_traffic = tj.get(f"{cfg}:qr")
    roof = {"bound": bound, "achieved": achieved, "peak": peak, "unit": unit, "frac": achieved / peak,
            "traffic": traffic, "kernel": "build_H", "kernel_ms": build_ms, "peak_source": peak_note}

    # ---- per-phase and overall fractions (the paper's Fig. 6 runtime
    # decomposition): lower bound of a phase = max over pipes of work / peak;
    # overall = sum of the phase bounds / measured step.  "burst" peaks: measured bf16
    # burst, derived FP32/FP64 at sm_max_mhz; "sustained": measured bf16 sustained,
    # derived FP32/FP64 at the median SM clock seen during the timed region.
    ck = clk.summary()
    mhz_max = float(peaks.get("sm_max_mhz", 1965.0))
    mhz_live = float(ck.get("sm_mhz") or mhz_max)
    hbm = peaks["hbm_gbs"] * 1e9
    passes = 2 if args.weight_grid == 1 else 3

    def lb_build(basis):
        f = flops
        by = algorithmic_bytes_per_sample(c["arch"], c["S"], c["M"], c["Q"]) * N_local
        mhz = mhz_max if basis == "burst" else mhz_live
        t = {"hbm": by / hbm}
        if path == 2 and c["arch"] in ("lstm", "gru", "fc"):
            tens = peaks["bf16_tflops" if basis == "burst" else "bf16_tflops_sustained"] * 1e12 / passes
            t["tensor"] = f / tens
        else:
            t["alu"] = f / (148 * 128 * 2 * mhz * 1e6)
        return t

    def lb_qr(basis):
        mhz = mhz_max if basis == "burst" else mhz_live
        return {"fp64": qr_flops(c["M"], N_local) / (148 * 64 * 2 * mhz * 1e6),
                "hbm": 4.0 * (c["M"] + 1) * N_local / hbm}

    reps = 2 if two_pass else 1   # C2n_ef: two builds and two solves per step
    phases = {}
    for name, fn, meas in (("build_H", lb_build, build_ms), ("solve", lb_qr, ms_step_eager - build_ms)):
        b, su = fn("burst"), fn("sustained")
        lb_b = reps * max(b.values()) * 1e3
        lb_s = reps * max(su.values()) * 1e3
        phases[name] = {"bound": max(b, key=b.get), "lb_ms_burst": lb_b, "lb_ms_sustained": lb_s, "ms": meas,
                        "frac_burst": lb_b / meas if meas > 0 else None,
                        "frac_sustained": lb_s / meas if meas > 0 else None}
    lb_tot_b = phases["build_H"]["lb_ms_burst"] + phases["solve"]["lb_ms_burst"]
    lb_tot_s = phases["build_H"]["lb_ms_sustained"] + phases["solve"]["lb_ms_sustained"]
    phases["overall"] = {"lb_ms_burst": lb_tot_b, "lb_ms_sustained": lb_tot_s, "ms": ms_step,
                         "frac_burst": lb_tot_b / ms_step, "frac_sustained": lb_tot_s / ms_step}
    roof["phases"] = phases
    roof["qr_traffic"] = qr_traffic
    roof["peaks_note"] = (f"tensor = {src} bf16 (burst {peaks['bf16_tflops']}, sustained "
                          f"{peaks.get('bf16_tflops_sustained')}) / {passes}; FP64 = 148 SMs x 64 FMA x 2 x clock "
                          f"({mhz_max:.0f} MHz burst, {mhz_live:.0f} MHz live); FP32 FFMA likewise x 128 lanes; "
                          f"HBM = {src} copy {peaks['hbm_gbs']} GB/s")

    cpu = None
    if not args.no_cpu_baseline and not args.profile and world == 1:
        n_sub = oracle_sample_rows(cfg)
        threads = os.cpu_count() or 1
        rate, dt = cpu_oracle_rate(cfg, n_sub, X, Y, threads, args.weight_grid)
        # single-thread figure on a smaller bounded sample (same per-row work)
        n1 = max(2 * (c["M"] + 1), n_sub // threads)
        rate1, dt1 = cpu_oracle_rate(cfg, n1, X, Y, 1, args.weight_grid)
        cpu = {"value": rate, "unit": UNIT, "cores": threads, "kind": "oracle",
               "sample": f"{n_sub} windows of the same workload, fp64 H build ({threads} threads, OpenMP row "
                         f"split) + unblocked fp64 Householder QR (1 thread), {dt:.1f} s; per-row work is "
                         f"independent of N, so the rate extrapolates linearly to the full N",
               "threads_1": {"value": rate1, "unit": UNIT, "cores": 1,
                             "sample": f"{n1} windows, H build and QR on 1 thread, {dt1:.1f} s"},
               "cpu_model": cpu_model(), "nproc": threads}

    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K, "warmup": args.warmup,
            "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f32+f64", "data": "synthetic",
            "config": {"workload": WORKLOAD_NAMES[cfg], "N_total": N_total, "rows_per_gpu": N_local,
                       "path": "tcgen05" if path == 2 else "fp32-fma", "weights": ("fp16 grid (weight_grid=1)" if args.weight_grid == 1 else "fp32 (grid 0)") + ", seed 1",
                       "qr": "fp64 Householder TSQR", "parallelism": f"dp{world} rows + all-gather R",
                       "l2": ("256 MB L2 flush between timed steps (inputs fit in L2)" if small and world == 1
                              else "no flush: X and H exceed the 126 MB L2"),
                       "cuda_graph": graph is not None,
                       "phases_ms": {"build_H": build_ms, "solve": ms_step_eager - build_ms,
                                     "step_eager": ms_step_eager}},
            "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
            "clocks": ck}
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
