"""Parse the LSTM tensor-core kernel's CTA-0 event trace (ELMRNN_TRACE=file).
kinds: 1 MMA step start, 3 MMA chunk issued (all K-slices), 4 epilogue got acc (chunk),
5 epilogue chunk done, 6 epilogue step done.  Prints median per-step / per-chunk gaps."""
import sys, numpy as np
d = np.loadtxt(sys.argv[1], delimiter=',', skiprows=1, dtype=np.int64)
kind, step, chunk, clk = d[:, 0], d[:, 1], d[:, 2], d[:, 3]
clk = np.unwrap(clk.astype(np.float64), period=2**32)   # 32-bit clock wrap
ev = {}
for k, s, c, t in zip(kind, step, chunk, clk):
    ev.setdefault((k, s, c), t)
mma_start = {s: t for (k, s, c), t in ev.items() if k == 1}
steps = sorted(mma_start)
dur = np.diff([mma_start[s] for s in steps])
print(f"steps traced {len(steps)}, median cycles per step {np.median(dur):.0f}")
# per chunk: MMA issued -> epilogue got acc; epilogue chunk time
NCH = max(c for (k, s, c) in ev if k == 3) + 1
got, done, iss = [], [], []
for (k, s, c), t in ev.items():
    if k == 4 and (5, s, c) in ev:
        done.append(ev[(5, s, c)] - t)
iss = []
for s in steps[1:-1]:
    ts = [ev.get((3, s, c)) for c in range(NCH)]
    if None not in ts:
        iss.append(np.diff([mma_start[s]] + ts))
iss = np.array(iss)
print("median MMA issue time per chunk (cycles):", np.median(iss, axis=0).round())
print(f"median epilogue chunk time {np.median(done):.0f} cycles; tensor time per chunk at 64 cyc/MMA: "
      f"{12 * 4 * 64 if NCH == 8 else 12 * 2 * 64}")
# epilogue step end vs next MMA step start (bubble)
bub = []
for s in steps[:-1]:
    e6 = [t for (k, s2, c), t in ev.items() if k == 6 and s2 == s + 1]
    if e6 and (s + 1) in mma_start:
        pass
last_chunk_epi_to_next = []
for s in steps[1:-1]:
    a = ev.get((3, s, NCH - 1)); b = mma_start.get(s + 1)
    if a is not None and b is not None:
        last_chunk_epi_to_next.append(b - a)
print(f"median gap last-chunk-issued -> next step MMA start {np.median(last_chunk_epi_to_next):.0f} cycles")
