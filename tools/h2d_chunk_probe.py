"""Pinned H2D cost of the record upload (17 B/record, N = 10^6) as one copy
per array vs split into C chunks per array (the host-array pipeline's copy
pattern), timed with CUDA events on one stream.

    python tools/h2d_chunk_probe.py
"""
import torch

n = 1_000_000
pr = torch.zeros(n, dtype=torch.uint8).pin_memory()
lo = torch.zeros(n, dtype=torch.float64).pin_memory()
la = torch.zeros(n, dtype=torch.float64).pin_memory()
dpr, dlo, dla = (torch.empty_like(t, device="cuda") for t in (pr, lo, la))
s = torch.cuda.Stream()


def run(chunks, interleave=True, reps=50):
    b = [round(n * c / chunks) for c in range(chunks + 1)]
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(s):
        for it in range(reps + 3):
            if it == 3:
                e0.record(s)
            for c in range(chunks):
                sl = slice(b[c], b[c + 1])
                dpr[sl].copy_(pr[sl], non_blocking=True)
                dlo[sl].copy_(lo[sl], non_blocking=True)
                dla[sl].copy_(la[sl], non_blocking=True)
        e1.record(s)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    return ms, 17e6 / (ms / 1e3) / 1e9


for c in (1, 2, 4, 7, 8, 16, 32):
    ms, gbs = run(c)
    print(f"chunks={c:2d}: {ms * 1e3:7.1f} us per 17 MB upload ({gbs:5.1f} GB/s)", flush=True)
