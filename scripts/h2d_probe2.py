"""Pinned H2D of two 64 MB planes: both on one stream, or x and y on two streams (two copy engines),
8 chunks each, with and without a concurrent chunked D2H (device-event timed)."""
import torch

MB = 1 << 20
x = torch.empty(16 * MB, dtype=torch.uint32).pin_memory()
y = torch.empty(16 * MB, dtype=torch.uint32).pin_memory()
o = torch.empty(16 * MB, dtype=torch.uint32).pin_memory()
dx, dy, do = (torch.empty_like(t, device="cuda") for t in (x, y, o))
s1, s2, s3 = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()


def run(two, d2h, chunks=8, reps=5):
    n = x.numel() // chunks
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s1)
        s2.wait_event(e0)
        s3.wait_event(e0)
        for c in range(chunks):
            sl = slice(c * n, (c + 1) * n)
            with torch.cuda.stream(s1):
                dx[sl].copy_(x[sl], non_blocking=True)
            with torch.cuda.stream(s2 if two else s1):
                dy[sl].copy_(y[sl], non_blocking=True)
            if d2h:
                with torch.cuda.stream(s3):
                    o[sl].copy_(do[sl], non_blocking=True)
        s1.wait_stream(s2)
        s1.wait_stream(s3)
        e1.record(s1)
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best


for two in (False, True):
    for d2h in (False, True):
        ms = run(two, d2h)
        print(f"two streams {two!s:5s} d2h {d2h!s:5s}: {ms:.3f} ms, H2D {2 * x.nbytes / ms / 1e6:.1f} GB/s", flush=True)
