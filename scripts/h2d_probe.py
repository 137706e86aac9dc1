"""PCIe copy rates as the host-streamed e2e run issues them: pinned H2D of a 2 x 64 MB input as one
copy per plane, and as 8 / 16 chunk copies per plane on one stream, alone and with a concurrent D2H
of 64 MB in chunks on a second stream (device-event timed)."""
import torch

MB = 1 << 20
x = torch.empty(16 * MB, dtype=torch.uint32).pin_memory()
y = torch.empty(16 * MB, dtype=torch.uint32).pin_memory()
o = torch.empty(16 * MB, dtype=torch.uint32).pin_memory()
dx = torch.empty_like(x, device="cuda")
dy = torch.empty_like(y, device="cuda")
do = torch.empty_like(o, device="cuda")
h2d, d2h = torch.cuda.Stream(), torch.cuda.Stream()


def run(chunks, with_d2h, reps=5):
    n = x.numel() // chunks
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(h2d)
        d2h.wait_event(e0)
        for c in range(chunks):
            with torch.cuda.stream(h2d):
                dx[c * n:(c + 1) * n].copy_(x[c * n:(c + 1) * n], non_blocking=True)
                dy[c * n:(c + 1) * n].copy_(y[c * n:(c + 1) * n], non_blocking=True)
            if with_d2h:
                with torch.cuda.stream(d2h):
                    o[c * n:(c + 1) * n].copy_(do[c * n:(c + 1) * n], non_blocking=True)
        h2d.wait_stream(d2h)
        e1.record(h2d)
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best


for chunks in (1, 8, 16):
    for wd in (False, True):
        ms = run(chunks, wd)
        print(f"chunks {chunks:2d} d2h {'on ' if wd else 'off'}: {ms:.3f} ms, H2D {2 * x.nbytes / ms / 1e6:.1f} GB/s",
              flush=True)
