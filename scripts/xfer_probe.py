"""Host<->device transfer rates on the box: pageable vs pinned copies, and host memcpy
into pinned staging with 1..16 threads (the Backend host API's bottleneck)."""
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import torch

n = 16 << 20  # 64 MB of u32... use 16 MB chunks below
src = np.random.default_rng(0).integers(0, 2**32, (64 << 20) // 4, dtype=np.uint64).astype(np.uint32)
dev = torch.empty(src.size, dtype=torch.uint32, device="cuda")
pin = torch.empty(src.size, dtype=torch.uint32).pin_memory()
pin_np = pin.numpy()
B = src.nbytes


def t(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps


pageable = torch.from_numpy(src)
print("pageable H2D GB/s", B / t(lambda: dev.copy_(pageable, non_blocking=False)) / 1e9)
print("pinned   H2D GB/s", B / t(lambda: dev.copy_(pin, non_blocking=True)) / 1e9)
print("pageable D2H GB/s", B / t(lambda: pageable.copy_(dev)) / 1e9)
print("pinned   D2H GB/s", B / t(lambda: pin.copy_(dev, non_blocking=True)) / 1e9)
for th in (1, 2, 4, 8, 16):
    ex = ThreadPoolExecutor(th)
    parts = np.array_split(np.arange(src.size), th)

    def cp():
        list(ex.map(lambda p: np.copyto(pin_np[p[0]:p[-1] + 1], src[p[0]:p[-1] + 1]), parts))
    print(f"memcpy {th:2d} threads GB/s", B / t(cp) / 1e9)
