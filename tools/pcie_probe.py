"""Development aid (GPU box): pinned-memory copy rates, one direction at a time and both at
once, next to the box's NUMA layout -- the ceiling of bench.py's e2e figure."""
import subprocess
import time

import torch

print(subprocess.run("nvidia-smi topo -m | head -8; lscpu | grep -i -E 'numa|socket|model name|^CPU\\(s\\)'",
                     shell=True, capture_output=True, text=True).stdout)
n = 1 << 30  # 4 GiB of float32
h_in = torch.empty(n, dtype=torch.float32, pin_memory=True).fill_(1.0)
h_out = torch.empty(n, dtype=torch.float32, pin_memory=True)
d_a = torch.empty(n, dtype=torch.float32, device="cuda")
d_b = torch.empty(n, dtype=torch.float32, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
gb = n * 4 / 1e9


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps


def h2d():
    with torch.cuda.stream(s1):
        d_a.copy_(h_in, non_blocking=True)


def d2h():
    with torch.cuda.stream(s2):
        h_out.copy_(d_b, non_blocking=True)


def both():
    h2d()
    d2h()


for name, fn in (("H2D", h2d), ("D2H", d2h), ("both at once", both)):
    t = timed(fn)
    print(f"{name}: {gb / t:.1f} GB/s per direction ({1e3 * t:.1f} ms for {gb:.2f} GB each)")
