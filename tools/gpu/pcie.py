"""PCIe copy rates on the box: H2D alone, D2H alone, both at once (pinned host memory)."""
import time
import torch

n = 4 << 30  # 4 GiB per buffer
h_up = torch.empty(n, dtype=torch.uint8, pin_memory=True)
h_dn = torch.empty(n, dtype=torch.uint8, pin_memory=True)
d_up = torch.empty(n, dtype=torch.uint8, device="cuda")
d_dn = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=3):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        t = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t)
    return best


def up():
    with torch.cuda.stream(s1):
        d_up.copy_(h_up, non_blocking=True)


def dn():
    with torch.cuda.stream(s2):
        h_dn.copy_(d_dn, non_blocking=True)


def both():
    up()
    dn()


tu, td, tb = timed(up), timed(dn), timed(both)
print(f"H2D {n / tu / 1e9:.1f} GB/s  D2H {n / td / 1e9:.1f} GB/s  both {2 * n / tb / 1e9:.1f} GB/s total")
