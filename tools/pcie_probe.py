"""PCIe probe: pinned H2D / D2H bandwidth alone and concurrently (context for the e2e number)."""
import time

import torch

MB = 1 << 20
h = torch.empty(256 * MB, dtype=torch.uint8).pin_memory()
hd = torch.empty(128 * MB, dtype=torch.uint8).pin_memory()
d = torch.empty(256 * MB, dtype=torch.uint8, device="cuda")
dd = torch.empty(128 * MB, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / reps


for piece in (4, 16, 64, 256):
    def h2d():
        with torch.cuda.stream(s1):
            for o in range(0, 256, piece):
                d[o * MB:(o + piece) * MB].copy_(h[o * MB:(o + piece) * MB], non_blocking=True)
    t = timed(h2d)
    print(f"H2D 256 MB in {piece} MB pieces: {256 * MB / t / 1e9:.1f} GB/s")


def d2h():
    with torch.cuda.stream(s2):
        hd.copy_(dd, non_blocking=True)


print(f"D2H 128 MB: {128 * MB / timed(d2h) / 1e9:.1f} GB/s")


def both():
    with torch.cuda.stream(s1):
        d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2):
        hd.copy_(dd, non_blocking=True)


t = timed(both)
print(f"H2D 256 MB + D2H 128 MB concurrently: {t * 1e3:.2f} ms ({384 * MB / t / 1e9:.1f} GB/s total)")
