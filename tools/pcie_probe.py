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


# 2-D copies (the offload path's row panels of a column-major A), through cudaMemcpy2DAsync
# itself (torch copies strided host views another way): width = rows * 8 B, pitch 64 KB
import ctypes  # noqa: E402

rt = None
for name in ("libcudart.so.12", "libcudart.so"):
    try:
        rt = ctypes.CDLL(name)
        break
    except OSError:
        pass
if rt is None:
    import glob
    import os
    cands = glob.glob(os.path.join(os.path.dirname(torch.__file__), "..", "nvidia", "cuda_runtime", "lib", "libcudart.so*"))
    rt = ctypes.CDLL(cands[0])
rt.cudaMemcpy2DAsync.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p, ctypes.c_size_t,
                                 ctypes.c_size_t, ctypes.c_size_t, ctypes.c_int, ctypes.c_void_p]
A = torch.empty((8192, 8192), dtype=torch.float64).pin_memory()   # 512 MB, column j at j * 64 KB
dA = torch.empty((8192, 8192), dtype=torch.float64, device="cuda")
for rows in (512, 1024, 2048, 4096, 8192):
    def h2d2():
        rc = rt.cudaMemcpy2DAsync(ctypes.c_void_p(dA.data_ptr()), rows * 8, ctypes.c_void_p(A.data_ptr()),
                                  8192 * 8, rows * 8, 8192, 1, ctypes.c_void_p(s1.cuda_stream))
        assert rc == 0, rc
    t = timed(h2d2, 3)
    print(f"H2D cudaMemcpy2DAsync: {rows} rows x 8192 columns (pitch 64 KB, {rows * 8 // 1024} KB rows): "
          f"{rows * 8192 * 8 / t / 1e9:.1f} GB/s")
    def d2h2():
        rc = rt.cudaMemcpy2DAsync(ctypes.c_void_p(A.data_ptr()), 8192 * 8, ctypes.c_void_p(dA.data_ptr()),
                                  rows * 8, rows * 8, 8192, 2, ctypes.c_void_p(s2.cuda_stream))
        assert rc == 0, rc
    t = timed(d2h2, 3)
    print(f"D2H cudaMemcpy2DAsync: {rows} rows x 8192 columns: {rows * 8192 * 8 / t / 1e9:.1f} GB/s")
