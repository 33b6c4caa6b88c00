"""PCIe copy probe: pinned H2D / D2H bandwidth alone and concurrently (not a bench)."""
import time
import torch

torch.cuda.set_device(0)
for mb in (1, 2, 4, 8, 64):
    n = mb * (1 << 20) // 8
    h = torch.randn(n, dtype=torch.float64).pin_memory()
    h2 = torch.empty_like(h).pin_memory()
    d = torch.empty(n, dtype=torch.float64, device="cuda")
    d2 = torch.randn(n, dtype=torch.float64, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    for _ in range(3):
        d.copy_(h, non_blocking=True); h2.copy_(d2, non_blocking=True)
    torch.cuda.synchronize()
    def timeit(fn, reps=20):
        torch.cuda.synchronize()
        t = time.perf_counter()
        for _ in range(reps):
            fn()
        torch.cuda.synchronize()
        return (time.perf_counter() - t) / reps * 1e6
    t_h2d = timeit(lambda: d.copy_(h, non_blocking=True))
    t_d2h = timeit(lambda: h2.copy_(d2, non_blocking=True))
    def both():
        with torch.cuda.stream(s1):
            d.copy_(h, non_blocking=True)
        with torch.cuda.stream(s2):
            h2.copy_(d2, non_blocking=True)
    t_both = timeit(both)
    print(f"{mb:3d} MB: H2D {t_h2d:8.1f} us ({mb/1024/t_h2d*1e6:6.1f} GB/s)  D2H {t_d2h:8.1f} us ({mb/1024/t_d2h*1e6:6.1f} GB/s)"
          f"  both {t_both:8.1f} us")
