"""Async host-buffer contraction probe (not a bench): host enqueue cost per
call, steady-state time per call, and the PCIe copies alone at the same
cadence (H2D / D2H of 4 MB back to back on two streams)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2411_03029_b200 as tb  # noqa: E402
from paper_2411_03029_b200.configs import BY_NAME  # noqa: E402

cfg = BY_NAME[sys.argv[1] if len(sys.argv) > 1 else "green_cubes_n64"]
torch.cuda.set_device(0)
bf = tb.tbf_construct(cfg.spec, cfg.L, cfg.tol, seed=cfg.seed)
N = cfg.points
hF = torch.randn(2 * N, dtype=torch.float64).pin_memory()
hG = torch.empty_like(hF).pin_memory()
s = torch.cuda.Stream()
Fv, Gv = hF.numpy(), hG.numpy()
t0 = time.perf_counter()
while time.perf_counter() - t0 < 0.5:
    bf.contract_async(Fv, Gv, 1, s.cuda_stream)
s.synchronize()
for reps in (50, 200, 1000):
    enq = 0.0
    t = time.perf_counter()
    for _ in range(reps):
        a = time.perf_counter()
        bf.contract_async(Fv, Gv, 1, s.cuda_stream)
        enq += time.perf_counter() - a
    s.synchronize()
    tot = time.perf_counter() - t
    print(f"{reps:5d} calls: {1e6 * tot / reps:7.1f} us/call, host enqueue {1e6 * enq / reps:6.1f} us/call", flush=True)
dF = torch.empty(2 * N, dtype=torch.float64, device="cuda")
dG = torch.randn(2 * N, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(200):
    with torch.cuda.stream(s1):
        dF.copy_(hF, non_blocking=True)
    with torch.cuda.stream(s2):
        hG.copy_(dG, non_blocking=True)
torch.cuda.synchronize()
print(f"H2D || D2H 4 MB each, 200 back to back: {1e6 * (time.perf_counter() - t) / 200:.1f} us per pair")
dev = torch.empty_like(dG)
st = torch.cuda.current_stream()
for _ in range(5):
    bf.contract_device(dG.data_ptr(), dev.data_ptr(), 1, st.cuda_stream)
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(200):
    bf.contract_device(dG.data_ptr(), dev.data_ptr(), 1, st.cuda_stream)
torch.cuda.synchronize()
print(f"device contraction back to back: {1e6 * (time.perf_counter() - t) / 200:.1f} us")
