"""Apply timing probe (not a bench): box engine vs dataflow engine on one
config -- device path back to back, device path with an L2 flush before every
step (events around the contraction only), and the pinned-host e2e path."""
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2411_03029_b200 as tb  # noqa: E402
from paper_2411_03029_b200 import _lib  # noqa: E402
from paper_2411_03029_b200.configs import BY_NAME  # noqa: E402

cfg = BY_NAME[sys.argv[1] if len(sys.argv) > 1 else "green_cubes_n64"]
engines = sys.argv[2].split(",") if len(sys.argv) > 2 else ["box", "flow"]
torch.cuda.set_device(0)
bf = tb.tbf_construct(cfg.spec, cfg.L, cfg.tol, seed=cfg.seed)
N = cfg.points
F = torch.randn(2 * N, dtype=torch.float64, device="cuda")
G = torch.empty_like(F)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
st = torch.cuda.current_stream()
L = _lib.load()
hF = F.cpu().pin_memory()
hG = torch.empty_like(hF).pin_memory()
out = {}
for eng in engines:
    bf.set_apply_engine(eng)
    used = bf.apply_engine()
    for _ in range(5):
        bf.contract_device(F.data_ptr(), G.data_ptr(), 1, st.cuda_stream)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(50):
        bf.contract_device(F.data_ptr(), G.data_ptr(), 1, st.cuda_stream)
    e1.record()
    torch.cuda.synchronize()
    warm = e0.elapsed_time(e1) / 50 * 1e3
    ts = []
    for _ in range(30):
        flush.add_(1)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        bf.contract_device(F.data_ptr(), G.data_ptr(), 1, st.cuda_stream)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    cold = statistics.median(ts)
    res = G.cpu()
    for _ in range(5):
        _lib.check(L.oiobf_tbf_contract(bf.handle, hF.numpy(), hG.numpy(), 1))
    t0 = time.perf_counter()
    while time.perf_counter() - t0 < 0.3:  # PCIe link warm-up
        _lib.check(L.oiobf_tbf_contract(bf.handle, hF.numpy(), hG.numpy(), 1))
    es = []
    for _ in range(100):
        t = time.perf_counter()
        _lib.check(L.oiobf_tbf_contract(bf.handle, hF.numpy(), hG.numpy(), 1))
        es.append(time.perf_counter() - t)
    e2e_res = hG.clone()
    out[eng] = (res, e2e_res)
    print(f"{cfg.name} {eng}->{used}: device warm {warm:.1f} us  L2-flushed {cold:.1f} us  "
          f"e2e median {1e6 * statistics.median(es):.1f} us  min {1e6 * min(es):.1f} us", flush=True)
if len(out) > 1:
    (r0, h0), (r1, h1) = list(out.values())[:2]
    print("device rel diff", float((r0 - r1).norm() / r0.norm()), " e2e rel diff", float((h0 - h1).norm() / h0.norm()),
          " e2e vs device", float((h1 - r1).norm() / r1.norm()))
