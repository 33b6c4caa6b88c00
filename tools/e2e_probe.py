"""Apply timing probe (not a bench): device graph replay and the pinned-host
pipeline, for one config; env knobs are read by the library at load."""
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
torch.cuda.set_device(0)
bf = tb.tbf_construct(cfg.spec, cfg.L, cfg.tol, seed=cfg.seed)
N = cfg.points
F = torch.randn(2 * N, dtype=torch.float64, device="cuda")
G = torch.empty_like(F)
st = torch.cuda.current_stream()
for _ in range(5):
    bf.contract_device(F.data_ptr(), G.data_ptr(), 1, st.cuda_stream)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(50):
    bf.contract_device(F.data_ptr(), G.data_ptr(), 1, st.cuda_stream)
e1.record()
torch.cuda.synchronize()
dev_us = e0.elapsed_time(e1) / 50 * 1e3
hF = F.cpu().pin_memory()
hG = torch.empty_like(hF).pin_memory()
L = _lib.load()
for _ in range(5):
    _lib.check(L.oiobf_tbf_contract(bf.handle, hF.numpy(), hG.numpy(), 1))
ts = []
for _ in range(50):
    t = time.perf_counter()
    _lib.check(L.oiobf_tbf_contract(bf.handle, hF.numpy(), hG.numpy(), 1))
    ts.append(time.perf_counter() - t)
print(f"{cfg.name} env={os.environ.get('PROBE_TAG', '')}: device graph {dev_us:.1f} us  "
      f"e2e median {1e6 * statistics.median(ts):.1f} us  min {1e6 * min(ts):.1f} us")
