"""Multi-RHS apply probe (not a bench): device contraction time vs n_v on one
config, L2 flushed before each step.
"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2411_03029_b200 as tb  # noqa: E402
from paper_2411_03029_b200.configs import BY_NAME  # noqa: E402

cfg = BY_NAME[sys.argv[1] if len(sys.argv) > 1 else "green_cubes_n64"]
torch.cuda.set_device(0)
bf = tb.tbf_construct(cfg.spec, cfg.L, cfg.tol, seed=cfg.seed)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
st = torch.cuda.current_stream()
for nv in (1, 2, 4, 8, 16, 32):
    F = torch.randn(2 * cfg.points * nv, dtype=torch.float64, device="cuda")
    G = torch.empty_like(F)
    for _ in range(3):
        bf.contract_device(F.data_ptr(), G.data_ptr(), nv, st.cuda_stream)
    ts = []
    for _ in range(20):
        flush.add_(1)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        bf.contract_device(F.data_ptr(), G.data_ptr(), nv, st.cuda_stream)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    print(f"nv {nv:3d}: {statistics.median(ts):8.1f} us/step  {statistics.median(ts) / nv:7.1f} us/vector", flush=True)
