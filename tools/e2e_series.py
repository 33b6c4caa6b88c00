"""Time series of the pinned e2e call with the bench's loop shape (L2 flush + sync before each call)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2411_03029_b200 as tb  # noqa: E402
from paper_2411_03029_b200 import _lib  # noqa: E402
from paper_2411_03029_b200.configs import BY_NAME  # noqa: E402

cfg = BY_NAME["green_cubes_n64"]
torch.cuda.set_device(0)
bf = tb.tbf_construct(cfg.spec, cfg.L, cfg.tol, seed=cfg.seed)
hF = torch.randn(2 * cfg.points, dtype=torch.float64).pin_memory()
hG = torch.empty_like(hF).pin_memory()
Fv, Gv = hF.numpy(), hG.numpy()
L = _lib.load()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for mode in ("flush", "noflush", "flush"):
    ts = []
    for i in range(200):
        if mode == "flush":
            flush.zero_()
        torch.cuda.synchronize()
        t = time.perf_counter()
        _lib.check(L.oiobf_tbf_contract(bf.handle, Fv, Gv, 1))
        ts.append((time.perf_counter() - t) * 1e6)
    a = np.array(ts)
    print(mode, "first10", np.round(a[:10]).astype(int).tolist())
    print(mode, "blocks of 20 (median):", [int(np.median(a[i:i + 20])) for i in range(0, 200, 20)], flush=True)
