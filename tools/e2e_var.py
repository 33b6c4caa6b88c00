"""Host-side latency spread of the pinned e2e path vs plain torch copies (not a bench)."""
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
N = cfg.points
hF = torch.randn(2 * N, dtype=torch.float64).pin_memory()
hG = torch.empty_like(hF).pin_memory()
Fv, Gv = hF.numpy(), hG.numpy()
L = _lib.load()
dF = torch.empty(2 * N, dtype=torch.float64, device="cuda")
dG = torch.empty_like(dF)


def pct(ts):
    a = np.array(ts) * 1e6
    return " ".join(f"p{p}={np.percentile(a, p):.0f}" for p in (0, 10, 50, 90, 99))


def run(name, fn, reps=300):
    for _ in range(10):
        fn()
    ts = []
    for _ in range(reps):
        t = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t)
    print(f"{name:28s} {pct(ts)} us", flush=True)


def lib_call():
    _lib.check(L.oiobf_tbf_contract(bf.handle, Fv, Gv, 1))


def torch_copies():
    dF.copy_(hF, non_blocking=True)
    hG.copy_(dG, non_blocking=True)
    torch.cuda.synchronize()


def torch_copies_apply():
    dF.copy_(hF, non_blocking=True)
    bf.contract_device(dF.data_ptr(), dG.data_ptr(), 1, torch.cuda.current_stream().cuda_stream)
    hG.copy_(dG, non_blocking=True)
    torch.cuda.synchronize()


run("lib e2e (pipelined graph)", lib_call)
run("torch H2D+D2H only", torch_copies)
run("torch H2D+graph+D2H", torch_copies_apply)
run("lib e2e again", lib_call)
