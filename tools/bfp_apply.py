"""Profiling driver: config 3 apply on block-floating-point cores (tools/prof_apply.py twin)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2411_03029_b200 as tb
from paper_2411_03029_b200.configs import BY_NAME
cfg = BY_NAME[sys.argv[1] if len(sys.argv) > 1 else "green_cubes_n256"]
torch.cuda.set_device(0)
bf = tb.tbf_construct(cfg.spec, cfg.L, cfg.tol, seed=cfg.seed)
bf.set_core_format("bfp32")
F = torch.from_numpy(np.random.default_rng(0).standard_normal(2 * cfg.points)).cuda()
G = torch.empty_like(F)
for _ in range(2):
    bf.contract_device(F.data_ptr(), G.data_ptr(), 1, torch.cuda.current_stream().cuda_stream)
torch.cuda.synchronize()
print("ok")
