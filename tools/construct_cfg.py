"""Construct one config once (timings + per-level debug lines with OIOBF_DEBUG=1).
usage: construct_cfg.py CONFIG"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, paper_2411_03029_b200 as tb
from paper_2411_03029_b200.configs import BY_NAME
c = BY_NAME[sys.argv[1]]
torch.cuda.set_device(0)
t = time.perf_counter()
bf = tb.tbf_construct(c.spec, c.L, c.tol, seed=c.seed)
torch.cuda.synchronize()
print("construct", sys.argv[1], round(time.perf_counter() - t, 3), "s", bf.timings(), flush=True)
