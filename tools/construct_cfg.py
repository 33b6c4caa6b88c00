"""Construct one config once (timings + per-level debug lines with OIOBF_DEBUG=1).
usage: construct_cfg.py CONFIG"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, paper_2411_03029_b200 as tb
from paper_2411_03029_b200.configs import BY_NAME
c = BY_NAME[sys.argv[1]]
torch.cuda.set_device(0)
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
for i in range(reps):  # the first construction in a process includes pool growth / module loading
    t = time.perf_counter()
    bf = tb.tbf_construct(c.spec, c.L, c.tol, seed=c.seed)
    torch.cuda.synchronize()
    print("construct", sys.argv[1], i, round(time.perf_counter() - t, 3), "s", bf.timings(), flush=True)
    del bf
