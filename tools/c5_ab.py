import os, sys, time
sys.path.insert(0, "/root/repo")
import numpy as np, torch, paper_2411_03029_b200 as tb
from paper_2411_03029_b200.configs import BY_NAME
c = BY_NAME["radon2d_n1024"]
torch.cuda.set_device(0)
bf = tb.tbf_construct(c.spec, c.L, c.tol, seed=c.seed)
F = torch.randn(2 * c.points, dtype=torch.float64, device="cuda"); G = torch.empty_like(F)
s = torch.cuda.current_stream().cuda_stream
for _ in range(3): bf.contract_device(F.data_ptr(), G.data_ptr(), 1, s)
torch.cuda.synchronize()
for trial in range(3):
    p = bf.profile_contract(F.data_ptr(), G.data_ptr(), reps=5, stream=s)
    print(os.environ.get("TAG", ""), "trial", trial, {k: round(v, 3) for k, v in p.items()}, flush=True)
