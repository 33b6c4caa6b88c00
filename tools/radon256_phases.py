import os, sys
sys.path.insert(0, "/root/repo")
import torch, paper_2411_03029_b200 as tb
from paper_2411_03029_b200.configs import radon2d
torch.cuda.set_device(0)
bf = tb.tbf_construct(radon2d(256), 4, 1e-6, seed=3)
F = torch.randn(2 * 256 * 256, dtype=torch.float64, device="cuda"); G = torch.empty_like(F)
s = torch.cuda.current_stream().cuda_stream
for _ in range(3): bf.contract_device(F.data_ptr(), G.data_ptr(), 1, s)
torch.cuda.synchronize()
print(bf.plan_stats(), flush=True)
for trial in range(2):
    p = bf.profile_contract(F.data_ptr(), G.data_ptr(), reps=5, stream=s)
    print("trial", trial, {k: round(float(v), 3) for k, v in p.items()}, flush=True)
