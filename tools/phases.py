"""Per-phase device times of one config's contraction (V/W boxes, core GEMV,
P/U boxes; CUDA events), plus the launch-by-launch list under ncu if wanted.
usage: phases.py CONFIG"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, paper_2411_03029_b200 as tb
from paper_2411_03029_b200.configs import BY_NAME
c = BY_NAME[sys.argv[1]]
torch.cuda.set_device(0)
bf = tb.tbf_construct(c.spec, c.L, c.tol, seed=c.seed)
F = torch.randn(2 * c.points, dtype=torch.float64, device="cuda"); G = torch.empty_like(F)
s = torch.cuda.current_stream().cuda_stream
for _ in range(3): bf.contract_device(F.data_ptr(), G.data_ptr(), 1, s)
torch.cuda.synchronize()
print(sys.argv[1], bf.apply_engine(), bf.plan_stats(), flush=True)
for trial in range(2):
    p = bf.profile_contract(F.data_ptr(), G.data_ptr(), reps=5, stream=s)
    print("trial", trial, {k: round(v, 3) for k, v in p.items()}, flush=True)
