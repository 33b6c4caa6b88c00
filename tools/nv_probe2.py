"""Device contraction of config 2 with n_v vectors (argv[1]), for ncu launch lists."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, paper_2411_03029_b200 as tb
from paper_2411_03029_b200.configs import BY_NAME
nv = int(sys.argv[1])
c = BY_NAME["green_cubes_n64"]
torch.cuda.set_device(0)
bf = tb.tbf_construct(c.spec, c.L, c.tol, seed=c.seed)
F = torch.randn(2 * c.points * nv, dtype=torch.float64, device="cuda"); G = torch.empty_like(F)
s = torch.cuda.current_stream().cuda_stream
for _ in range(2): bf.contract_device(F.data_ptr(), G.data_ptr(), nv, s)
torch.cuda.synchronize()
print("ok")
