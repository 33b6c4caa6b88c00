"""Per-vector device time of a contraction with n_v vectors (argv[2]) for a config (argv[1])."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, paper_2411_03029_b200 as tb
from paper_2411_03029_b200.configs import BY_NAME
c = BY_NAME[sys.argv[1]]; nv = int(sys.argv[2])
torch.cuda.set_device(0)
bf = tb.tbf_construct(c.spec, c.L, c.tol, seed=c.seed)
F = torch.randn(2 * c.points * nv, dtype=torch.float64, device="cuda"); G = torch.empty_like(F)
st = torch.cuda.current_stream()
for _ in range(3): bf.contract_device(F.data_ptr(), G.data_ptr(), nv, st.cuda_stream)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(st)
for _ in range(20): bf.contract_device(F.data_ptr(), G.data_ptr(), nv, st.cuda_stream)
e1.record(st); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 20
print(f"{sys.argv[1]} nv={nv} chunk={os.environ.get('OIOBF_NV_CHUNK', '4')} {ms * 1e3:.1f} us/call {ms * 1e3 / nv:.1f} us/vector", flush=True)
