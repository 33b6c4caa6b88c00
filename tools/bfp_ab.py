"""FP64 vs block-floating-point cores on one config: device apply time (L2
flushed, CUDA events), core-stage time, relative difference of G."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2411_03029_b200 as tb
from paper_2411_03029_b200.configs import BY_NAME
cfg = BY_NAME[sys.argv[1]]
torch.cuda.set_device(0)
bf = tb.tbf_construct(cfg.spec, cfg.L, cfg.tol, seed=cfg.seed)
rng = np.random.default_rng(cfg.input_seed)
F = torch.from_numpy((rng.standard_normal(cfg.points) + 1j * rng.standard_normal(cfg.points)) / np.sqrt(2)).cuda()
G = torch.empty_like(F)
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
s = torch.cuda.current_stream()
out, ref = {}, None
for fmt in ("fp64", "bfp32"):
    bf.set_core_format(fmt)
    for _ in range(3):
        bf.contract_device(F.data_ptr(), G.data_ptr(), 1, s.cuda_stream)
    ts = []
    for _ in range(10):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s); bf.contract_device(F.data_ptr(), G.data_ptr(), 1, s.cuda_stream); b.record(s); b.synchronize()
        ts.append(a.elapsed_time(b))
    prof = bf.profile_contract(F.data_ptr(), G.data_ptr(), reps=5, stream=s.cuda_stream)
    g = G.cpu().numpy()
    if ref is None:
        ref = g
    out[fmt] = {"ms": float(np.median(ts)), "core_ms": prof["core_ms"], "core_bytes": bf.plan_stats()["core_bytes"],
                "rel_vs_fp64": float(np.linalg.norm(g - ref) / np.linalg.norm(ref))}
print(json.dumps({"config": cfg.name, **out}))
