"""Apply A/B: one construction, then per env variant (plans are rebuilt when
set_apply_engine is called) the device-resident apply time (CUDA events, L2
flushed before each step), the phase split and the result's agreement with
the first variant.  usage: apply_ab.py CONFIG [VAR=VAL ...]  (variant '-' =
defaults; variants are env assignments applied before the plan rebuild)"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2411_03029_b200 as tb
from paper_2411_03029_b200.configs import BY_NAME
cfg = BY_NAME[sys.argv[1]]
variants = sys.argv[2:] or ["-"]
torch.cuda.set_device(0)
bf = tb.tbf_construct(cfg.spec, cfg.L, cfg.tol, seed=cfg.seed)
rng = np.random.default_rng(cfg.input_seed)
N = cfg.points
F = torch.from_numpy((rng.standard_normal(N) + 1j * rng.standard_normal(N)) / np.sqrt(2)).cuda()
G = torch.empty_like(F)
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
s = torch.cuda.current_stream()
ref = None
for v in variants:
    for kv in filter(lambda x: x != "-", v.split(",")):
        k, val = kv.split("=", 1)
        os.environ[k] = val
    bf.set_apply_engine("tiny"); bf.set_apply_engine("auto")  # drops cached plans
    for _ in range(5):
        bf.contract_device(F.data_ptr(), G.data_ptr(), 1, s.cuda_stream)
    torch.cuda.synchronize()
    ts = []
    for _ in range(20):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        bf.contract_device(F.data_ptr(), G.data_ptr(), 1, s.cuda_stream)
        b.record(s)
        b.synchronize()
        ts.append(a.elapsed_time(b))
    prof = bf.profile_contract(F.data_ptr(), G.data_ptr(), reps=10, stream=s.cuda_stream)
    g = G.cpu().numpy()
    if ref is None:
        ref = g
    rel = float(np.linalg.norm(g - ref) / np.linalg.norm(ref))
    print(json.dumps({"config": cfg.name, "variant": v, "ms": float(np.median(ts)), "ms_min": float(min(ts)),
                      "phase_ms": prof, "rel_vs_first": rel}), flush=True)
    for kv in filter(lambda x: x != "-", v.split(",")):
        os.environ.pop(kv.split("=", 1)[0], None)
