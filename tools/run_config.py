"""Construct + apply one BASELINE config at full size on the GPU; report
timings, ranks, memory, apply throughput and the 1000-sample dense error."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2411_03029_b200 as tb
from paper_2411_03029_b200.configs import BY_NAME
name = sys.argv[1]
nsamp = int(sys.argv[2]) if len(sys.argv) > 2 else 1000
cfg = BY_NAME[name]
torch.cuda.set_device(0)
t0 = time.perf_counter()
bf = tb.tbf_construct(cfg.spec, cfg.L, cfg.tol, seed=cfg.seed)
tc = time.perf_counter() - t0
info = bf.info()
fz_r = bf.export().ranks if info[5] < 5_000_000 else None
out = {"config": name, "L": cfg.L, "construct_s": tc, "timings": bf.timings(), "memory": bf.memory(),
       "slots": int(info[5]), "ranks_max": int(fz_r.max()) if fz_r is not None else None,
       "ranks_min": int(fz_r.min()) if fz_r is not None else None}
print(json.dumps(out), flush=True)
st = bf.plan_stats()
rng = np.random.default_rng(cfg.input_seed)
N = cfg.points
Fh = ((rng.standard_normal(N) + 1j * rng.standard_normal(N)) / np.sqrt(2)).astype(np.complex128)
F = torch.from_numpy(Fh).cuda(); G = torch.empty_like(F)
s = torch.cuda.current_stream()
for _ in range(3): bf.contract_device(F.data_ptr(), G.data_ptr(), 1, s.cuda_stream)
torch.cuda.synchronize()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
ev[0].record(s)
for _ in range(10): bf.contract_device(F.data_ptr(), G.data_ptr(), 1, s.cuda_stream)
ev[1].record(s); torch.cuda.synchronize()
ms = ev[0].elapsed_time(ev[1]) / 10
prof = bf.profile_contract(F.data_ptr(), G.data_ptr(), reps=5, stream=s.cuda_stream)
Gh = G.cpu().numpy()
rows = rng.choice(N, nsamp, replace=False)
t1 = time.perf_counter()
exact = tb.dense_rows(cfg.spec, Fh.reshape((cfg.spec.n,) * cfg.spec.d, order="F"), rows)[:, 0]
td = time.perf_counter() - t1
err = float(np.linalg.norm(Gh[rows] - exact) / np.linalg.norm(exact))
out2 = {"apply_ms": ms, "pts_per_s": N / (ms / 1e3), "bytes_alg": st["bytes_alg"], "core_bytes": st["core_bytes"],
        "GBps_alg": st["bytes_alg"] / (ms / 1e3) / 1e9, "core_GBps": st["core_bytes"] / (prof["core_ms"] / 1e3) / 1e9,
        "phases": prof, "launches": st["launches"], "sampled_rel_err": err, "tol": cfg.tol, "err_over_tol": err / cfg.tol,
        "dense_check_s": td}
print(json.dumps(out2), flush=True)
