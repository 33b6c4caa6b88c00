"""Construction time + sampled error for one config and strategy, in a fresh
process per variant (env switches are read once per process)."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2411_03029_b200 as tb
from paper_2411_03029_b200.configs import BY_NAME
name = sys.argv[1]
q, cap = (int(sys.argv[2]), int(sys.argv[3])) if len(sys.argv) > 3 else (3, 17)
cfg = BY_NAME[name]
ps = tb.ProxyStrategy(q=q, row_cap=1 << cap)
t = time.perf_counter(); bf = tb.tbf_construct(cfg.spec, cfg.L, cfg.tol, ps, seed=cfg.seed); t1 = time.perf_counter() - t
del bf
t = time.perf_counter(); bf2 = tb.tbf_construct(cfg.spec, cfg.L, cfg.tol, ps, seed=cfg.seed); t2 = time.perf_counter() - t
N = cfg.points
rng = np.random.default_rng(cfg.input_seed)
F = ((rng.standard_normal(N) + 1j * rng.standard_normal(N)) / np.sqrt(2)).reshape((cfg.spec.n,) * cfg.spec.d, order="F")
rows = rng.choice(N, 1000, replace=False)
exact = tb.dense_rows(cfg.spec, F, rows)[:, 0]
G = bf2.contract(F).reshape(-1, order="F")
err = float(np.linalg.norm(G[rows] - exact) / np.linalg.norm(exact))
print(json.dumps({"config": name, "q": q, "cap": cap, "legacy": bool(os.environ.get("OIOBF_PANEL_LEGACY")),
                  "first_s": round(t1, 3), "warm_s": round(t2, 3), "timings": bf2.timings(), "err": err,
                  "ratio": err / cfg.tol}), flush=True)
