"""One construction of a config (profiling driver)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2411_03029_b200 as tb
from paper_2411_03029_b200.configs import BY_NAME
from paper_2411_03029_b200.configs import Config
PROBES = {"radon256": Config("radon256", tb.radon2d(256), 1e-6, cb=16), "radon512": Config("radon512", tb.radon2d(512), 1e-6)}
cfg = BY_NAME.get(sys.argv[1]) or PROBES[sys.argv[1]]
q, cap = (int(sys.argv[2]), int(sys.argv[3])) if len(sys.argv) > 3 else (3, 17)
bf = tb.tbf_construct(cfg.spec, cfg.L, cfg.tol, tb.ProxyStrategy(q=q, row_cap=1 << cap), seed=cfg.seed)
print(bf.timings())
