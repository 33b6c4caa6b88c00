import os, sys, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2411_03029_b200 as tb
from paper_2411_03029_b200 import _lib
n, L = int(sys.argv[1]), int(sys.argv[2])
spec = tb.radon2d(n)
bf = tb.tbf_construct(spec, L, 1e-6, seed=2411_03029)
Lc = L // 2
out = np.zeros(4 * (Lc + 1) + 1, np.int64)
_lib.check(_lib.load().oiobf_tbf_check_finite(bf.handle, out))
print("n", n, "L", L, "nonfinite per (side,level) [count, maxrank]:", out[:-1].reshape(-1, 2).tolist(), "cores:", out[-1], flush=True)
rng = np.random.default_rng(0)
F = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
G = bf.contract(F)
print("G nonfinite", int(np.sum(~np.isfinite(G))), flush=True)
