import sys, os, numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2411_03029_b200 as tb
spec = {"radon64": tb.radon2d(64), "plates32": tb.green_plates(32)}[sys.argv[1]]
L = int(sys.argv[2]); nv = int(sys.argv[3])
bf = tb.tbf_construct(spec, L, 1e-6, seed=3)
fz = bf.export()
print("ranks", fz.ranks.max(), "core rows", fz.core_rows[:8], "cols", fz.core_cols[:8], flush=True)
rng = np.random.default_rng(0)
shape = (spec.n,) * spec.d + ((nv,) if nv > 1 else ())
F = rng.standard_normal(shape) + 1j * rng.standard_normal(shape)
G = bf.contract(F)
print("ok", np.linalg.norm(G), flush=True)
