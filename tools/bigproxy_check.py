"""GPU vs oracle on a butterfly whose proxy lists exceed 64 per mode
(k_gen_proxies_big): ranks, skeletons (ties replayed) and apply."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2411_03029_b200 as tb
from oracle import Oracle, build
build(ref=False)
spec = tb.radon2d(128)
ps = tb.ProxyStrategy(q=10)
bf = tb.tbf_construct(spec, 4, 1e-6, ps, seed=5)
gz = bf.export()
o = Oracle()
ob = o.tbf_construct(spec, 4, 1e-6, q=10, seed=5, replay=gz)
oz = ob.export()
print("rows max", gz.rows.max(), oz.rows.max(), "mismatch flags", int((oz.flags & 2).sum()))
print("ranks equal", np.array_equal(gz.ranks, oz.ranks), "skel equal", np.array_equal(gz.skel, oz.skel))
rng = np.random.default_rng(0)
F = rng.standard_normal((128, 128)) + 1j * rng.standard_normal((128, 128))
G, Go = bf.contract(F), ob.contract(F)
print("apply rel", np.linalg.norm(G - Go) / np.linalg.norm(Go))
