import os, sys, numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import paper_2411_03029_b200 as tb
from paper_2411_03029_b200.butterfly import Factorization
from oracle import Oracle
from helpers import slot_geometry, slot_target
o = Oracle()
ranks = np.load("gpurun_out/ranks5.npy"); ncols = np.load("gpurun_out/ncols5.npy"); skel = np.load("gpurun_out/skel5.npy"); perm = np.load("gpurun_out/perm5.npy")
bad = np.load("gpurun_out/bad_slots.npy")
fz = Factorization(2, 1024, 6, 3, 64, ranks, ncols, None, skel, None, perm, None, None, None, None)
g = int(bad[0]); sd, l = 0, 3; base = 7168; idx = g - base
geo = slot_geometry(2, 1024, 6, 3, sd, l, idx)
target = slot_target(fz, sd, l, idx)
r_est = 40  # level-synchronous r_est for level 3 = max(8, max rank of levels < 3)
r_est = int(max(8, ranks[:base].max()))
lists = o.proxy_lists(geo["ranges"], geo["skip"], 3 * r_est, seed=o.derive_seed(2411_03029, geo["tags"]))
lists[geo["skip"]] = target
A = o.unfolding(tb.radon2d(1024), lists, geo["skip"])
print("slot", g, "A", A.shape, "finite", np.all(np.isfinite(A)), "r_est", r_est, flush=True)
oc = o.column_id(A, 1e-6)
print("oracle rank", oc["rank"], "interp finite", np.all(np.isfinite(oc["interp"])), "max", np.abs(oc["interp"]).max())
gc = tb.column_id(A, 1e-6)
print("gpu matrix-path rank", gc.rank, "interp finite", np.all(np.isfinite(gc.interp)), "n nonfinite", int(np.sum(~np.isfinite(gc.interp))))
sv = np.linalg.svd(A, compute_uv=False)
print("singular values rel", (sv / sv[0])[[0, 10, 20, 21, 30, 40, 50, min(63, len(sv)-1)]])
print("col norms min/max", np.linalg.norm(A, axis=0).min(), np.linalg.norm(A, axis=0).max())
