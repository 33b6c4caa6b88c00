import ctypes as C, os, sys, numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2411_03029_b200 as tb
from paper_2411_03029_b200 import _lib
n, L = 1024, 6
bf = tb.tbf_construct(tb.radon2d(n), L, 1e-6, seed=2411_03029)
info = bf.info()
ns, nsk, nip, npm = int(info[5]), int(info[6]), int(info[7]), int(info[9])
ranks = np.zeros(ns, np.int64); ncols = np.zeros(ns, np.int64); rows = np.zeros(ns, np.int64)
skel = np.zeros(nsk, np.int64); interp = np.zeros(2 * nip); perm = np.zeros(npm, np.int64)
P = _lib.ptr
_lib.check(_lib.load().oiobf_tbf_export(bf.handle, P(ranks), P(ncols), P(rows), P(skel), P(interp), P(perm), None, None, None, None))
z = interp.view(np.complex128)
io = np.concatenate([[0], np.cumsum(ranks * ncols)])
bad = [g for g in range(ns) if not np.all(np.isfinite(z[io[g]:io[g + 1]]))]
print("bad slots", len(bad), bad[:10])
for g in bad[:5]:
    blk = z[io[g]:io[g + 1]].reshape(ranks[g], ncols[g], order="F")
    print(g, "rank", ranks[g], "w", ncols[g], "nonfinite", int(np.sum(~np.isfinite(blk))), "max finite", np.nanmax(np.abs(blk[np.isfinite(blk)])) if np.any(np.isfinite(blk)) else None)
lvl = np.cumsum([0] + [64 * (4 ** l) * 2 * (2 ** (3 - l)) for l in range(4)] * 2)
print("level bounds", lvl.tolist())
np.save("gpurun_out/bad_slots.npy", np.array(bad))
np.save("gpurun_out/ranks5.npy", ranks); np.save("gpurun_out/ncols5.npy", ncols); np.save("gpurun_out/skel5.npy", skel); np.save("gpurun_out/perm5.npy", perm)
