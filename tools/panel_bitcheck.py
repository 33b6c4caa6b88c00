"""Register-cached vs generic absorb (OIOBF_PANEL_GENERIC=1) must give the same
factorization BIT FOR BIT (same operations, same order; the register-cached
absorb also folds the zero rows of a partial last panel, which add +0 to every
sum).  Wide IDs: Radon n=256, L=4 (widths up to 64)."""
import os, subprocess, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if len(sys.argv) > 1:
    import numpy as np, torch
    import paper_2411_03029_b200 as tb
    from paper_2411_03029_b200.configs import radon2d
    torch.cuda.set_device(0)
    bf = tb.tbf_construct(radon2d(256), 4, 1e-6, seed=3)
    fz = bf.export()
    np.savez(sys.argv[1], ranks=fz.ranks, skel=fz.skel, interp=fz.interp, ncols=fz.ncols)
    sys.exit(0)
import numpy as np
subprocess.run([sys.executable, __file__, "/tmp/pb_a.npz"], check=True)
subprocess.run([sys.executable, __file__, "/tmp/pb_b.npz"], check=True, env={**os.environ, "OIOBF_PANEL_GENERIC": "1"})
a, b = np.load("/tmp/pb_a.npz"), np.load("/tmp/pb_b.npz")
ok = all(np.array_equal(a[k], b[k]) for k in ("ranks", "skel", "interp", "ncols"))
print("bit-identical:", ok, "max width", int(a["ncols"].max()))
