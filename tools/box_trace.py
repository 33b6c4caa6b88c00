"""Per-CTA timeline of every box launch (debug; stamps from oiobf_debug_box_trace)."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2411_03029_b200 as tb  # noqa: E402
from paper_2411_03029_b200 import _lib  # noqa: E402

cfg = tb.BY_NAME[sys.argv[1] if len(sys.argv) > 1 else "green_cubes_n64"]
torch.cuda.set_device(0)
bf = tb.tbf_construct(cfg.spec, cfg.L, cfg.tol, seed=cfg.seed)
F = torch.randn(2 * cfg.points, dtype=torch.float64, device="cuda")
G = torch.empty_like(F)
L = _lib.load()
L.oiobf_debug_box_trace.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p]
out = np.zeros(1 << 22)
w = np.zeros(1, np.int64)
for rep in range(2):  # second pass is warm
    _lib.check(L.oiobf_debug_box_trace(bf.handle, C.c_void_p(F.data_ptr()), C.c_void_p(G.data_ptr()),
                                       out.ctypes.data, out.size, w.ctypes.data))
pos, li = 0, 0
names = ["start->pre-wait", "wait", "stage", "mode d-1", "middle", "mode 0"]
while pos < w[0]:
    nct, cs, smem, stage = out[pos:pos + 4]
    st = out[pos + 4:pos + 4 + int(nct) * 8].reshape(int(nct), 8)
    pos += 4 + int(nct) * 8
    ph = np.diff(st[:, :7], axis=1) / 1e3
    print(f"launch {li}: ctas {int(nct)} cs {int(cs)} smem {smem/1024:.0f}KB stage {int(stage)}  "
          f"start spread {st[:, 0].max()/1e3:.2f} us  end max {st[:, 6].max()/1e3:.2f} us")
    for j, n in enumerate(names):
        print(f"    {n:16s} mean {ph[:, j].mean():6.2f}  max {ph[:, j].max():6.2f} us")
    li += 1
