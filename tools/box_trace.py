import ctypes as C, os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2411_03029_b200 as tb
from paper_2411_03029_b200 import _lib
cfg = tb.BY_NAME[sys.argv[1] if len(sys.argv) > 1 else "green_cubes_n64"]
torch.cuda.set_device(0)
bf = tb.tbf_construct(cfg.spec, cfg.L, cfg.tol, seed=cfg.seed)
F = torch.randn(2 * cfg.points, dtype=torch.float64, device="cuda"); G = torch.empty_like(F)
bf.contract_device(F.data_ptr(), G.data_ptr(), 1, 0); torch.cuda.synchronize()
L = _lib.load()
out = np.zeros(11 * 16)
L.oiobf_debug_box_trace.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32]
for rep in range(2):
    _lib.check(L.oiobf_debug_box_trace(bf.handle, C.c_void_p(F.data_ptr()), C.c_void_p(G.data_ptr()), out.ctypes.data, 16))
for i in range(16):
    o = out[11 * i: 11 * i + 11]
    if o[0] == 0: break
    clk = (o[0] - int(o[0])) * 1e6
    print(f"launch {i}: clk {clk:.0f} MHz ctas {int(o[0])} desc {o[1]/1e3:.2f}/{o[2]/1e3:.2f} stage {o[3]/1e3:.2f}/{o[4]/1e3:.2f} "
          f"modes cold {o[5]/1e3:.2f} warm {o[6]/1e3:.2f} reduce {o[7]/1e3:.2f}/{o[8]/1e3:.2f} us (mean/max); span {o[9]/1e3:.2f} us, last start {o[10]/1e3:.2f} us")
