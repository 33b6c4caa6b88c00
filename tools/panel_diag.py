"""Panel time split per (side, level): full / entry generation alone / absorb
alone (OIOBF_PANEL_DIAG=1 makes launch_panel re-run each level's panel in the
three modes and print the times).  usage: panel_diag.py CONFIG|radon256"""
import os, sys, time
os.environ["OIOBF_PANEL_DIAG"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, paper_2411_03029_b200 as tb
from paper_2411_03029_b200.configs import BY_NAME
torch.cuda.set_device(0)
name = sys.argv[1]
if name == "radon256":
    spec, L, tol, seed = tb.radon2d(256), 4, 1e-6, 1
else:
    c = BY_NAME[name]
    spec, L, tol, seed = c.spec, c.L, c.tol, c.seed
t = time.perf_counter()
bf = tb.tbf_construct(spec, L, tol, seed=seed)
torch.cuda.synchronize()
print("construct", name, round(time.perf_counter() - t, 3), "s", bf.timings(), flush=True)
