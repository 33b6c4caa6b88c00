"""Construction timing of one config with the runtime's per-level debug prints
(OIOBF_DEBUG=1) -- optionally with the two sides serialised
(OIOBF_SERIAL_SIDES=1).  usage: construct_dbg.py CONFIG [reps]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import time, torch, paper_2411_03029_b200 as tb
from paper_2411_03029_b200.configs import BY_NAME
torch.cuda.set_device(0)
c = BY_NAME[sys.argv[1]]
for i in range(int(sys.argv[2]) if len(sys.argv) > 2 else 2):
    torch.cuda.synchronize(); t = time.perf_counter()
    bf = tb.tbf_construct(c.spec, c.L, c.tol, seed=c.seed)
    torch.cuda.synchronize()
    print("construct", i, round((time.perf_counter() - t) * 1e3, 1), "ms", bf.timings(), flush=True)
    del bf
