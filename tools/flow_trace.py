"""Dataflow-engine timeline (debug, not a bench): runs config contractions with
OIOBF_FLOW_TRACE set (the library dumps per-item %globaltimer stamps of the
last launch) and summarises per op: items, claim -> inputs-ready wait, run
time, and the op's window in the launch."""
import os
import sys

path = os.path.abspath(sys.argv[2] if len(sys.argv) > 2 else "gpurun_out/flow_trace.csv")
os.makedirs(os.path.dirname(path), exist_ok=True)
os.environ["OIOBF_FLOW_TRACE"] = path
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2411_03029_b200 as tb  # noqa: E402
from paper_2411_03029_b200.configs import BY_NAME  # noqa: E402

cfg = BY_NAME[sys.argv[1] if len(sys.argv) > 1 else "green_cubes_n64"]
torch.cuda.set_device(0)
bf = tb.tbf_construct(cfg.spec, cfg.L, cfg.tol, seed=cfg.seed)
bf.set_apply_engine("flow")
F = torch.randn(2 * cfg.points, dtype=torch.float64, device="cuda")
G = torch.empty_like(F)
for _ in range(5):
    bf.contract_device(F.data_ptr(), G.data_ptr(), 1, torch.cuda.current_stream().cuda_stream)
torch.cuda.synchronize()
a = np.genfromtxt(path, delimiter=",", names=True, dtype=np.int64)
t0 = a["claimed"].min()
print(f"{cfg.name}: {len(a)} items, launch span {(a['done'].max() - t0) / 1e3:.1f} us")
for op in np.unique(a["op"]):
    m = a[a["op"] == op]
    wait = (m["ready"] - m["claimed"]) / 1e3
    run = (m["done"] - m["ready"]) / 1e3
    print(f"op {op} kind {m['kind'][0]}: {len(m):5d} items, deps/item {m['ndep'].mean():6.1f}, "
          f"wait mean {wait.mean():6.2f} max {wait.max():6.2f} us, run mean {run.mean():6.2f} max {run.max():6.2f} us, "
          f"window {(m['claimed'].min() - t0) / 1e3:7.1f} .. {(m['done'].max() - t0) / 1e3:7.1f} us")
    if m["kind"][0] == 0:
        ph = [m["ready"], m["staged"], m["first"], m["middle"], m["last"], m["done"]]
        names = ["stage", "mode d-1", "middle", "mode 0", "publish"]
        print("      phases: " + ", ".join(f"{n} {((b - a) / 1e3).mean():.2f}" for n, a, b in zip(names, ph, ph[1:])))
