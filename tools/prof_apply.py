"""Small driver for ncu captures: construct one config, run a few device
contractions (graph replays) and exit.  Not a benchmark (numbers under ncu
are never bench values)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2411_03029_b200 as tb  # noqa: E402
from paper_2411_03029_b200.configs import BY_NAME  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="green_cubes_n64")
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--construct-only", action="store_true")
ap.add_argument("--engine", default="auto")
a = ap.parse_args()
cfg = BY_NAME[a.config]
torch.cuda.set_device(0)
bf = tb.tbf_construct(cfg.spec, cfg.L, cfg.tol, seed=cfg.seed)
bf.set_apply_engine(a.engine)
if not a.construct_only:
    rng = np.random.default_rng(0)
    F = torch.from_numpy(rng.standard_normal(2 * cfg.points)).cuda()
    G = torch.empty_like(F)
    s = torch.cuda.current_stream().cuda_stream
    for _ in range(a.reps):
        bf.contract_device(F.data_ptr(), G.data_ptr(), 1, s)
    torch.cuda.synchronize()
print("ok", bf.plan_stats())
