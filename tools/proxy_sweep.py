"""Accuracy vs ProxyStrategy sweep on the GPU (construction time, ranks,
1000-sample relative error against GPU dense sums).

usage: python tools/proxy_sweep.py CONFIG[:L] mode,q,log2cap [mode,q,log2cap ...]
CONFIG is a BASELINE config name or one of the probe names below.
One JSON line per strategy."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2411_03029_b200 as tb
from paper_2411_03029_b200.configs import BY_NAME, Config

PROBES = {
    "radon128": Config("radon128", tb.radon2d(128), 1e-6),
    "radon256": Config("radon256", tb.radon2d(256), 1e-6),
    "radon512": Config("radon512", tb.radon2d(512), 1e-6),
    "cubes32": Config("cubes32", tb.green_cubes(32), 1e-6),
    "cubes128": Config("cubes128", tb.green_cubes(128), 1e-4),
    "plates256": Config("plates256", tb.green_plates(256), 1e-6),
}


def main():
    name = sys.argv[1]
    L = None
    if ":" in name:
        name, L = name.split(":")
        L = int(L)
    cfg = BY_NAME.get(name) or PROBES[name]
    L = cfg.L if L is None else L
    N = cfg.points
    rng = np.random.default_rng(cfg.input_seed)
    F = ((rng.standard_normal(N) + 1j * rng.standard_normal(N)) / np.sqrt(2)).reshape((cfg.spec.n,) * cfg.spec.d,
                                                                                      order="F")
    rows = rng.choice(N, 1000, replace=False)
    t = time.perf_counter()
    exact = tb.dense_rows(cfg.spec, F, rows)[:, 0]
    tdense = time.perf_counter() - t
    for a in sys.argv[2:]:
        mode, q, cap = (int(x) for x in a.split(","))
        ps = tb.ProxyStrategy(mode=mode, q=q, row_cap=1 << cap)
        t = time.perf_counter()
        bf = tb.tbf_construct(cfg.spec, L, cfg.tol, ps, seed=cfg.seed)
        tc = time.perf_counter() - t
        G = bf.contract(F).reshape(-1, order="F")
        err = float(np.linalg.norm(G[rows] - exact) / np.linalg.norm(exact))
        info = bf.info()
        rk = None
        if info[5] < 5_000_000:
            fz = bf.export()
            rk = [int(fz.ranks.min()), int(fz.ranks.max()), int(fz.rows.max())]
        print(json.dumps({"config": name, "L": L, "tol": cfg.tol, "mode": mode, "q": q, "cap": cap,
                          "construct_s": round(tc, 3), "err": err, "ratio": err / cfg.tol,
                          "ranks_min_max_rows": rk, "cores_GB": bf.memory()["cores"] / 1e9,
                          "dense_s": round(tdense, 2)}), flush=True)
        del bf


if __name__ == "__main__":
    main()
