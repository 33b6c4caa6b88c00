"""Construction A/B over env variants (each in a fresh process: env switches
are read once): time per config and factor agreement with the first variant
(ranks / skeletons exact, interps close).
  python tools/panel_ab.py cfg[,cfg...] 'ENV=V;ENV2=V2' '' ...   ('' = defaults)"""
import json, os, subprocess, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if len(sys.argv) > 2 and sys.argv[1] == "--one":
    import numpy as np
    import paper_2411_03029_b200 as tb
    from paper_2411_03029_b200.configs import BY_NAME, Config
    probes = {"radon256": Config("radon256", tb.radon2d(256), 1e-6, cb=16), "cubes32": Config("cubes32", tb.green_cubes(32), 1e-6)}
    cfg = BY_NAME.get(sys.argv[2]) or probes[sys.argv[2]]
    q, cap = int(sys.argv[4]), int(sys.argv[5])
    ps = tb.ProxyStrategy(q=q, row_cap=1 << cap)
    t = time.perf_counter(); bf = tb.tbf_construct(cfg.spec, cfg.L, cfg.tol, ps, seed=cfg.seed); t1 = time.perf_counter() - t
    first_ms = bf.timings()["total_ms"]
    if os.environ.get("AB_WARM", "1") == "1":  # report the second construction (module loading, pool growth excluded)
        del bf
        t = time.perf_counter(); bf = tb.tbf_construct(cfg.spec, cfg.L, cfg.tol, ps, seed=cfg.seed); t1 = time.perf_counter() - t
    tim = bf.timings()
    fz = bf.export(pairs=[])
    np.savez(sys.argv[3], ranks=fz.ranks, skel=fz.skel, interp=fz.interp, ncols=fz.ncols)
    print(json.dumps({"config": cfg.name, "env": os.environ.get("AB_TAG", ""), "construct_s": round(t1, 3),
                      "panel_ms": round(tim["panel_ms"], 1), "total_ms": round(tim["total_ms"], 1), "first_total_ms": round(first_ms, 1),
                      "max_w": int(fz.ncols.max())}), flush=True)
    sys.exit(0)
import numpy as np
q, cap = os.environ.get("AB_Q", "3"), os.environ.get("AB_CAP", "17")
variants = sys.argv[2:] or [""]
for name in sys.argv[1].split(","):
    outs = []
    for vi, v in enumerate(variants):
        f = f"/tmp/pab_{name}_{vi}.npz"
        env = dict(os.environ, AB_TAG=v)
        for kv in filter(None, v.split(";")):
            k, val = kv.split("=", 1)
            env[k] = val
        r = subprocess.run([sys.executable, __file__, "--one", name, f, q, cap], env=env, capture_output=True, text=True)
        print(r.stdout.strip() or r.stderr[-2000:], flush=True)
        outs.append(f)
    a = np.load(outs[0])
    for f in outs[1:]:
        b = np.load(f)
        same_r = a["ranks"].shape == b["ranks"].shape and np.array_equal(a["ranks"], b["ranks"])
        same_s = same_r and np.array_equal(a["skel"], b["skel"])
        di = float(np.abs(a["interp"] - b["interp"]).max()) if same_s and a["interp"].shape == b["interp"].shape else None
        print(json.dumps({"config": name, "vs_first": f, "ranks_equal": bool(same_r), "skel_equal": bool(same_s),
                          "interp_maxdiff": di}), flush=True)
