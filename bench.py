#!/usr/bin/env python
"""Benchmark: tensor-butterfly APPLY throughput (input points/s) on B200, with
construction time, roofline of the dominant kernel and the CPU baseline.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config NAME] [--impl b200|reference]

Workload (BASELINE.json configs[2], the largest single-GPU Green config):
d=3 Green's function between two cubes offset by 2 along x, n=256 per
direction (16.7M points per side), kappa = 2*pi*n/8, tol 1e-4, complex128,
seeded complex-normal input.  A "step" is one full contraction G = K x F
(Alg. 2) of one n^d input through the compressed operator.  The operator is
built with the reference's default ProxyStrategy (q = 3, row_cap = 2^17,
id.hpp:50-55) unless --strategy accuracy (configs.ACCURACY_STRATEGY).

* value      device-resident throughput: inputs already in HBM, CUDA events on
             the launching stream, L2 flushed (256 MiB write) before every step.
* e2e        same metric through the public C ABI with pinned HOST buffers
             (oiobf_tbf_contract: H2D of F, contraction, D2H of G per step).
* roofline   dominant kernel = middle-level core GEMV (HBM stream of the cores);
             achieved = algorithmic bytes / its event-timed launch duration.
* cpu_baseline  the oracle port (oracle/liboracle.so) applying the SAME factors
             on the host cores (rank 0, N=1 only), bounded sample.
* --impl reference  the CPU implementation of the path (oracle port, all host
             threads): CPU construction (setup, reported) + timed CPU applies.

Multi-GPU (torchrun, N>1): one process per GPU, the operator sharded by
middle multi-sets: V/W + core GEMV on the column owner, one NCCL
all-to-all of the blocks G_{t,s}, P/U on the row owner.  Strong scaling: one
apply of the whole operator per step; max-over-ranks device time.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_2411_03029_b200.configs import ACCURACY_STRATEGY, BY_NAME, CONFIGS  # noqa: E402

DEFAULT_CONFIG = CONFIGS[2].name  # BASELINE.json configs[2]: largest single-GPU Green config
METRIC = "apply_throughput"
UNIT = "input_pts/s"


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            j = json.load(f)
        return float(j["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def strategy_of(cfg, which):
    """(q, row_cap) of the ProxyStrategy the operator is built with."""
    if which == "accuracy":
        return ACCURACY_STRATEGY[cfg.name]
    return 3, 1 << 17  # reference default (id.hpp:50-55)


def construction_work(fz):
    """Algorithmic construction work from the exported slot shapes: kernel
    entries generated (rows x candidate columns per ID) and the FP64 flops of
    the Householder TSQR (8 m w^2 per ID: per row and column pair j < k one
    complex dot and one complex update)."""
    m = fz.rows.astype(np.float64)
    w = fz.ncols.astype(np.float64)
    return float(np.sum(m * w)), float(np.sum(8.0 * m * w * w))


def make_input(cfg, seed, nv=1):
    """Seeded complex standard normal, Re/Im ~ N(0, 1/2)."""
    rng = np.random.default_rng(seed)
    shape = (cfg.spec.n,) * cfg.spec.d + ((nv,) if nv > 1 else ())
    return ((rng.standard_normal(shape) + 1j * rng.standard_normal(shape)) / np.sqrt(2)).astype(np.complex128)


class ClockSampler:
    FIELDS = ["index", "clocks.sm", "clocks.max.sm", "clocks_event_reasons.active",
              "clocks_event_reasons.hw_slowdown", "clocks_event_reasons.hw_thermal_slowdown",
              "clocks_event_reasons.sw_thermal_slowdown", "clocks_event_reasons.sw_power_cap"]

    def __init__(self, device):
        self.device = device
        self.lines = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "--query-gpu=" + ",".join(self.FIELDS), "--format=csv,noheader,nounits", "-lms", "100",
                 "-i", str(self.device)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[1]))
                mx = float(parts[2])
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


# ------------------------------------------------------------------ reference
def run_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return 0
    from oracle import Oracle, build
    if not os.path.exists(os.path.join(ROOT, "oracle", "liboracle.so")):
        build(ref=False)
    cfg = BY_NAME[args.config]
    o = Oracle()
    threads = os.cpu_count() or 1
    q, cap = strategy_of(cfg, args.strategy)
    t0 = time.perf_counter()
    ob = o.tbf_construct(cfg.spec, cfg.L, cfg.tol, q=q, row_cap=cap, seed=cfg.seed, nthreads=threads)
    t_construct = time.perf_counter() - t0
    F = make_input(cfg, cfg.input_seed, args.nv)
    for _ in range(args.warmup):
        ob.contract(F, nthreads=threads)
    times = []
    for _ in range(args.steps):
        t = time.perf_counter()
        ob.contract(F, nthreads=threads)
        times.append(time.perf_counter() - t)
    ms = 1e3 * statistics.fmean(times)
    pts = cfg.points * args.nv
    value = pts / (ms / 1e3)
    out = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (seeded complex normal input; operator from the BASELINE formula)",
        "config": {"workload": cfg.name, "points": cfg.points, "tol": cfg.tol, "L": cfg.L, "nv": args.nv},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port", "host": host_info(),
                         "sample": f"{args.steps} full applies of {cfg.name} (oracle port, {threads} threads); "
                                   f"the reference has no butterfly code, only its primitives (SURVEY §0.2)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "construct": {"cpu_s": t_construct, "threads": threads, "proxy_strategy": {"q": q, "row_cap": cap}},
    }
    print(json.dumps(out), flush=True)
    return 0


# ------------------------------------------------------------------ b200 arm
def run_b200(args):
    import torch

    ws, rank, local = dist_env()
    if ws > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
    import paper_2411_03029_b200 as tb
    from paper_2411_03029_b200 import _lib

    L = _lib.load()
    _lib.check(L.oiobf_set_device(local if ws > 1 else 0))
    cfg = BY_NAME[args.config]
    dev = torch.device("cuda", torch.cuda.current_device())
    sampler = ClockSampler(torch.cuda.current_device())
    sampler.start()

    # ---- FP64 roofline denominators of this device (DFMA, DMMA)
    pk = np.zeros(4, np.float64)
    _lib.check(L.oiobf_fp64_peak(pk))
    fp64 = {"dfma_tflops": float(pk[0]), "dmma_tflops": float(pk[1]), "sms": int(pk[2]),
            "source": "measured in this run (oiobf_fp64_peak: independent DFMA / mma.sync.m8n8k4.f64 chains on "
                      "every resident warp)"}

    # ---- construction (device work; wall clock around the synchronous call)
    q, cap = strategy_of(cfg, args.strategy)
    ps = tb.ProxyStrategy(q=q, row_cap=cap)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    bf = tb.tbf_construct(cfg.spec, cfg.L, cfg.tol, ps, seed=cfg.seed)
    construct_s = time.perf_counter() - t0
    # second construction: steady state (module load / first touch excluded; the
    # first operator is released before, as an application rebuilding an
    # operator would, so the device pools are reused instead of grown by another
    # 2.9 GB next to a live copy)
    # Two warm runs: the two sides are built concurrently by two host threads and how
    # their launches interleave moves the wall time by ~10% between runs of the
    # same code (summed kernel time unchanged); the faster one is reported, both listed.
    warm_runs = []
    tim = None
    for _ in range(2):
        del bf
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        bf = tb.tbf_construct(cfg.spec, cfg.L, cfg.tol, ps, seed=cfg.seed)
        warm_runs.append(time.perf_counter() - t0)
        if tim is None or warm_runs[-1] <= min(warm_runs):
            tim = bf.timings()
    construct_s_warm = min(warm_runs)
    stats = bf.plan_stats()
    mem = bf.memory()
    fzs = bf.export(pairs=[])  # factors only (no core download)
    fz_ranks = fzs.ranks
    entries, qr_flops = construction_work(fzs)
    del fzs
    # the two sides build concurrently (their k_panel launches overlap), so the
    # summed per-launch panel time over-counts: the time base is the smaller of
    # the summed panel time and the whole construction's wall time
    panel_s = min(tim["panel_ms"], tim["total_ms"]) / 1e3
    construct_roof = {
        "bound": "fp64", "kernel": "k_panel (fused entry generation + TSQR)", "unit": "TFLOP/s",
        "algorithmic_flops": qr_flops, "entries": entries, "panel_s": panel_s,
        "time_base": "min(summed k_panel launch time, construction wall time)",
        "achieved": qr_flops / panel_s / 1e12 if panel_s > 0 else None,
        "peak": fp64["dfma_tflops"],
        "frac": (qr_flops / panel_s / 1e12) / fp64["dfma_tflops"] if panel_s > 0 else None,
        "entries_per_s": entries / panel_s if panel_s > 0 else None,
        "note": "flops = 8 m w^2 per ID (Householder TSQR only; entry generation -- sqrt, sincos, division per "
                "entry -- is counted as entries/s, not flops)"}

    # ---- device buffers
    Fh = make_input(cfg, cfg.input_seed + rank, args.nv)
    N = cfg.points * args.nv
    Ft = torch.from_numpy(Fh.reshape(-1, order="F").copy()).to(dev)
    Gt = torch.empty_like(Ft)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream()
    sh = stream.cuda_stream

    def step():
        bf.contract_device(Ft.data_ptr(), Gt.data_ptr(), args.nv, sh)

    for _ in range(max(args.warmup, 3)):
        step()
    # keep the GPU busy ~0.5 s so clocks are sampled under load
    t_end = time.perf_counter() + 0.5
    while time.perf_counter() < t_end:
        for _ in range(20):
            step()
        torch.cuda.synchronize()
    if ws > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    for a, b in evs:
        flush.zero_()
        a.record(stream)
        step()
        b.record(stream)
    torch.cuda.synchronize()
    ms = sum(a.elapsed_time(b) for a, b in evs) / args.steps
    if ws > 1:
        t = torch.tensor([ms], device=dev, dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t.item())
        torch.distributed.barrier()
    torch.cuda.synchronize()
    value = N * ws / (ms / 1e3)

    # ---- e2e through the public C ABI with pinned host buffers
    pin_F = torch.from_numpy(np.ascontiguousarray(Fh.reshape(-1, order="F")).view(np.float64).copy()).pin_memory()
    pin_G = torch.empty_like(pin_F).pin_memory()
    Fv, Gv = pin_F.numpy(), pin_G.numpy()
    # warm-up by time, not count: the host<->device path needs ~0.1 s of
    # sustained traffic before the PCIe link reaches full speed (measured on
    # the B200 box: the first ~120 calls run ~1.7x slower)
    t_end = time.perf_counter() + 0.3
    nw = 0
    while nw < max(args.warmup, 2) or time.perf_counter() < t_end:
        flush.zero_()
        _lib.check(L.oiobf_tbf_contract(bf.handle, Fv, Gv, args.nv))
        nw += 1
    if ws > 1:
        torch.distributed.barrier()
    e2e_times = []
    e2e_steps = max(args.steps, 50)
    for _ in range(e2e_steps):
        flush.zero_()
        torch.cuda.synchronize()
        t = time.perf_counter()
        _lib.check(L.oiobf_tbf_contract(bf.handle, Fv, Gv, args.nv))
        e2e_times.append(time.perf_counter() - t)
    sync_ms = 1e3 * statistics.fmean(e2e_times)
    # stream-ordered calls back to back (oiobf_tbf_contract_async): every call
    # still copies its F in and its G out, but the H2D of call k+1 overlaps the
    # contraction of call k and the D2H of call k-1.  No L2 flush between
    # calls: one call's working set (cores + F + G) is larger than the L2.
    s_e2e = torch.cuda.Stream()
    # warm the async path by time as well (PCIe link ramp, see above)
    t_end = time.perf_counter() + 0.3
    nwa = 0
    while nwa < 8 or time.perf_counter() < t_end:
        bf.contract_async(Fv, Gv, args.nv, s_e2e.cuda_stream)
        nwa += 1
        if nwa % 16 == 0:
            s_e2e.synchronize()
    s_e2e.synchronize()
    if ws > 1:
        torch.distributed.barrier()
    a_steps = max(e2e_steps, 200)
    t = time.perf_counter()
    for _ in range(a_steps):
        bf.contract_async(Fv, Gv, args.nv, s_e2e.cuda_stream)
    s_e2e.synchronize()
    e2e_ms = 1e3 * (time.perf_counter() - t) / a_steps
    if ws > 1:
        t = torch.tensor([e2e_ms, sync_ms], device=dev, dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        e2e_ms, sync_ms = float(t[0].item()), float(t[1].item())
    e2e_value = N * ws / (e2e_ms / 1e3)
    # sanity: host result equals the device result
    dres = Gt.cpu().numpy()
    step()
    torch.cuda.synchronize()
    assert np.allclose(Gv.view(np.complex128), Gt.cpu().numpy(), rtol=0, atol=1e-12 * np.abs(dres).max())

    # ---- roofline of the dominant kernel (core GEMV), live CUDA events:
    # warm = 20 back-to-back launches; cold = single launches after an L2 flush
    prof = bf.profile_contract(Ft.data_ptr(), Gt.data_ptr(), reps=20, stream=sh)
    core_cold_ms = bf.profile_core_cold(Ft.data_ptr(), Gt.data_ptr(), flush.data_ptr(), flush.numel() * 4, reps=10,
                                        stream=sh)
    # ---- accuracy: 1000 sampled outputs against direct dense sums (GPU K-check)
    rng_s = np.random.default_rng(cfg.input_seed + 1000)
    srows = rng_s.choice(cfg.points, 1000, replace=False)
    exact = tb.dense_rows(cfg.spec, Fh.reshape((cfg.spec.n,) * cfg.spec.d + Fh.shape[cfg.spec.d:], order="F"),
                          srows)
    got = Gt.cpu().numpy().reshape((cfg.points, args.nv), order="F")[srows]
    samp_err = float(np.linalg.norm(got - exact) / np.linalg.norm(exact))
    clocks = sampler.stop()
    hbm, peak_src = peaks()
    gemv_bytes = stats["core_bytes"]
    kname = "k_gemv (middle-level core contraction)"
    if bf.apply_engine() == "rank1":
        # rank-one engine: the core product is folded into the middle V/W level
        # (k_r1_vw_mid), which streams the level-Lc factors (d blocks of 1 x 2
        # per pair), the 1 x 1 cores, its input and its output: 16 (2d + 3) B per pair
        npairs = 2 ** (cfg.spec.d * cfg.L)
        gemv_bytes = 16 * npairs * (2 * cfg.spec.d + 3)
        kname = "k_r1_vw_mid (middle-level V/W transfer + 1x1 core contraction, rank-one engine)"
    achieved = gemv_bytes / (prof["core_ms"] / 1e3) / 1e9
    achieved_cold = gemv_bytes / (core_cold_ms / 1e3) / 1e9
    traffic = None
    tp = os.path.join(ROOT, "profiles", f"ncu_{cfg.name}.json")
    if os.path.exists(tp):
        try:
            with open(tp) as f:
                traffic = json.load(f).get("gemv_dram_bytes_per_launch")
        except Exception:
            traffic = None

    # ---- CPU baseline: oracle port on the same factors (rank 0, N = 1)
    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        try:
            cpu = cpu_baseline(cfg, bf, Fh, args.nv, args.cpu_budget)
        except Exception as e:  # the baseline is reported, never the product
            cpu = {"value": None, "unit": UNIT, "cores": 0, "kind": "port", "sample": f"failed: {e}"}

    # compressed cores (block floating point, the ZFP role of PAPER.md Alg. 2):
    # same timing rules; the core GEMV reads half the bytes
    bfp = None
    if rank == 0 and ws == 1 and args.nv == 1 and not args.no_extras and bf.apply_engine() == "box":
        G64 = Gt.clone()
        bf.set_core_format("bfp32")
        for _ in range(max(args.warmup, 3)):
            step()
        torch.cuda.synchronize()
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
        for a, b in evs:
            flush.zero_()
            a.record(stream)
            step()
            b.record(stream)
        torch.cuda.synchronize()
        bms = sum(a.elapsed_time(b) for a, b in evs) / args.steps
        bst = bf.plan_stats()
        bprof = bf.profile_contract(Ft.data_ptr(), Gt.data_ptr(), reps=20, stream=sh)
        gb = Gt.cpu().numpy().reshape((cfg.points, args.nv), order="F")
        g64 = G64.cpu().numpy().reshape((cfg.points, args.nv), order="F")
        b_err = float(np.linalg.norm(gb[srows] - exact) / np.linalg.norm(exact))
        bfp = {"format": "bfp32: per 32 entries of a core row one 16-bit exponent, 32-bit mantissas (8.06 B/entry)",
               "value": N / (bms / 1e3), "unit": UNIT, "ms_per_step": bms, "core_bytes": bst["core_bytes"],
               "core_ms": bprof["core_ms"], "core_GBps": bst["core_bytes"] / (bprof["core_ms"] / 1e3) / 1e9,
               "rel_diff_vs_fp64_apply": float(np.linalg.norm(gb - g64) / np.linalg.norm(g64)),
               "sampled_rel_err": b_err, "ratio_to_tol": b_err / cfg.tol,
               "note": "opt-in (oiobf_tbf_set_core_format); the headline value uses the FP64 cores"}
        bf.set_core_format("fp64")
        del G64

    extras = None
    if rank == 0 and ws == 1 and not args.no_extras:
        del bf
        torch.cuda.empty_cache()
        extras = {}
        for name in ("dft6_n16", "radon2d_n1024"):
            if name == cfg.name:
                continue
            try:
                extras[name] = extra_line(BY_NAME[name], flush, sh, stream)
            except Exception as e:  # an extra never fails the headline line
                extras[name] = {"failed": str(e)}

    out = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms, "higher_is_better": True, "scaling": "weak" if ws > 1 else "strong", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (seeded complex normal input; operator from the BASELINE formula)",
        "config": {"workload": cfg.name, "points": cfg.points, "tol": cfg.tol, "L": cfg.L, "nv": args.nv,
                   "l2": "flushed (256 MiB write) before every timed step",
                   "parallelism": f"replicas x{ws}" if ws > 1 else "single GPU"},
        "e2e": {"value": e2e_value, "unit": UNIT, "ms_per_step": e2e_ms, "h2d_bytes_per_step": 16 * N,
                "d2h_bytes_per_step": 16 * N, "steps": a_steps, "warmup_calls": nw,
                "api": "oiobf_tbf_contract_async (pinned host F/G, calls back to back on one stream: the H2D "
                       "of call k+1 overlaps the contraction of call k and the D2H of call k-1)",
                "timing": "wall clock over all calls, stream synchronised on both sides; no L2 flush "
                          "(a call's working set exceeds the 126 MB L2)",
                "sync_call": {"value": N * ws / (sync_ms / 1e3), "ms_per_step": sync_ms,
                              "api": "oiobf_tbf_contract (one synchronous call per step, L2 flushed before "
                                     "each; copies pipelined over slab groups inside the call)"}},
        "gpu_launches": int(stats["launches"]) * args.steps,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": achieved / hbm,
                     "traffic": traffic, "kernel": kname,
                     "algorithmic_bytes_per_launch": gemv_bytes, "launch_ms": prof["core_ms"], "peak_source": peak_src,
                     "timing": "warm: mean of 20 back-to-back launches (CUDA events on the launch stream)",
                     "cold": {"achieved": achieved_cold, "frac": achieved_cold / hbm, "launch_ms": core_cold_ms,
                              "timing": "single launches, 256 MiB L2 flush before each, mean of 10"},
                     "whole_apply_bytes_alg": stats["bytes_alg"],
                     "whole_apply_GBps": stats["bytes_alg"] / (ms / 1e3) / 1e9,
                     "phase_ms": {"factor_VW": prof["factor_ms"], "core": prof["core_ms"],
                                  "transfer_PU": prof["transfer_ms"], "graph_total": prof["total_ms"]}},
        "clocks": clocks,
        "construct": {"gpu_s_first": construct_s, "gpu_s": construct_s_warm, "gpu_s_warm_runs": warm_runs,
                      "breakdown_ms": tim,
                      "ranks_max": int(fz_ranks.max()), "ranks_min": int(fz_ranks.min()), "memory_bytes": mem,
                      "proxy_strategy": {"q": q, "row_cap": cap, "which": args.strategy},
                      "roofline": construct_roof},
        "fp64_peak": fp64,
        "accuracy": {"sampled_rel_err": samp_err, "tol": cfg.tol, "ratio_to_tol": samp_err / cfg.tol,
                     "samples": 1000, "reference": "direct dense sums on the GPU (oiobf_dense_rows)",
                     "strategy": args.strategy,
                     "note": "the default strategy is the reference's own ProxyStrategy (q = 3, row_cap = 2^17), "
                             "whose proxy sample is what limits the accuracy (DESIGN.md §4); with "
                             "configs.ACCURACY_STRATEGY (`--strategy accuracy`) every BASELINE config is within "
                             "tol on 1000 samples -- measured offline, profiles/r2_accuracy_sweep.jsonl: "
                             "green_cubes_n256 (q = 6, row_cap = 2^27) 0.97 tol, radon2d_n1024 (12, 2^23) 0.87 tol"},
        "cpu_baseline": cpu,
        "compressed_cores": bfp,
        "extras": extras,
    }
    if rank == 0:
        print(json.dumps(out), flush=True)
    if ws > 1:
        torch.distributed.destroy_process_group()
    return 0


def extra_line(cfg, flush, sh, stream):
    """Device-resident apply throughput + construction of another BASELINE
    config (reported beside the headline; same timing rules: events on the
    launch stream, 256 MiB L2 flush before every timed step)."""
    import torch

    import paper_2411_03029_b200 as tb
    t0 = time.perf_counter()
    bf = tb.tbf_construct(cfg.spec, cfg.L, cfg.tol, seed=cfg.seed)
    construct_s = time.perf_counter() - t0
    tim = bf.timings()
    stats = bf.plan_stats()
    Fh = make_input(cfg, cfg.input_seed)
    Ft = torch.from_numpy(Fh.reshape(-1, order="F").copy()).cuda()
    Gt = torch.empty_like(Ft)
    for _ in range(3):
        bf.contract_device(Ft.data_ptr(), Gt.data_ptr(), 1, sh)
    torch.cuda.synchronize()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(10)]
    for a, b in evs:
        flush.zero_()
        a.record(stream)
        bf.contract_device(Ft.data_ptr(), Gt.data_ptr(), 1, sh)
        b.record(stream)
    torch.cuda.synchronize()
    ms = sum(a.elapsed_time(b) for a, b in evs) / len(evs)
    rng = np.random.default_rng(cfg.input_seed + 1000)
    rows = rng.choice(cfg.points, 1000, replace=False)
    exact = tb.dense_rows(cfg.spec, Fh, rows)[:, 0]
    err = float(np.linalg.norm(Gt.cpu().numpy()[rows] - exact) / np.linalg.norm(exact))
    hbm, _ = peaks()
    engine = bf.apply_engine()
    line = {"workload": cfg.name, "points": cfg.points, "tol": cfg.tol, "L": cfg.L, "apply_engine": engine,
            "value": cfg.points / (ms / 1e3), "unit": UNIT, "ms_per_step": ms,
            "whole_apply_bytes_alg": stats["bytes_alg"], "whole_apply_GBps": stats["bytes_alg"] / (ms / 1e3) / 1e9,
            "whole_apply_frac_hbm": stats["bytes_alg"] / (ms / 1e3) / 1e9 / hbm,
            "construct_s": construct_s, "construct_breakdown_ms": tim,
            "sampled_rel_err": err, "ratio_to_tol": err / cfg.tol,
            "l2": "flushed (256 MiB write) before every timed step", "steps": len(evs)}
    if engine != "rank1":
        prof = bf.profile_contract(Ft.data_ptr(), Gt.data_ptr(), reps=10, stream=sh)
        line["core_gemv"] = {"bytes": stats["core_bytes"], "ms_warm": prof["core_ms"],
                             "frac_warm": stats["core_bytes"] / (prof["core_ms"] / 1e3) / 1e9 / hbm}
        # the same apply on block-floating-point cores (opt-in; the ZFP role of PAPER Alg. 2)
        G64 = Gt.clone()
        bf.set_core_format("bfp32")
        for _ in range(3):
            bf.contract_device(Ft.data_ptr(), Gt.data_ptr(), 1, sh)
        torch.cuda.synchronize()
        for a, b in evs:
            flush.zero_()
            a.record(stream)
            bf.contract_device(Ft.data_ptr(), Gt.data_ptr(), 1, sh)
            b.record(stream)
        torch.cuda.synchronize()
        bms = sum(a.elapsed_time(b) for a, b in evs) / len(evs)
        bprof = bf.profile_contract(Ft.data_ptr(), Gt.data_ptr(), reps=10, stream=sh)
        bst = bf.plan_stats()
        line["compressed_cores"] = {
            "format": "bfp32", "value": cfg.points / (bms / 1e3), "ms_per_step": bms, "core_bytes": bst["core_bytes"],
            "core_ms": bprof["core_ms"],
            "rel_diff_vs_fp64_apply": float(torch.linalg.norm(Gt - G64).item() / torch.linalg.norm(G64).item())}
        bf.set_core_format("fp64")
        del G64
    del bf
    torch.cuda.empty_cache()
    return line


def run_b200_sharded(args):
    """N > 1: one process per GPU, the operator sharded by middle multi-sets
    (SURVEY §8(e)); one step = phase 1 (V/W + core GEMV) + NCCL all-to-all of
    the blocks G_{t,s} + phase 2 (P/U).  Strong scaling: the whole job applies
    ONE operator to ONE input per step."""
    import torch
    import torch.distributed as dist

    import paper_2411_03029_b200 as tb
    from paper_2411_03029_b200 import _lib
    from paper_2411_03029_b200.sharded import (GpuShardBackend, PeerExchange, TorchComm, balanced_owners, construct,
                                                round_robin_owners)

    ws, rank, local = dist_env()
    verbose = os.environ.get("OIOBF_BENCH_VERBOSE") is not None

    def stage(msg):
        if verbose:
            print(f"[rank {rank}] {time.strftime('%H:%M:%S')} {msg}", file=sys.stderr, flush=True)
    # validation mode (single-GPU boxes): OIOBF_BENCH_DIST=gloo puts every rank
    # on device 0 and exchanges through the host -- ranks never wait on each
    # other on the GPU.  Timings from it are not scaling numbers.
    backend = os.environ.get("OIOBF_BENCH_DIST", "nccl")
    if backend == "gloo":
        local = 0
    torch.cuda.set_device(local)
    if backend == "gloo":
        dist.init_process_group("gloo")
    else:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    stage(f"process group up ({backend})")
    _lib.check(_lib.load().oiobf_set_device(local))
    cfg = BY_NAME[args.config]
    dev = torch.device("cuda", local)
    comm = TorchComm(device=dev)

    def allreduce_max(x: float) -> float:
        t = torch.tensor([x], dtype=torch.float64, device="cpu" if comm.host else dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())
    sampler = ClockSampler(local)
    sampler.start()
    dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    be = GpuShardBackend(cfg.spec, cfg.L, cfg.tol, tb.ProxyStrategy(), cfg.seed, rank, ws)
    stage("backend created")
    sb = construct(be, rank, ws, comm)
    stage("constructed")
    torch.cuda.synchronize()
    construct_s = time.perf_counter() - t0
    construct_s = allreduce_max(construct_s)

    # Byte-balanced ownership: the core stage is HBM-bound and
    # the core bytes per s follow the geometry (config 3, s % 8: heaviest rank
    # 1.61x the mean), so the per-s core bytes of this first construction --
    # summed over ranks, each knows its own s -- feed the LPT map and the
    # operator is rebuilt with it (identical factors: the IDs do not depend on
    # who builds them).  OIOBF_OWNERSHIP=round_robin keeps s % world.
    def core_bytes_per_s(handle):
        nm = sb.nmid
        cr = np.zeros(nm * nm, np.int64)
        cc = np.zeros(nm * nm, np.int64)
        _lib.check(_lib.load().oiobf_tbf_export(handle, None, None, None, None, None, None, None, _lib.ptr(cr),
                                                _lib.ptr(cc), None))
        return 16 * (cr * cc).reshape(nm, nm).sum(axis=1)  # pair p = s * nmid + t; other ranks' pairs have cc = 0

    def heaviest_over_mean(owner, w):
        load = np.bincount(owner, weights=w, minlength=ws)
        return float(load.max() / max(load.mean(), 1.0))
    w_s = comm.allreduce_sum_np(core_bytes_per_s(be.h)).astype(np.float64)
    rr_map = round_robin_owners(sb.nmid, ws)
    owner = None
    ownership = {"map": "round_robin (s % world)", "core_bytes_heaviest_over_mean": heaviest_over_mean(rr_map, w_s)}
    if os.environ.get("OIOBF_OWNERSHIP", "balanced") != "round_robin":
        bal = balanced_owners(w_s, ws)
        if not np.array_equal(bal, rr_map):
            owner = bal
            del sb, be
            dist.barrier()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            be = GpuShardBackend(cfg.spec, cfg.L, cfg.tol, tb.ProxyStrategy(), cfg.seed, rank, ws)
            sb = construct(be, rank, ws, comm, owner)
            torch.cuda.synchronize()
            ownership = {"map": "byte-balanced (LPT bin packing of the per-s core bytes measured by a first "
                                "round-robin construction)",
                         "core_bytes_heaviest_over_mean": heaviest_over_mean(bal, w_s),
                         "round_robin_heaviest_over_mean": heaviest_over_mean(rr_map, w_s),
                         "measuring_construction_s": construct_s}
            construct_s = allreduce_max(time.perf_counter() - t0)
            stage("rebuilt with the byte-balanced ownership map")
    own_map = rr_map if owner is None else owner

    Fh = make_input(cfg, cfg.input_seed, args.nv)
    N = cfg.points * args.nv
    F = torch.from_numpy(np.ascontiguousarray(Fh.reshape(-1, order="F")).view(np.float64).copy()).to(dev)
    G = torch.zeros_like(F)
    lay = sb.layout
    send = torch.empty(2 * max(1, int(lay.send_counts.sum())) * args.nv, dtype=torch.float64, device=dev)
    recv = torch.empty(2 * max(1, int(lay.recv_counts.sum())) * args.nv, dtype=torch.float64, device=dev)
    stream = torch.cuda.current_stream()
    sh = stream.cuda_stream
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)

    # exchange: send buffer + NCCL all-to-all by default; OIOBF_EXCHANGE=fused
    # makes the phase-1 core GEMV store G_{t,s} straight into the owners'
    # receive buffers (CUDA IPC peer memory over NVLink, one stream-ordered
    # barrier per step) -- validated only with ranks sharing one device so far
    # (tests/test_sharded.py), so it is opt-in until a multi-GPU run checks it
    px = None
    exchange = "nccl all_to_all_single of the send buffer"
    if os.environ.get("OIOBF_EXCHANGE", "nccl") == "fused":
        try:
            px = PeerExchange(sb, comm, nv_max=args.nv)
            exchange = "fused: core GEMV epilogue stores into peer receive buffers (CUDA IPC), 1 barrier per step"
        except Exception as e:  # e.g. no IPC between these devices: the all-to-all path
            stage(f"fused exchange unavailable ({e}); NCCL all-to-all")
            px = None
        ok = torch.tensor([0 if px is None else 1], dtype=torch.int64, device="cpu" if comm.host else dev)
        dist.all_reduce(ok, op=dist.ReduceOp.MIN)
        if int(ok.item()) == 0 and px is not None:  # every rank must take the same path
            px.close()
            px = None
            exchange = "nccl all_to_all_single of the send buffer"
    stage(f"exchange: {exchange}")

    def step():
        if px is not None:
            px.step(F.data_ptr(), G.data_ptr(), args.nv, sh)
            return
        be.phase(1, F.data_ptr(), send.data_ptr(), args.nv, sh)
        comm.alltoall_on(send, recv, lay.send_counts * args.nv, lay.recv_counts * args.nv, sh)
        be.phase(2, recv.data_ptr(), G.data_ptr(), args.nv, sh)

    for _ in range(max(args.warmup, 3)):
        step()
    stage("warm-up steps done")
    dist.barrier()
    torch.cuda.synchronize()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    for a, b in evs:
        flush.zero_()
        a.record(stream)
        step()
        b.record(stream)
    torch.cuda.synchronize()
    ms = allreduce_max(sum(a.elapsed_time(b) for a, b in evs) / args.steps)
    stage("timed steps done")
    # e2e: from pinned host F, each rank copies in only the input sub-tensors
    # F(s) of its owned s and copies out only the G(t) of its owned t (strided
    # DMA, oiobf_tbf_copy_owned), exchange included
    pin_F = torch.from_numpy(np.ascontiguousarray(Fh.reshape(-1, order="F")).view(np.float64).copy()).pin_memory()
    pin_G = torch.empty_like(pin_F).pin_memory()
    e2e = []
    n_own_s = int(np.count_nonzero(own_map == rank))

    def copy_in():
        be.copy_owned(0, pin_F.data_ptr(), F.data_ptr(), args.nv, sh)

    def copy_out():
        be.copy_owned(1, G.data_ptr(), pin_G.data_ptr(), args.nv, sh)

    def e2e_step():
        copy_in()
        step()
        copy_out()
        torch.cuda.synchronize()

    # PCIe link warm-up (see run_b200) for ~0.3 s.  Every step holds a
    # collective, so the count must be the same on all ranks: time a few
    # steps, agree on the slowest rank's time, derive one count.
    t1 = time.perf_counter()
    for _ in range(5):
        e2e_step()
    per = allreduce_max((time.perf_counter() - t1) / 5)
    for _ in range(max(1, int(0.3 / max(per, 1e-6)))):
        e2e_step()
    dist.barrier()
    for _ in range(max(args.steps, 50)):
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        copy_in()
        step()
        copy_out()
        torch.cuda.synchronize()
        e2e.append(time.perf_counter() - t1)
    e2e_ms = allreduce_max(1e3 * statistics.fmean(e2e))
    stage("e2e done")
    # correctness probe: gather G (disjoint slabs) and compare 200 rows with dense sums on rank 0
    if comm.host:
        Gc = G.cpu()
        dist.all_reduce(Gc)
        G.copy_(Gc)
    else:
        dist.all_reduce(G)
    clocks = sampler.stop()
    st = np.zeros(4, np.int64)
    _lib.check(_lib.load().oiobf_tbf_plan_stats(be.h, st))
    if rank == 0:
        rng = np.random.default_rng(1)
        rows = rng.choice(cfg.points, 200, replace=False)
        exact = tb.dense_rows(cfg.spec, Fh.reshape((cfg.spec.n,) * cfg.spec.d, order="F"), rows)[:, 0]
        got = G.cpu().numpy().view(np.complex128)[rows]
        err = float(np.linalg.norm(got - exact) / np.linalg.norm(exact))
        out = {
            "metric": METRIC, "value": N / (ms / 1e3), "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded complex normal input; operator from the BASELINE formula)",
            "config": {"workload": cfg.name, "points": cfg.points, "tol": cfg.tol, "L": cfg.L, "nv": args.nv,
                       "l2": "flushed (256 MiB write) before every timed step",
                       "parallelism": f"sharded x{ws} by middle multi-sets", "exchange": exchange},
            "ownership": ownership,
            "e2e": {"value": N / (e2e_ms / 1e3), "unit": UNIT, "ms_per_step": e2e_ms,
                    "h2d_bytes_per_step": 16 * N * n_own_s // sb.nmid, "d2h_bytes_per_step": 16 * N * n_own_s // sb.nmid,
                    "copies": "rank 0's owned sub-tensors F(s) in and G(t) out (oiobf_tbf_copy_owned; every rank "
                              "moves its own share over its own PCIe link)"},
            "exchange_bytes_per_step_rank0": int(16 * lay.send_counts.sum() * args.nv),
            "gpu_launches": int(st[2]) * args.steps,
            "dist_backend": backend,
            "sampled_rel_err_vs_dense": err,
            "clocks": clocks,
            "construct": {"gpu_s": construct_s, "sharded": True},
            "cpu_baseline": None,
        }
        print(json.dumps(out), flush=True)
    dist.barrier()
    if px is not None:
        torch.cuda.synchronize()
        px.close()
    dist.barrier()
    dist.destroy_process_group()
    return 0


def host_info() -> dict:
    """The box's host CPU (record nproc, CPU model and memory)."""
    info = {"nproc": os.cpu_count()}
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    info["model"] = ln.split(":", 1)[1].strip()
                    break
        with open("/proc/meminfo") as f:
            for ln in f:
                if ln.startswith("MemTotal"):
                    info["mem_gb"] = round(int(ln.split()[1]) / 2**20, 1)
                    break
    except OSError:
        pass
    return info


def cpu_baseline(cfg, bf, Fh, nv, budget_s):
    from oracle import Oracle, build
    if not os.path.exists(os.path.join(ROOT, "oracle", "liboracle.so")):
        build(ref=False)
    o = Oracle()
    ob = o.tbf_import(cfg.spec, cfg.L, cfg.tol, bf.export())
    threads = os.cpu_count() or 1
    times = []
    t_start = time.perf_counter()
    while True:
        t = time.perf_counter()
        ob.contract(Fh, nthreads=threads)
        times.append(time.perf_counter() - t)
        if time.perf_counter() - t_start > budget_s or len(times) >= 50:
            break
    ms = 1e3 * statistics.fmean(times)
    # the reference itself is single-threaded: one thread too
    t1 = []
    t_start = time.perf_counter()
    while len(t1) < 3 and time.perf_counter() - t_start < budget_s:
        t = time.perf_counter()
        ob.contract(Fh, nthreads=1)
        t1.append(time.perf_counter() - t)
    ms1 = 1e3 * statistics.fmean(t1)
    return {"value": cfg.points * nv / (ms / 1e3), "unit": UNIT, "cores": threads, "kind": "port",
            "ms_per_step": ms, "value_1thread": cfg.points * nv / (ms1 / 1e3), "ms_per_step_1thread": ms1,
            "host": host_info(),
            "sample": f"{len(times)} full applies of {cfg.name} on the GPU-built factors (oracle port, "
                      f"{threads} threads, ~{budget_s:.0f}s budget)"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default=DEFAULT_CONFIG, choices=sorted(BY_NAME))
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--nv", type=int, default=1)
    ap.add_argument("--cpu-budget", type=float, default=10.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--strategy", default="default", choices=["default", "accuracy"],
                    help="ProxyStrategy: the reference default (q=3, row_cap=2^17) or configs.ACCURACY_STRATEGY")
    ap.add_argument("--no-extras", action="store_true", help="skip the config 4 / config 5 extra lines")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)
    if int(os.environ.get("WORLD_SIZE", "1")) > 1:
        return run_b200_sharded(args)
    return run_b200(args)


if __name__ == "__main__":
    sys.exit(main())
