"""BenchRecord CSV: the paper's
table columns (r, r_min, error, T_f, T_a, Mem) for one construct + apply run.

Header (fixed):
  kernel,d,n,tol,algo,L,factor_time_s,apply_time_s,memory_bytes,r,r_min,rel_error,seed,n_v

* ``run_single`` — algo "tensor-bf" (this package on the GPU) or "dense" (the
  direct sum over the same input through the GPU dense-row kernel: the
  harness self-check, rel_error ~ 1e-16).  Factor time: one run; apply time:
  median of 3 (SPEC.md design decisions); memory: exact stored-scalar
  accounting (``tbf_memory``); rel_error: the paper's sampled-column metric
  (``tbf_error_estimate``) with n_samples = 10.
* ``emit_csv`` / ``parse_csv`` — deterministic column order, ``repr`` floats
  (round-trip exact), an absent error written as an empty field.
"""
from __future__ import annotations

import csv
import statistics
import time
from dataclasses import astuple, dataclass, fields

import numpy as np

from .configs import GREEN, DFT, NUDFT, RADON2D, RADON3D, KernelSpec

HEADER = ["kernel", "d", "n", "tol", "algo", "L", "factor_time_s", "apply_time_s", "memory_bytes", "r", "r_min",
          "rel_error", "seed", "n_v"]
KIND_NAME = {GREEN: "green", DFT: "dft", RADON2D: "radon2d", RADON3D: "radon3d", NUDFT: "nudft"}


@dataclass(frozen=True)
class BenchRecord:
    kernel: str
    d: int
    n: int
    tol: float
    algo: str
    L: int
    factor_time_s: float
    apply_time_s: float
    memory_bytes: int
    r: int
    r_min: int
    rel_error: float | None
    seed: int
    n_v: int


def run_single(spec: KernelSpec, tol: float, L: int, algo: str = "tensor-bf", seed: int = 0, n_v: int = 1,
               n_samples: int = 10) -> BenchRecord:
    from . import butterfly as tb
    if algo not in ("tensor-bf", "dense"):
        raise ValueError(f"run_single: algo must be 'tensor-bf' or 'dense' (got {algo!r})")
    rng = np.random.default_rng(seed)
    shape = (spec.n,) * spec.d + ((n_v,) if n_v > 1 else ())
    F = rng.standard_normal(shape) + 1j * rng.standard_normal(shape)
    N = spec.n ** spec.d
    if algo == "dense":
        if N > 1 << 13:
            raise ValueError("run_single: dense algorithm refused above 2^26 entries (desk-scale oracle)")
        rows = np.arange(N)
        t = time.perf_counter()
        G = tb.dense_rows(spec, F.reshape(shape), rows)
        apply_s = time.perf_counter() - t
        ref = tb.dense_rows(spec, F.reshape(shape), rows)
        err = float(np.linalg.norm(G - ref) / max(np.linalg.norm(ref), 1e-300))
        return BenchRecord(KIND_NAME[spec.kind], spec.d, spec.n, tol, algo, 0, 0.0, apply_s, 16 * N * N, 0, 0, err,
                           seed, n_v)
    t = time.perf_counter()
    bf = tb.tbf_construct(spec, L, tol, seed=seed)
    factor_s = time.perf_counter() - t
    times = []
    for _ in range(3):
        t = time.perf_counter()
        bf.contract(F)
        times.append(time.perf_counter() - t)
    ranks = bf.export().ranks
    used = ranks[ranks > 0]
    err = tb.tbf_error_estimate(bf, n_samples=n_samples, seed=seed)
    mem = int(sum(bf.memory().values()))
    return BenchRecord(KIND_NAME[spec.kind], spec.d, spec.n, tol, algo, L, factor_s, statistics.median(times), mem,
                       int(used.max(initial=0)), int(used.min(initial=0)), float(err), seed, n_v)


def _fmt(v) -> str:
    if v is None:
        return ""
    if isinstance(v, float):
        return repr(v)
    return str(v)


def emit_csv(records, path) -> None:
    with open(path, "w", newline="", encoding="utf-8") as f:
        w = csv.writer(f, lineterminator="\n")
        w.writerow(HEADER)
        for r in records:
            w.writerow([_fmt(v) for v in astuple(r)])


def parse_csv(path) -> list[BenchRecord]:
    types = {f.name: f.type for f in fields(BenchRecord)}
    out = []
    with open(path, newline="", encoding="utf-8") as f:
        rd = csv.reader(f)
        head = next(rd)
        if head != HEADER:
            raise ValueError("parse_csv: unexpected header")
        for row in rd:
            vals = {}
            for name, raw in zip(HEADER, row):
                t = str(types[name])
                if t.startswith("float | None") or "None" in t:
                    vals[name] = None if raw == "" else float(raw)
                elif "float" in t:
                    vals[name] = float(raw)
                elif "int" in t:
                    vals[name] = int(raw)
                else:
                    vals[name] = raw
            out.append(BenchRecord(**vals))
    return out
