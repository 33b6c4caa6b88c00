"""Small workload for compute-sanitizer (racecheck / synccheck / memcheck):
construction + apply of a few small butterflies that exercise every kernel
family -- k_panel / k_finish (construction), k_box (d = 3 boxes), k_box2
(d = 2 GEMM boxes), k_gemv and k_gemv_short (core contraction), the rank-one
engine (d = 6 DFT), the host-buffer pipeline and contract_async."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2411_03029_b200 as tb

rng = np.random.default_rng(0)
cases = [(tb.green_cubes(16), 2, 1e-6), (tb.green_cubes(32), 2, 1e-6), (tb.radon2d(64), 2, 1e-6),
         (tb.dft(6, 4), 2, 1e-8), (tb.green_plates(64), 4, 1e-4)]
for spec, L, tol in cases:
    bf = tb.tbf_construct(spec, L, tol, seed=3)
    shape = (spec.n,) * spec.d
    F = rng.standard_normal(shape + (2,)) + 1j * rng.standard_normal(shape + (2,))
    G = bf.contract(F)
    assert np.isfinite(G).all()
    print(spec.describe(), "engine", bf.apply_engine(), "ok", flush=True)
A = rng.standard_normal((300, 40)) + 1j * rng.standard_normal((300, 40))
print("column_id rank", tb.column_id(A, 1e-6).rank)
