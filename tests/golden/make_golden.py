"""Generate tests/golden/reference_primitives.npz from the REFERENCE's own code.

Run in the build container (needs /root/reference): oracle/_ref/libref.so is
the reference's proj/src/{tensor,id}.cpp compiled in place (oracle/Makefile).
Every array in the fixture is an output of that library on seeded inputs; the
inputs are stored next to them.  tests/test_golden.py checks the oracle (CPU)
and the CUDA path (GPU) against these vectors, so the pin also holds where the
reference sources are absent (e.g. on the GPU box).

    python tests/golden/make_golden.py
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import Ref, build  # noqa: E402
from paper_2411_03029_b200.configs import green_cubes, green_plates  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "reference_primitives.npz")


def ragged(lists):
    flat = np.concatenate([np.asarray(x, np.int64) for x in lists]) if lists else np.zeros(0, np.int64)
    off = np.concatenate([[0], np.cumsum([len(x) for x in lists])]).astype(np.int64)
    return flat, off


def low_rank(rng, m, n, r, noise):
    A = (rng.standard_normal((m, r)) + 1j * rng.standard_normal((m, r))) @ (
        rng.standard_normal((r, n)) + 1j * rng.standard_normal((r, n)))
    return A + noise * (rng.standard_normal((m, n)) + 1j * rng.standard_normal((m, n)))


def main():
    build(ref=True)
    ref = Ref()
    rng = np.random.default_rng(20241103)
    g = {}
    # rng.hpp: splitmix64 streams and derive_seed
    seeds = np.array([0, 1, 12345, 2 ** 63 + 5], np.uint64)
    g["splitmix_seeds"] = seeds
    g["splitmix_out"] = np.stack([ref.splitmix(int(s), 8) for s in seeds])
    tags = [[0x56, 1, 2, 3, 0, 1, 0], [0x55, 0, 7, 0, 2, 0, 0], [0x70, 3], [], [2 ** 40, 5, 9]]
    g["derive_seeds"] = seeds
    g["derive_tags_flat"], g["derive_tags_off"] = ragged(tags)
    g["derive_out"] = np.array([[ref.derive_seed(int(s), t) for t in tags] for s in seeds], np.uint64)
    # id.hpp: select_proxies_count (modes All / UniformRandom / EvenlySpaced)
    cases = [(64, 8, 1, 7), (1000, 37, 1, 9), (5, 9, 1, 3), (1 << 20, 64, 1, 11), (1000, 37, 2, 5), (40, 3, 0, 1),
             (16, 16, 1, 2), (3, 1, 1, 4)]
    g["sel_cases"] = np.array(cases, np.int64)
    g["sel_flat"], g["sel_off"] = ragged([ref.select_proxies_count(e, c, m, s) for e, c, m, s in cases])
    # id.cpp:199-231 proxy_lists (row cap halving), d = 2 and d = 3 unfoldings
    pl_cases = [
        ([(1, 32), (1, 32), (9, 16), (1, 32)], 2, 24, 1 << 17, 3),
        ([(1, 64), (1, 64), (1, 64), (17, 32), (1, 64), (1, 64)], 3, 24, 1 << 17, 5),
        ([(1, 16), (1, 16), (1, 16), (1, 16), (5, 8), (1, 16)], 4, 30, 1 << 10, 7),
    ]
    flat, offs, meta = [], [], []
    for ranges, skip, per_mode, cap, seed in pl_cases:
        lists = ref.proxy_lists(ranges, skip, per_mode, mode=1, q=3, row_cap=cap, seed=seed)
        f, o = ragged(lists)
        flat.append(f)
        offs.append(o)
        meta.append([len(ranges), skip, per_mode, cap, seed])
    g["pl_ranges"] = np.array([r for c in pl_cases for r in c[0]], np.int64)
    g["pl_meta"] = np.array(meta, np.int64)
    g["pl_flat"], g["pl_flat_off"] = ragged(flat)
    g["pl_list_off"] = np.concatenate(offs)
    # id.cpp:17-130 qrcp / column_id on seeded matrices (full rank, low rank + noise, exact low rank)
    mats = [low_rank(rng, 60, 12, 12, 0.0), low_rank(rng, 120, 16, 5, 1e-9), low_rank(rng, 80, 10, 3, 0.0),
            low_rank(rng, 200, 24, 9, 1e-7), low_rank(rng, 40, 8, 8, 0.0), low_rank(rng, 300, 32, 20, 1e-12)]
    tols = [1e-6, 1e-6, 1e-10, 1e-5, 1e-8, 1e-9]
    shapes = np.array([m.shape for m in mats], np.int64)
    g["cid_shapes"] = shapes
    g["cid_tols"] = np.array(tols)
    g["cid_A"] = np.concatenate([m.reshape(-1, order="F") for m in mats])
    ranks, skel, interp, perm, R = [], [], [], [], []
    for A, tol in zip(mats, tols):
        c = ref.column_id(A, tol)
        q = ref.qrcp(A, tol)
        ranks.append(c["rank"])
        skel.append(c["skeleton"])
        interp.append(c["interp"].reshape(-1, order="F"))
        perm.append(q["perm"])
        R.append(q["R"].reshape(-1, order="F"))
    g["cid_rank"] = np.array(ranks, np.int64)
    g["cid_skel_flat"], g["cid_skel_off"] = ragged(skel)
    g["cid_interp"] = np.concatenate(interp)
    g["cid_interp_off"] = np.concatenate([[0], np.cumsum([x.size for x in interp])]).astype(np.int64)
    g["qrcp_perm_flat"], g["qrcp_perm_off"] = ragged(perm)
    g["qrcp_R"] = np.concatenate(R)
    g["qrcp_R_off"] = np.concatenate([[0], np.cumsum([x.size for x in R])]).astype(np.int64)
    # one butterfly ID slot each for Green plates / cubes: proxy_lists -> subtensor_at -> unfold -> column_id
    slots = [(green_plates(32), [(1, 32), (1, 32), (17, 32), (1, 8)], 3, list(range(1, 9)), 24, 1e-6, 99),
             (green_cubes(16), [(1, 16), (1, 16), (1, 16), (9, 16), (1, 16), (1, 4)], 5, list(range(1, 5)), 24,
              1e-4, 7)]
    srows, sranks, sskel, sinterp = [], [], [], []
    for spec, ranges, skip, target, per_mode, tol, seed in slots:
        o = ref.slot_id(spec, ranges, skip, target, per_mode, tol, seed)
        srows.append(o["rows"])
        sranks.append(o["rank"])
        sskel.append(o["skeleton"])
        sinterp.append(o["interp"].reshape(-1, order="F"))
    g["slot_rows"] = np.array(srows, np.int64)
    g["slot_rank"] = np.array(sranks, np.int64)
    g["slot_skel_flat"], g["slot_skel_off"] = ragged(sskel)
    g["slot_interp"] = np.concatenate(sinterp)
    # id.hpp:84 tucker_id on a small Green block + tensor.cpp mode_product_blockdiag
    t = ref.tucker_id(green_plates(16), [(1, 8), (1, 8), (9, 16), (1, 8)], 1e-6, seed=3)
    g["tucker_ranks"] = np.asarray(t["ranks"], np.int64)
    g["tucker_core"] = np.asarray(t["core"]).reshape(-1, order="F")
    T = rng.standard_normal((6, 5, 4)) + 1j * rng.standard_normal((6, 5, 4))
    blocks = [rng.standard_normal((3, 2)) + 1j * rng.standard_normal((3, 2)),
              rng.standard_normal((2, 3)) + 1j * rng.standard_normal((2, 3))]
    g["mp_T"] = T.reshape(-1, order="F")
    g["mp_blocks"] = np.concatenate([b.reshape(-1, order="F") for b in blocks])
    g["mp_out"] = ref.mode_product_blockdiag(T, 2, blocks).reshape(-1, order="F")  # mode 2 (1-based): 2 + 3 = 5 columns
    np.savez_compressed(OUT, **g)
    print("wrote", OUT, os.path.getsize(OUT), "bytes")


if __name__ == "__main__":
    main()
