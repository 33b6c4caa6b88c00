"""Golden vectors from the reference's own code (tests/golden/make_golden.py runs
oracle/_ref/libref.so = proj/src/{tensor,id}.cpp compiled in place).

CPU: the oracle reproduces every vector bit for bit (the pin that also holds
where /root/reference is absent).  GPU: the CUDA path against the same vectors
(ranks, skeletons, pivots exact; factors to rounding)."""
import os

import numpy as np
import pytest

from paper_2411_03029_b200.configs import green_cubes, green_plates

G = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "reference_primitives.npz"))


def _ragged(flat, off, i):
    return flat[off[i]:off[i + 1]]


def _mats():
    out, pos = [], 0
    for (m, n) in G["cid_shapes"]:
        out.append(G["cid_A"][pos:pos + m * n].reshape((m, n), order="F"))
        pos += m * n
    return out


def _tags():
    return [list(map(int, _ragged(G["derive_tags_flat"], G["derive_tags_off"], i)))
            for i in range(len(G["derive_tags_off"]) - 1)]


# ------------------------------------------------------------------ CPU (oracle)
def test_golden_rng_and_proxies(oracle):
    for a, s in enumerate(G["derive_seeds"]):
        for b, t in enumerate(_tags()):
            assert oracle.derive_seed(int(s), t) == int(G["derive_out"][a, b])
    for i, (e, c, m, s) in enumerate(G["sel_cases"]):
        np.testing.assert_array_equal(oracle.select_proxies_count(int(e), int(c), int(m), int(s)),
                                      _ragged(G["sel_flat"], G["sel_off"], i))
    rpos = lpos = 0
    for i, (nr, skip, per_mode, cap, seed) in enumerate(G["pl_meta"]):
        ranges = [tuple(r) for r in G["pl_ranges"][rpos:rpos + nr]]
        rpos += nr
        lists = oracle.proxy_lists(ranges, int(skip), int(per_mode), mode=1, q=3, row_cap=int(cap), seed=int(seed))
        flat = _ragged(G["pl_flat"], G["pl_flat_off"], i)
        offs = G["pl_list_off"][lpos:lpos + nr + 1]
        lpos += nr + 1
        for p in range(nr):
            np.testing.assert_array_equal(lists[p], flat[offs[p]:offs[p + 1]])


def test_golden_column_ids(oracle):
    for i, (A, tol) in enumerate(zip(_mats(), G["cid_tols"])):
        o = oracle.column_id(A, float(tol))
        assert o["rank"] == G["cid_rank"][i]
        np.testing.assert_array_equal(o["skeleton"], _ragged(G["cid_skel_flat"], G["cid_skel_off"], i))
        gi = G["cid_interp"][G["cid_interp_off"][i]:G["cid_interp_off"][i + 1]]
        np.testing.assert_array_equal(o["interp"].reshape(-1, order="F"), gi)  # bit-exact
        np.testing.assert_array_equal(o["perm"], _ragged(G["qrcp_perm_flat"], G["qrcp_perm_off"], i))


def test_golden_slot_ids_and_tucker(oracle):
    slots = [(green_plates(32), [(1, 32), (1, 32), (17, 32), (1, 8)], 3, list(range(1, 9)), 24, 1e-6, 99),
             (green_cubes(16), [(1, 16), (1, 16), (1, 16), (9, 16), (1, 16), (1, 4)], 5, list(range(1, 5)), 24,
              1e-4, 7)]
    ip = 0
    for i, (spec, ranges, skip, target, per_mode, tol, seed) in enumerate(slots):
        lists = oracle.proxy_lists(ranges, skip, per_mode, seed=seed)
        lists[skip] = np.array(target, np.int64)
        A = oracle.unfolding(spec, lists, skip)
        assert A.shape[0] == G["slot_rows"][i]
        o = oracle.column_id(A, tol)
        assert o["rank"] == G["slot_rank"][i]
        np.testing.assert_array_equal(np.array(target)[o["skeleton"] - 1],
                                      _ragged(G["slot_skel_flat"], G["slot_skel_off"], i))
        n = o["interp"].size
        np.testing.assert_array_equal(o["interp"].reshape(-1, order="F"), G["slot_interp"][ip:ip + n])
        ip += n
    t = oracle.tucker_id(green_plates(16), [(1, 8), (1, 8), (9, 16), (1, 8)], 1e-6, seed=3)
    np.testing.assert_array_equal(t["ranks"], G["tucker_ranks"])
    np.testing.assert_array_equal(np.asarray(t["core"]).reshape(-1, order="F"), G["tucker_core"])


def test_golden_mode_product(oracle):
    T = G["mp_T"].reshape((6, 5, 4), order="F")
    b = G["mp_blocks"]
    blocks = [b[:6].reshape((3, 2), order="F"), b[6:12].reshape((2, 3), order="F")]
    np.testing.assert_array_equal(oracle.mode_product_blockdiag(T, 2, blocks).reshape(-1, order="F"), G["mp_out"])


# ------------------------------------------------------------- GPU (CUDA path)
@pytest.mark.gpu
def test_golden_on_device():
    import paper_2411_03029_b200 as tb
    for a, s in enumerate(G["derive_seeds"]):
        for b, t in enumerate(_tags()):
            assert tb.derive_seed(int(s), t) == int(G["derive_out"][a, b])
    for i, (e, c, m, s) in enumerate(G["sel_cases"]):
        np.testing.assert_array_equal(tb.select_proxies_count(int(e), int(c), int(m), int(s)),
                                      _ragged(G["sel_flat"], G["sel_off"], i))
    ids = tb.column_id_batch(_mats(), float(G["cid_tols"][0]))
    for i, (A, tol) in enumerate(zip(_mats(), G["cid_tols"])):
        c = tb.column_id_batch([A], float(tol))[0]
        assert c.rank == G["cid_rank"][i]
        np.testing.assert_array_equal(c.skeleton, _ragged(G["cid_skel_flat"], G["cid_skel_off"], i))
        gi = G["cid_interp"][G["cid_interp_off"][i]:G["cid_interp_off"][i + 1]].reshape((c.rank, A.shape[1]),
                                                                                        order="F")
        # interpolation matrices agree up to the conditioning of R11 (reconstruction check, as for the oracle)
        recon = A[:, c.skeleton - 1] @ (c.interp - gi)
        assert np.linalg.norm(recon) <= 1e-12 * max(np.linalg.norm(A), 1e-300)
    assert len(ids) == len(_mats())
    T = G["mp_T"].reshape((6, 5, 4), order="F")
    b = G["mp_blocks"]
    blocks = [b[:6].reshape((3, 2), order="F"), b[6:12].reshape((2, 3), order="F")]
    out = tb.mode_product_blockdiag(T, 2, blocks).reshape(-1, order="F")
    assert np.max(np.abs(out - G["mp_out"])) <= 1e-13 * np.max(np.abs(G["mp_out"]))
