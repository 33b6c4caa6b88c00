"""ctypes bindings for the oracle (liboracle.so) and the reference harness
(_ref/libref.so).  TEST INFRASTRUCTURE ONLY (see oracle/__init__.py)."""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = os.path.join(HERE, "liboracle.so")
_REF = os.path.join(HERE, "_ref", "libref.so")
REF_SRC = "/root/reference/proj"

i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")
f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")


def build(ref: bool | None = None) -> None:
    """Compile liboracle.so (and _ref/libref.so when the reference exists)."""
    subprocess.run(["make", "-s", "-C", HERE, "liboracle.so"], check=True)
    if ref is None:
        ref = os.path.isdir(REF_SRC)
    if ref:
        subprocess.run(["make", "-s", "-C", HERE, "ref"], check=True)


def ref_available() -> bool:
    return os.path.exists(_REF)


def spec_arrays(spec) -> tuple[np.ndarray, np.ndarray]:
    """(int32[5] = kind, d, n, bitrev, seed ; float64[4] = kappa, offset xyz)."""
    seed = int(getattr(spec, "seed", 0)) & 0xFFFFFFFF
    si = np.array([spec.kind, spec.d, spec.n, int(spec.bitrev), np.int64(seed).astype(np.int32)], dtype=np.int32)
    off = list(spec.offset) + [0.0] * (3 - len(spec.offset))
    sf = np.array([spec.kappa, *off[:3]], dtype=np.float64)
    return si, sf


def cx(a) -> np.ndarray:
    """complex128 array -> contiguous interleaved float64 view (Fortran order for 2-D)."""
    a = np.asarray(a, dtype=np.complex128)
    if a.ndim == 2:
        a = np.asfortranarray(a)
        return a.reshape(-1, order="F").view(np.float64).copy()
    return np.ascontiguousarray(a).reshape(-1).view(np.float64).copy()


def from_cx(buf: np.ndarray, shape=None, order="F") -> np.ndarray:
    z = buf.view(np.complex128)
    return z.reshape(shape, order=order) if shape is not None else z


def _check(lib, rc, errfn):
    if rc != 0:
        raise ValueError(getattr(lib, errfn)().decode())


@dataclass
class Factorization:
    """Flat export of a tensor butterfly (canonical slot order: V/W levels
    0..Lc, then U/P levels 0..Lc; pair p = s*nmid + t)."""
    d: int
    n: int
    L: int
    Lc: int
    nmid: int
    ranks: np.ndarray
    ncols: np.ndarray
    rows: np.ndarray
    gaps: np.ndarray
    flags: np.ndarray
    skel: np.ndarray
    interp: np.ndarray
    perm: np.ndarray
    cores: np.ndarray
    core_rows: np.ndarray
    core_cols: np.ndarray
    r_est: np.ndarray

    def level_counts(self):
        out = []
        for sd in range(2):
            for l in range(self.Lc + 1):
                out.append((sd, l, self.nmid * (2 ** (self.d * l)) * self.d * (2 ** (self.Lc - l))))
        return out

    def offsets(self):
        so = np.concatenate([[0], np.cumsum(self.ranks)])
        io = np.concatenate([[0], np.cumsum(self.ranks * self.ncols)])
        po = np.concatenate([[0], np.cumsum(self.ncols)])
        co = np.concatenate([[0], np.cumsum(self.core_rows * self.core_cols)])
        return so, io, po, co


class Oracle:
    def __init__(self, path: str = _LIB):
        if not os.path.exists(path):
            build(ref=False)
        L = self.lib = C.CDLL(path)
        L.oracle_last_error.restype = C.c_char_p
        L.oracle_derive_seed.restype = C.c_uint64
        L.oracle_derive_seed.argtypes = [C.c_uint64, u64p, C.c_int]
        L.oracle_select_proxies_count.argtypes = [C.c_int64, C.c_int64, C.c_int, C.c_uint64, i64p, i64p]
        L.oracle_proxy_lists.argtypes = [C.c_int, i64p, i64p, C.c_int, C.c_int64, C.c_int, C.c_int64, C.c_int64,
                                         C.c_uint64, i64p, i64p]
        L.oracle_column_id.argtypes = [C.c_int64, C.c_int64, f64p, C.c_double, C.c_int64, C.c_void_p, C.c_int64,
                                       C.c_double, i64p, i64p, f64p, i64p, i32p, f64p, f64p, i32p]
        L.oracle_kernel_eval.argtypes = [i32p, f64p, C.c_int64, i64p, i64p, f64p]
        L.oracle_unfolding.argtypes = [i32p, f64p, i64p, i64p, C.c_int, f64p, i64p]
        L.oracle_mode_product_blockdiag.argtypes = [C.c_int, i64p, f64p, C.c_int, C.c_int, i64p, i64p, f64p, C.c_int,
                                                    f64p]
        L.oracle_tucker_id.argtypes = [i32p, f64p, i64p, i64p, C.c_double, C.c_int, C.c_int64, C.c_int64, C.c_int64,
                                       C.c_uint64, i64p, i64p, f64p, f64p]
        L.oracle_level_rule.argtypes = [C.c_int64, C.c_int64]
        L.oracle_tbf_construct.argtypes = [i32p, f64p, C.c_int, C.c_double, C.c_int, C.c_int64, C.c_int64, C.c_int64,
                                           C.c_uint64, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_double,
                                           C.POINTER(C.c_void_p)]
        L.oracle_tbf_free.argtypes = [C.c_void_p]
        L.oracle_tbf_import.argtypes = [i32p, f64p, C.c_int, C.c_double, i64p, i64p, i64p, f64p, f64p, i64p, i64p,
                                        C.POINTER(C.c_void_p)]
        L.oracle_tbf_info.argtypes = [C.c_void_p, i64p]
        L.oracle_tbf_export.argtypes = [C.c_void_p, i64p, i64p, i64p, f64p, i32p, i64p, f64p, i64p, f64p, i64p, i64p,
                                        i64p]
        L.oracle_tbf_memory.argtypes = [C.c_void_p, i64p]
        L.oracle_tbf_contract.argtypes = [C.c_void_p, f64p, f64p, C.c_int64, C.c_int]
        L.oracle_dense_rows.argtypes = [i32p, f64p, f64p, C.c_int64, C.c_int64, i64p, f64p, C.c_int]

    def _ck(self, rc):
        _check(self.lib, rc, "oracle_last_error")

    # -- primitives ----------------------------------------------------------
    def derive_seed(self, seed: int, tags) -> int:
        t = np.array(list(tags), dtype=np.uint64)
        if t.size == 0:
            t = np.zeros(1, np.uint64)
            return self.lib.oracle_derive_seed(seed, t, 0)
        return self.lib.oracle_derive_seed(seed, t, len(tags))

    def select_proxies_count(self, extent, count, mode, seed):
        out = np.zeros(max(extent, 1), np.int64)
        n = np.zeros(1, np.int64)
        self._ck(self.lib.oracle_select_proxies_count(extent, count, mode, seed, out, n))
        return out[: n[0]]

    def proxy_lists(self, ranges, skip, per_mode, mode=1, q=3, row_cap=1 << 17, seed=0):
        lo = np.array([r[0] for r in ranges], np.int64)
        hi = np.array([r[1] for r in ranges], np.int64)
        counts = np.zeros(len(ranges), np.int64)
        out = np.zeros(int(np.sum(hi - lo + 1)), np.int64)
        self._ck(self.lib.oracle_proxy_lists(len(ranges), lo, hi, skip, per_mode, mode, q, row_cap, seed, counts, out))
        res, pos = [], 0
        for c in counts:
            res.append(out[pos:pos + c].copy())
            pos += c
        return res

    def column_id(self, A, tol, max_rank=-1, forced_perm=None, forced_rank=-1, tie_eps=1e-12):
        A = np.asarray(A, np.complex128)
        m, n = A.shape
        rank = np.zeros(1, np.int64)
        skel = np.zeros(n, np.int64)
        interp = np.zeros(2 * n * n, np.float64)
        perm = np.zeros(n, np.int64)
        sat = np.zeros(1, np.int32)
        imax = np.zeros(1, np.float64)
        gaps = np.zeros(2, np.float64)
        mism = np.zeros(1, np.int32)
        fp = None
        if forced_perm is not None:
            fpa = np.ascontiguousarray(forced_perm, dtype=np.int64)
            fp = fpa.ctypes.data
        self._ck(self.lib.oracle_column_id(m, n, cx(A), tol, max_rank, fp, forced_rank, tie_eps, rank, skel, interp,
                                           perm, sat, imax, gaps, mism))
        r = int(rank[0])
        return dict(rank=r, skeleton=skel[:r].copy(), interp=from_cx(interp[: 2 * r * n], (r, n)).copy(),
                    perm=perm.copy(), saturated=bool(sat[0]), interp_max_abs=float(imax[0]),
                    min_gap=float(gaps[0]), rank_gap=float(gaps[1]), mismatch=bool(mism[0]))

    def kernel_eval(self, spec, I, J):
        si, sf = spec_arrays(spec)
        I = np.ascontiguousarray(I, np.int64)
        J = np.ascontiguousarray(J, np.int64)
        cnt = I.shape[0]
        out = np.zeros(2 * cnt, np.float64)
        self._ck(self.lib.oracle_kernel_eval(si, sf, cnt, I.reshape(-1), J.reshape(-1), out))
        return from_cx(out)

    def unfolding(self, spec, lists, skip):
        si, sf = spec_arrays(spec)
        counts = np.array([len(l) for l in lists], np.int64)
        flat = np.concatenate([np.asarray(l, np.int64) for l in lists])
        m = int(np.prod([c for p, c in enumerate(counts) if p != skip]))
        out = np.zeros(2 * m * counts[skip], np.float64)
        mo = np.zeros(1, np.int64)
        self._ck(self.lib.oracle_unfolding(si, sf, counts, flat, skip, out, mo))
        return from_cx(out, (m, int(counts[skip])))

    def mode_product_blockdiag(self, T, mode, blocks, transpose=False):
        T = np.asarray(T, np.complex128)
        shape = np.array(T.shape, np.int64)
        br = np.array([b.shape[0] for b in blocks], np.int64)
        bc = np.array([b.shape[1] for b in blocks], np.int64)
        bl = np.concatenate([cx(b) for b in blocks])
        out_total = int(np.sum(bc if transpose else br))
        oshape = list(T.shape)
        oshape[mode - 1] = out_total
        out = np.zeros(2 * int(np.prod(oshape)), np.float64)
        self._ck(self.lib.oracle_mode_product_blockdiag(T.ndim, shape, cx(T.reshape(-1, order="F")), mode, len(blocks),
                                                        br, bc, bl, int(transpose), out))
        return from_cx(out).reshape(oshape, order="F")

    def tucker_id(self, spec, ranges, tol, mode=1, q=3, max_retries=3, row_cap=1 << 17, seed=0):
        si, sf = spec_arrays(spec)
        lo = np.array([r[0] for r in ranges], np.int64)
        hi = np.array([r[1] for r in ranges], np.int64)
        sz = hi - lo + 1
        ranks = np.zeros(len(ranges), np.int64)
        skel = np.zeros(int(sz.sum()), np.int64)
        interp = np.zeros(2 * int(np.sum(sz * sz)), np.float64)
        core = np.zeros(2 * int(np.prod(sz)), np.float64)
        self._ck(self.lib.oracle_tucker_id(si, sf, lo, hi, tol, mode, q, max_retries, row_cap, seed, ranks, skel,
                                           interp, core))
        return _unpack_tucker(ranks, sz, skel, interp, core)

    def level_rule(self, n, cb=8):
        return self.lib.oracle_level_rule(n, cb)

    # -- butterfly -------------------------------------------------------------
    def tbf_construct(self, spec, L, tol, mode=1, q=3, max_retries=3, row_cap=1 << 17, seed=0, nthreads=0,
                      replay: Factorization | None = None, tie_eps=1e-12):
        si, sf = spec_arrays(spec)
        if nthreads <= 0:
            nthreads = os.cpu_count() or 1
        h = C.c_void_p()
        fr = po = fp = None
        keep = []
        if replay is not None:
            fra = np.ascontiguousarray(replay.ranks, np.int64)
            poa = np.concatenate([[0], np.cumsum(replay.ncols)[:-1]]).astype(np.int64)
            fpa = np.ascontiguousarray(replay.perm, np.int64)
            if fpa.size == 0:
                fpa = np.zeros(1, np.int64)
            keep = [fra, poa, fpa]
            fr, po, fp = fra.ctypes.data, poa.ctypes.data, fpa.ctypes.data
        self._ck(self.lib.oracle_tbf_construct(si, sf, L, tol, mode, q, max_retries, row_cap, seed, nthreads, fr, po,
                                               fp, tie_eps, C.byref(h)))
        del keep
        return OracleTBF(self, h, spec)

    def tbf_import(self, spec, L, tol, fz):
        """Oracle TBF holding exactly the factors of an exported factorization."""
        si, sf = spec_arrays(spec)
        h = C.c_void_p()
        skel = np.ascontiguousarray(fz.skel, np.int64)
        interp = np.ascontiguousarray(np.asarray(fz.interp, np.complex128)).view(np.float64)
        cores = np.ascontiguousarray(np.asarray(fz.cores, np.complex128)).view(np.float64)
        self._ck(self.lib.oracle_tbf_import(si, sf, L, tol, np.ascontiguousarray(fz.ranks, np.int64),
                                            np.ascontiguousarray(fz.ncols, np.int64),
                                            skel if skel.size else np.zeros(1, np.int64),
                                            interp if interp.size else np.zeros(2), cores if cores.size else np.zeros(2),
                                            np.ascontiguousarray(fz.core_rows, np.int64),
                                            np.ascontiguousarray(fz.core_cols, np.int64), C.byref(h)))
        return OracleTBF(self, h, spec)

    def dense_rows(self, spec, F, rows_flat, nthreads=0):
        si, sf = spec_arrays(spec)
        F = np.asarray(F, np.complex128)
        nv = 1 if F.ndim == spec.d else F.shape[-1]
        rows = np.ascontiguousarray(rows_flat, np.int64)
        out = np.zeros(2 * rows.size * nv, np.float64)
        if nthreads <= 0:
            nthreads = os.cpu_count() or 1
        self._ck(self.lib.oracle_dense_rows(si, sf, cx(F.reshape(-1, order="F")), nv, rows.size, rows, out,
                                            nthreads))
        return from_cx(out).reshape((rows.size, nv), order="F")


class OracleTBF:
    def __init__(self, o: Oracle, h, spec):
        self.o, self.h, self.spec = o, h, spec

    def __del__(self):
        try:
            self.o.lib.oracle_tbf_free(self.h)
        except Exception:
            pass

    def info(self):
        info = np.zeros(10, np.int64)
        self.o._ck(self.o.lib.oracle_tbf_info(self.h, info))
        return info

    def export(self) -> Factorization:
        d, n, L, Lc, nmid, ns, nsk, nip, nco, npm = (int(x) for x in self.info())
        ranks, ncols, rows = (np.zeros(ns, np.int64) for _ in range(3))
        gaps = np.zeros(2 * ns, np.float64)
        flags = np.zeros(ns, np.int32)
        skel = np.zeros(max(nsk, 1), np.int64)
        interp = np.zeros(2 * max(nip, 1), np.float64)
        perm = np.zeros(max(npm, 1), np.int64)
        cores = np.zeros(2 * max(nco, 1), np.float64)
        cr = np.zeros(nmid * nmid, np.int64)
        cc = np.zeros(nmid * nmid, np.int64)
        r_est = np.zeros(2 * (Lc + 1), np.int64)
        self.o._ck(self.o.lib.oracle_tbf_export(self.h, ranks, ncols, rows, gaps, flags, skel, interp, perm, cores, cr,
                                                cc, r_est))
        return Factorization(d, n, L, Lc, nmid, ranks, ncols, rows, gaps.reshape(ns, 2), flags, skel[:nsk],
                             from_cx(interp)[:nip], perm[:npm], from_cx(cores)[:nco], cr, cc, r_est)

    def memory(self):
        out = np.zeros(5, np.int64)
        self.o._ck(self.o.lib.oracle_tbf_memory(self.h, out))
        return dict(zip(["V", "W", "U", "P", "cores"], out.tolist()))

    def contract(self, F, nthreads=0):
        F = np.asarray(F, np.complex128)
        d = self.spec.d
        nv = 1 if F.ndim == d else F.shape[-1]
        out = np.zeros(2 * F.size, np.float64)
        if nthreads <= 0:
            nthreads = os.cpu_count() or 1
        self.o._ck(self.o.lib.oracle_tbf_contract(self.h, cx(F.reshape(-1, order="F")), out, nv, nthreads))
        return from_cx(out).reshape(F.shape, order="F")


def _unpack_tucker(ranks, sz, skel, interp, core):
    D = len(ranks)
    sk, fac = [], []
    sp = ip = 0
    for m in range(D):
        r = int(ranks[m])
        sk.append(skel[sp:sp + r].copy())
        sp += r
        fac.append(from_cx(interp[2 * ip: 2 * (ip + r * sz[m])], (r, int(sz[m]))).copy())
        ip += r * int(sz[m])
    ncore = int(np.prod(ranks))
    return dict(ranks=ranks.copy(), skeletons=sk, factors=fac,
                core=from_cx(core[: 2 * ncore]).reshape([int(r) for r in ranks], order="F").copy())


class Ref:
    """The reference's own primitives (oracle/_ref/libref.so)."""

    def __init__(self, path: str = _REF):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} not built (needs /root/reference; run `make -C oracle ref`)")
        L = self.lib = C.CDLL(path)
        L.ref_last_error.restype = C.c_char_p
        L.ref_splitmix_next.restype = C.c_uint64
        L.ref_splitmix_next.argtypes = [u64p]
        L.ref_splitmix_bounded.restype = C.c_uint64
        L.ref_splitmix_bounded.argtypes = [u64p, C.c_uint64]
        L.ref_derive_seed.restype = C.c_uint64
        L.ref_derive_seed.argtypes = [C.c_uint64, u64p, C.c_int]
        L.ref_select_proxies_count.argtypes = [C.c_int64, C.c_int64, C.c_int, C.c_uint64, i64p, i64p]
        L.ref_select_proxies.argtypes = [C.c_int64, C.c_int64, C.c_int, C.c_int64, C.c_uint64, i64p, i64p]
        L.ref_proxy_lists.argtypes = [C.c_int, i64p, i64p, C.c_int, C.c_int64, C.c_int, C.c_int64, C.c_int64,
                                      C.c_uint64, i64p, i64p]
        L.ref_qrcp.argtypes = [C.c_int64, C.c_int64, f64p, C.c_double, C.c_int64, i64p, f64p, i64p, i32p]
        L.ref_column_id.argtypes = [C.c_int64, C.c_int64, f64p, C.c_double, C.c_int64, i64p, i64p, f64p, i32p, f64p]
        L.ref_slot_id.argtypes = [i32p, f64p, i64p, i64p, C.c_int, i64p, C.c_int64, C.c_int64, C.c_int, C.c_int64,
                                  C.c_int64, C.c_uint64, C.c_double, i64p, i64p, i64p, f64p]
        L.ref_subtensor_at.argtypes = [i32p, f64p, i64p, i64p, f64p]
        L.ref_tucker_id.argtypes = [i32p, f64p, i64p, i64p, C.c_double, C.c_int, C.c_int64, C.c_int64, C.c_int64,
                                    C.c_uint64, i64p, i64p, f64p, f64p, i64p]
        L.ref_tucker_contract.argtypes = [i32p, f64p, i64p, i64p, C.c_double, C.c_int, C.c_int64, C.c_int64,
                                          C.c_int64, C.c_uint64, C.c_int64, f64p, f64p]
        L.ref_mode_product_blockdiag.argtypes = [C.c_int, i64p, f64p, C.c_int, C.c_int, i64p, i64p, f64p, C.c_int,
                                                 f64p]

    def _ck(self, rc):
        _check(self.lib, rc, "ref_last_error")

    def splitmix(self, seed, count):
        st = np.array([seed], np.uint64)
        return np.array([self.lib.ref_splitmix_next(st) for _ in range(count)], np.uint64)

    def bounded(self, seed, bound, count):
        st = np.array([seed], np.uint64)
        return np.array([self.lib.ref_splitmix_bounded(st, bound) for _ in range(count)], np.uint64)

    def derive_seed(self, seed, tags):
        t = np.array(list(tags) or [0], dtype=np.uint64)
        return self.lib.ref_derive_seed(seed, t, len(tags))

    def select_proxies_count(self, extent, count, mode, seed):
        out = np.zeros(max(extent, 1), np.int64)
        n = np.zeros(1, np.int64)
        self._ck(self.lib.ref_select_proxies_count(extent, count, mode, seed, out, n))
        return out[: n[0]]

    def select_proxies(self, extent, rank_estimate, mode, q, seed):
        out = np.zeros(max(extent, 1), np.int64)
        n = np.zeros(1, np.int64)
        self._ck(self.lib.ref_select_proxies(extent, rank_estimate, mode, q, seed, out, n))
        return out[: n[0]]

    def proxy_lists(self, ranges, skip, per_mode, mode=1, q=3, row_cap=1 << 17, seed=0):
        lo = np.array([r[0] for r in ranges], np.int64)
        hi = np.array([r[1] for r in ranges], np.int64)
        counts = np.zeros(len(ranges), np.int64)
        out = np.zeros(int(np.sum(hi - lo + 1)), np.int64)
        self._ck(self.lib.ref_proxy_lists(len(ranges), lo, hi, skip, per_mode, mode, q, row_cap, seed, counts, out))
        res, pos = [], 0
        for c in counts:
            res.append(out[pos:pos + c].copy())
            pos += c
        return res

    def qrcp(self, A, tol, limit=None):
        A = np.asarray(A, np.complex128)
        m, n = A.shape
        if limit is None:
            limit = min(m, n)
        perm = np.zeros(n, np.int64)
        r = np.zeros(2 * n * n, np.float64)
        rank = np.zeros(1, np.int64)
        sat = np.zeros(1, np.int32)
        self._ck(self.lib.ref_qrcp(m, n, cx(A), tol, limit, perm, r, rank, sat))
        k = int(rank[0])
        return dict(perm=perm, R=from_cx(r[: 2 * k * n], (k, n)).copy(), rank=k, saturated=bool(sat[0]))

    def column_id(self, A, tol, max_rank=-1):
        A = np.asarray(A, np.complex128)
        m, n = A.shape
        rank = np.zeros(1, np.int64)
        skel = np.zeros(n, np.int64)
        interp = np.zeros(2 * n * n, np.float64)
        sat = np.zeros(1, np.int32)
        imax = np.zeros(1, np.float64)
        self._ck(self.lib.ref_column_id(m, n, cx(A), tol, max_rank, rank, skel, interp, sat, imax))
        r = int(rank[0])
        return dict(rank=r, skeleton=skel[:r].copy(), interp=from_cx(interp[: 2 * r * n], (r, n)).copy(),
                    saturated=bool(sat[0]), interp_max_abs=float(imax[0]))

    def slot_id(self, spec, ranges, skip, target, per_mode, tol, seed, mode=1, q=3, row_cap=1 << 17):
        si, sf = spec_arrays(spec)
        lo = np.array([r[0] for r in ranges], np.int64)
        hi = np.array([r[1] for r in ranges], np.int64)
        t = np.ascontiguousarray(target, np.int64)
        w = t.size
        rows = np.zeros(1, np.int64)
        rank = np.zeros(1, np.int64)
        skel = np.zeros(w, np.int64)
        interp = np.zeros(2 * w * w, np.float64)
        self._ck(self.lib.ref_slot_id(si, sf, lo, hi, skip, t, w, per_mode, mode, q, row_cap, seed, tol, rows, rank,
                                      skel, interp))
        r = int(rank[0])
        return dict(rows=int(rows[0]), rank=r, skeleton=skel[:r].copy(),
                    interp=from_cx(interp[: 2 * r * w], (r, w)).copy())

    def subtensor_at(self, spec, lists):
        si, sf = spec_arrays(spec)
        counts = np.array([len(l) for l in lists], np.int64)
        flat = np.concatenate([np.asarray(l, np.int64) for l in lists])
        out = np.zeros(2 * int(np.prod(counts)), np.float64)
        self._ck(self.lib.ref_subtensor_at(si, sf, counts, flat, out))
        return from_cx(out).reshape([int(c) for c in counts], order="F")

    def tucker_id(self, spec, ranges, tol, mode=1, q=3, max_retries=3, row_cap=1 << 17, seed=0):
        si, sf = spec_arrays(spec)
        lo = np.array([r[0] for r in ranges], np.int64)
        hi = np.array([r[1] for r in ranges], np.int64)
        sz = hi - lo + 1
        ranks = np.zeros(len(ranges), np.int64)
        skel = np.zeros(int(sz.sum()), np.int64)
        interp = np.zeros(2 * int(np.sum(sz * sz)), np.float64)
        core = np.zeros(2 * int(np.prod(sz)), np.float64)
        mem = np.zeros(1, np.int64)
        self._ck(self.lib.ref_tucker_id(si, sf, lo, hi, tol, mode, q, max_retries, row_cap, seed, ranks, skel,
                                        interp, core, mem))
        out = _unpack_tucker(ranks, sz, skel, interp, core)
        out["memory_bytes"] = int(mem[0])
        return out

    def tucker_contract(self, spec, ranges, tol, F, mode=1, q=3, max_retries=3, row_cap=1 << 17, seed=0):
        si, sf = spec_arrays(spec)
        lo = np.array([r[0] for r in ranges], np.int64)
        hi = np.array([r[1] for r in ranges], np.int64)
        F = np.asarray(F, np.complex128)
        d = spec.d
        nv = F.shape[d] if F.ndim == d + 1 else 1
        rows = [int(hi[p] - lo[p] + 1) for p in range(d)]
        g = np.zeros(2 * int(np.prod(rows)) * nv, np.float64)
        self._ck(self.lib.ref_tucker_contract(si, sf, lo, hi, tol, mode, q, max_retries, row_cap, seed, nv,
                                              cx(F.reshape(-1, order="F")), g))
        return from_cx(g).reshape(rows + [nv], order="F")

    def mode_product_blockdiag(self, T, mode, blocks, transpose=False):
        T = np.asarray(T, np.complex128)
        shape = np.array(T.shape, np.int64)
        br = np.array([b.shape[0] for b in blocks], np.int64)
        bc = np.array([b.shape[1] for b in blocks], np.int64)
        bl = np.concatenate([cx(b) for b in blocks])
        out_total = int(np.sum(bc if transpose else br))
        oshape = list(T.shape)
        oshape[mode - 1] = out_total
        out = np.zeros(2 * int(np.prod(oshape)), np.float64)
        self._ck(self.lib.ref_mode_product_blockdiag(T.ndim, shape, cx(T.reshape(-1, order="F")), mode, len(blocks),
                                                     br, bc, bl, int(transpose), out))
        return from_cx(out).reshape(oshape, order="F")
