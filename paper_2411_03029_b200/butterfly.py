"""Python mirror of the oiobf construct/apply interface, backed by the sm_100a
library through the C ABI (include/oiobf_b200.h).

Names, argument meaning and error behaviour follow the reference
(/root/reference/proj/include/oiobf/id.hpp, tensor.hpp) and the spec's
tensor-butterfly module:

  column_id(K, tol, max_rank)            id.hpp:40     -> ColumnID
  select_proxies(_count)                 id.hpp:60-66
  derive_seed                            rng.hpp:39
  subtensor_at(spec, rows, cols)         tensor.hpp:96
  mode_product_blockdiag(t, mode, blks)  tensor.hpp:60
  tbf_construct(spec, L, tol, proxies, seed)
  tbf_contract(bf, F)
  tbf_memory(bf)
  tbf_error_estimate(bf, n_samples, seed)

ValueError corresponds to the reference's std::invalid_argument.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib
from .configs import KernelSpec

ALL, UNIFORM_RANDOM, EVENLY_SPACED = 0, 1, 2


@dataclass
class ProxyStrategy:  # id.hpp:50-55
    mode: int = UNIFORM_RANDOM
    q: int = 3
    max_retries: int = 3
    row_cap: int = 1 << 17

    def c(self):
        return _lib.ProxyStrategyC(self.mode, 0, self.q, self.max_retries, self.row_cap)


@dataclass
class ColumnID:  # id.hpp:15-21
    skeleton: np.ndarray
    interp: np.ndarray
    rank: int
    saturated: bool
    interp_max_abs: float
    perm: np.ndarray


def _cx_f(a: np.ndarray) -> np.ndarray:
    """complex array -> first-index-fastest interleaved float64."""
    return np.ascontiguousarray(np.asarray(a, np.complex128).reshape(-1, order="F")).view(np.float64)


def _from_f(buf: np.ndarray, shape) -> np.ndarray:
    return buf.view(np.complex128).reshape(shape, order="F")


def derive_seed(seed: int, tags) -> int:
    L = _lib.load()
    t = np.array(list(tags) or [0], np.uint64)
    return int(L.oiobf_derive_seed(seed, t, len(tags)))


def select_proxies_count(extent: int, count: int, mode: int, seed: int) -> np.ndarray:
    L = _lib.load()
    out = np.zeros(max(extent, 1), np.int64)
    n = np.zeros(1, np.int64)
    _lib.check(L.oiobf_select_proxies_count(extent, count, mode, seed, out, n))
    return out[: n[0]].copy()


def select_proxies(extent: int, rank_estimate: int, strategy: ProxyStrategy, seed: int) -> np.ndarray:
    count = extent if strategy.mode == ALL else min(extent, strategy.q * max(rank_estimate, 1))
    return select_proxies_count(extent, count, strategy.mode, seed)


def column_id_batch(mats, tol: float, max_rank=None) -> list[ColumnID]:
    """Batched column_id on the GPU (id.cpp:124-130)."""
    L = _lib.load()
    mats = [np.asarray(a, np.complex128) for a in mats]
    b = len(mats)
    if b == 0:
        return []
    for a in mats:
        if a.ndim != 2 or a.shape[0] == 0 or a.shape[1] == 0:
            raise ValueError("column_id: empty matrix")
    m = np.array([a.shape[0] for a in mats], np.int64)
    n = np.array([a.shape[1] for a in mats], np.int64)
    a_off = np.concatenate([[0], np.cumsum(m * n)[:-1]]).astype(np.int64)
    A = np.concatenate([_cx_f(a) for a in mats])
    s_off = np.concatenate([[0], np.cumsum(n)[:-1]]).astype(np.int64)
    i_off = np.concatenate([[0], np.cumsum(n * n)[:-1]]).astype(np.int64)
    rank = np.zeros(b, np.int64)
    skel = np.zeros(int(n.sum()), np.int64)
    perm = np.zeros(int(n.sum()), np.int64)
    interp = np.zeros(2 * int(np.sum(n * n)), np.float64)
    sat = np.zeros(b, np.int32)
    imax = np.zeros(b, np.float64)
    mr = None
    if max_rank is not None:
        seq = list(max_rank) if isinstance(max_rank, (list, tuple, np.ndarray)) else [max_rank] * b
        mr = np.array([-1 if x is None else int(x) for x in seq], np.int64)
    _lib.check(L.oiobf_column_id_batch(b, m, n, a_off, A, tol, _lib.ptr(mr), rank, s_off, skel, i_off, interp, perm,
                                       sat, imax))
    out = []
    for q in range(b):
        r, w = int(rank[q]), int(n[q])
        out.append(ColumnID(skel[s_off[q]:s_off[q] + r].copy(),
                            _from_f(interp[2 * i_off[q]: 2 * (i_off[q] + r * w)], (r, w)).copy(), r, bool(sat[q]),
                            float(imax[q]), perm[s_off[q]:s_off[q] + w].copy()))
    return out


def column_id(K, tol: float, max_rank: int | None = None) -> ColumnID:
    return column_id_batch([K], tol, None if max_rank is None else [max_rank])[0]


def subtensor_at(spec: KernelSpec, rows, cols) -> np.ndarray:
    """K(rows, cols) with explicit per-mode lists (tensor.cpp:249-266)."""
    L = _lib.load()
    lists = [np.asarray(l, np.int64) for l in list(rows) + list(cols)]
    if len(lists) != 2 * spec.d:
        raise ValueError("subtensor_at: wrong mode count")
    counts = np.array([len(l) for l in lists], np.int64)
    flat = np.concatenate(lists) if lists else np.zeros(0, np.int64)
    if flat.size == 0:
        flat = np.zeros(1, np.int64)
    out = np.zeros(2 * max(int(np.prod(counts)), 1), np.float64)
    sc = _lib.spec_c(spec)
    _lib.check(L.oiobf_subtensor_at(C.byref(sc), counts, np.ascontiguousarray(flat), out))
    return _from_f(out[: 2 * int(np.prod(counts))], tuple(int(c) for c in counts))


def mode_product_blockdiag(t, mode: int, blocks, transpose_blocks: bool = False) -> np.ndarray:
    L = _lib.load()
    t = np.asarray(t, np.complex128)
    shape = np.array(t.shape, np.int64)
    br = np.array([b.shape[0] for b in blocks], np.int64)
    bc = np.array([b.shape[1] for b in blocks], np.int64)
    bl = np.concatenate([_cx_f(b) for b in blocks])
    oshape = list(t.shape)
    if not (1 <= mode <= t.ndim):
        raise ValueError("mode_product_blockdiag: mode out of range")
    oshape[mode - 1] = int(np.sum(bc if transpose_blocks else br))
    out = np.zeros(2 * max(int(np.prod(oshape)), 1), np.float64)
    _lib.check(L.oiobf_mode_product_blockdiag(t.ndim, shape, _cx_f(t), mode, len(blocks), br, bc, bl,
                                              int(transpose_blocks), out))
    return _from_f(out[: 2 * int(np.prod(oshape))], tuple(oshape))


def dense_rows(spec: KernelSpec, F, rows_flat) -> np.ndarray:
    """K-check on the GPU: exact G(i,:) = sum_j K(i,j) F(j,:) for sampled flat i."""
    L = _lib.load()
    F = np.asarray(F, np.complex128)
    nv = 1 if F.ndim == spec.d else F.shape[-1]
    rows = np.ascontiguousarray(rows_flat, np.int64)
    out = np.zeros(2 * max(rows.size * nv, 1), np.float64)
    sc = _lib.spec_c(spec)
    _lib.check(L.oiobf_dense_rows(C.byref(sc), _cx_f(F), nv, rows.size, rows, out))
    return _from_f(out[: 2 * rows.size * nv], (rows.size, nv))


@dataclass
class Factorization:
    """Flat export (same layout as oracle.bindings.Factorization)."""
    d: int
    n: int
    L: int
    Lc: int
    nmid: int
    ranks: np.ndarray
    ncols: np.ndarray
    rows: np.ndarray
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


class TensorButterfly:
    """Device-resident tensor butterfly."""

    def __init__(self, handle, spec: KernelSpec, L: int, tol: float):
        self._h = handle
        self.spec, self.L, self.tol = spec, L, tol
        self.d, self.n = spec.d, spec.n

    def __del__(self):
        try:
            if self._h:
                _lib.load().oiobf_tbf_destroy(self._h)
                self._h = None
        except Exception:
            pass

    @property
    def handle(self):
        return self._h

    def info(self):
        out = np.zeros(10, np.int64)
        _lib.check(_lib.load().oiobf_tbf_info(self._h, out))
        return out

    def memory(self) -> dict:
        out = np.zeros(5, np.int64)
        _lib.check(_lib.load().oiobf_tbf_memory(self._h, out))
        return dict(zip(["V", "W", "U", "P", "cores"], out.tolist()))

    def timings(self) -> dict:
        out = np.zeros(6, np.float64)
        _lib.check(_lib.load().oiobf_tbf_timings(self._h, out))
        return dict(zip(["proxies_targets_ms", "panel_ms", "finish_ms", "compact_ms", "cores_ms", "total_ms"],
                        out.tolist()))

    def plan_stats(self) -> dict:
        out = np.zeros(4, np.int64)
        _lib.check(_lib.load().oiobf_tbf_plan_stats(self._h, out))
        return dict(bytes_alg=int(out[0]), core_bytes=int(out[1]), launches=int(out[2]), macs=int(out[3]))

    def export(self, pairs=None) -> Factorization:
        """Flat export of every factor.  `pairs` (sorted middle-pair indices
        p = s * nmid + t) restricts the cores to those pairs (core_cols = 0
        elsewhere), for block-wise checks of operators whose cores do not fit
        host memory twice."""
        d, n, L, Lc, nmid, ns, nsk, nip, nco, npm = (int(x) for x in self.info())
        ranks, ncols, rows = (np.zeros(ns, np.int64) for _ in range(3))
        skel = np.zeros(max(nsk, 1), np.int64)
        interp = np.zeros(2 * max(nip, 1), np.float64)
        perm = np.zeros(max(npm, 1), np.int64)
        cr = np.zeros(nmid * nmid, np.int64)
        cc = np.zeros(nmid * nmid, np.int64)
        r_est = np.zeros(2 * (Lc + 1), np.int64)
        P = _lib.ptr
        Lb = _lib.load()
        if pairs is None:
            cores = np.zeros(2 * max(nco, 1), np.float64)
            _lib.check(Lb.oiobf_tbf_export(self._h, P(ranks), P(ncols), P(rows), P(skel), P(interp), P(perm),
                                           P(cores), P(cr), P(cc), P(r_est)))
            cores = cores.view(np.complex128)[:nco]
        else:
            sel = np.ascontiguousarray(np.sort(np.asarray(pairs, np.int64)))
            _lib.check(Lb.oiobf_tbf_export(self._h, P(ranks), P(ncols), P(rows), P(skel), P(interp), P(perm),
                                           None, P(cr), P(cc), P(r_est)))
            tot = int(np.sum(cr[sel] * cc[sel]))
            cores = np.zeros(2 * max(tot, 1), np.float64)
            _lib.check(Lb.oiobf_tbf_export_cores(self._h, sel.size, P(sel), P(cores), P(cr), P(cc)))
            cores = cores.view(np.complex128)[:tot]
        return Factorization(d, n, L, Lc, nmid, ranks, ncols, rows, skel[:nsk], interp.view(np.complex128)[:nip],
                             perm[:npm], cores, cr, cc, r_est)


    def contract(self, F) -> np.ndarray:
        """tbf_contract with host arrays (F: n^d or n^d x nv)."""
        F = np.asarray(F, np.complex128)
        d = self.d
        if F.shape[:d] != (self.n,) * d or F.ndim not in (d, d + 1):
            raise ValueError("tbf_contract: shape mismatch")
        nv = 1 if F.ndim == d else F.shape[d]
        out = np.zeros(2 * F.size, np.float64)
        _lib.check(_lib.load().oiobf_tbf_contract(self._h, _cx_f(F), out, nv))
        return _from_f(out, F.shape)

    def save(self, path: str) -> None:
        """TBF1 file: bit-exact round trip through tbf_load."""
        _lib.check(_lib.load().oiobf_tbf_save(self._h, str(path).encode()))

    def set_core_format(self, fmt: str) -> None:
        """'fp64' (exact, default) | 'bfp32': block-floating-point cores (one
        16-bit exponent per 32 entries of a core row, 32-bit mantissas; half the
        core bytes, ~5e-10 relative per entry) read by the n_v = 1 core GEMV --
        the role ZFP plays in PAPER.md Alg. 2.  The FP64 cores stay resident."""
        code = {"fp64": 0, "bfp32": 1}[fmt]
        _lib.check(_lib.load().oiobf_tbf_set_core_format(self._h, code))

    def set_apply_engine(self, engine: str) -> None:
        """'auto' | 'box' | 'tiny' | 'rank1'.  box: one fused-box launch per
        level (CUDA graph); tiny: thread-per-output engine for d = 6 scale;
        rank1: implicit-geometry engine for butterflies whose every ID has
        rank 1 (two-sided bit-reversed DFT; auto picks it when eligible)."""
        code = {"auto": 0, "box": 1, "tiny": 2, "rank1": 4}[engine]
        _lib.check(_lib.load().oiobf_tbf_set_apply_engine(self._h, code))

    def apply_engine(self) -> str:
        e = C.c_int32(0)
        _lib.check(_lib.load().oiobf_tbf_apply_engine(self._h, C.byref(e)))
        return {1: "box", 2: "tiny", 4: "rank1"}[e.value]

    def contract_async(self, F: np.ndarray, G: np.ndarray, nv: int = 1, stream: int = 0) -> None:
        """Stream-ordered contraction with PINNED host buffers (float64 views of
        complex128 data, e.g. ``torch.empty(..., pin_memory=True).numpy()``):
        enqueues H2D -> contraction -> D2H and returns; `stream` (cudaStream_t)
        waits for G.  Consecutive calls overlap their copies and compute."""
        if nv < 1:
            raise ValueError("tbf_contract: n_v must be positive")
        need = 2 * self.n ** self.d * nv  # float64 words of an n^d x n_v complex tensor
        for name, a in (("F", F), ("G", G)):
            if not isinstance(a, np.ndarray) or a.dtype != np.float64 or not a.flags.c_contiguous:
                raise ValueError(f"tbf_contract_async: {name} must be a C-contiguous float64 array")
            if a.size != need:
                raise ValueError(f"tbf_contract_async: {name} has {a.size} float64 words, expected {need}")
        if not G.flags.writeable:
            raise ValueError("tbf_contract_async: G is read-only")
        _lib.check(_lib.load().oiobf_tbf_contract_async(self._h, F, G, nv, C.c_void_p(stream)))

    def contract_device(self, dF: int, dG: int, nv: int = 1, stream: int = 0) -> None:
        """Device pointers (double2*) already in HBM; enqueued on `stream`."""
        _lib.check(_lib.load().oiobf_tbf_contract_device(self._h, C.c_void_p(dF), C.c_void_p(dG), nv,
                                                         C.c_void_p(stream)))

    def profile_core_cold(self, dF: int, dG: int, flush_ptr: int, flush_bytes: int, reps: int = 10,
                          stream: int = 0) -> float:
        """Mean duration (ms) of the core-contraction phase launched alone with
        a cold L2 (the flush buffer is overwritten before every launch)."""
        out = np.zeros(1, np.float64)
        _lib.check(_lib.load().oiobf_tbf_profile_core_cold(self._h, C.c_void_p(dF), C.c_void_p(dG), reps,
                                                           C.c_void_p(stream), C.c_void_p(flush_ptr), flush_bytes,
                                                           out))
        return float(out[0])

    def profile_contract(self, dF: int, dG: int, reps: int = 10, stream: int = 0) -> dict:
        out = np.zeros(4, np.float64)
        _lib.check(_lib.load().oiobf_tbf_profile_contract(self._h, C.c_void_p(dF), C.c_void_p(dG), reps,
                                                          C.c_void_p(stream), out))
        return dict(factor_ms=out[0], core_ms=out[1], transfer_ms=out[2], total_ms=out[3])


def tbf_construct(spec: KernelSpec, L: int, tol: float, proxies: ProxyStrategy | None = None,
                  seed: int = 0) -> TensorButterfly:
    Lb = _lib.load()
    proxies = proxies or ProxyStrategy()
    h = C.c_void_p()
    sc = _lib.spec_c(spec)
    ps = proxies.c()
    _lib.check(Lb.oiobf_tbf_construct(C.byref(sc), L, tol, C.byref(ps), seed, C.byref(h)))
    return TensorButterfly(h, spec, L, tol)


def tbf_load(path: str) -> TensorButterfly:
    """Load a TBF1 file written by TensorButterfly.save onto the current device."""
    from .tbf1 import read_header
    spec, L, tol, _, _ = read_header(path)  # the library parses the rest and verifies the checksum
    h = C.c_void_p()
    _lib.check(_lib.load().oiobf_tbf_load(str(path).encode(), C.byref(h)))
    return TensorButterfly(h, spec, L, tol)


def tbf_contract(bf: TensorButterfly, F) -> np.ndarray:
    return bf.contract(F)


def tbf_memory(bf: TensorButterfly) -> dict:
    return bf.memory()


def tbf_error_estimate(bf: TensorButterfly, n_samples: int = 10, seed: int = 0) -> float:
    """PAPER.md:515-519 metric: F_e = 1 at n_samples random entries; exact
    K x F_e = sum of those kernel columns, evaluated on the GPU."""
    rng = np.random.default_rng(seed)
    d, n = bf.d, bf.n
    N = n ** d
    cols = rng.choice(N, size=min(n_samples, N), replace=False)
    Fe = np.zeros(N, np.complex128)
    Fe[cols] = 1.0
    Fe = Fe.reshape((n,) * d, order="F")
    G = bf.contract(Fe)
    exact = np.zeros((n,) * d, np.complex128)
    full = [np.arange(1, n + 1)] * d
    for c in cols:
        j = np.unravel_index(int(c), (n,) * d, order="F")
        exact += subtensor_at(bf.spec, full, [[int(x) + 1] for x in j]).reshape((n,) * d, order="F")
    return float(np.linalg.norm(G - exact) / np.linalg.norm(exact))
