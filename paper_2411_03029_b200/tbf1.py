"""TBF1 file format — pure-Python reader.

Written by ``oiobf_tbf_save`` (C ABI); read back on the GPU by
``oiobf_tbf_load`` and here, without a GPU, so a factorization built once can
be inspected or applied by another process (the CPU oracle in the tests).
Little-endian throughout:

  "TBF1"  u32 version
  kernel: i32 kind, i32 d, i64 n, i32 bitrev, u32 seed, f64 kappa, f64 offset[3]
  i32 L, f64 tol
  proxies: i32 mode, i64 q, i64 max_retries, i64 row_cap;  u64 seed
  per level (V/W l = 0..Lc, then U/P l = 0..Lc), canonical slot order
  ((outer * nin + inner) * d + k) * nj + j:
      i64 r_est, nslots, rows, wmax, total_skel, total_interp
      i32 rank[nslots], i32 width[nslots], i32 perm[nslots * wmax]
      i32 skel[total_skel]                (sorted 1-based global indices)
      f64 interp[2 * total_interp]        (r x w column-major per slot)
  i64 npairs, i64 total_core;  i32 R[npairs], i32 C[npairs] (interleaved)
  f64 cores[2 * total_core]               (per pair p = s * nmid + t, row-major R x C)
  u64 FNV-1a checksum of all preceding bytes
"""
from __future__ import annotations

import struct
from dataclasses import dataclass

import numpy as np

from .configs import KernelSpec

MAGIC = b"TBF1"
VERSION = 1


def _fnv1a(data: bytes) -> int:
    """FNV-1a 64 (sequential; ~20 MB/s in Python -- pass verify_checksum=False for big files)."""
    h = 1469598103934665603
    for b in data:
        h = ((h ^ b) * 1099511628211) & 0xFFFFFFFFFFFFFFFF
    return h


@dataclass
class TBF1:
    spec: KernelSpec
    L: int
    tol: float
    proxies: tuple  # (mode, q, max_retries, row_cap)
    seed: int
    levels: list  # per (side, level): dict(r_est, rows, wmax, rank, width, perm, skel, interp)
    core_rows: np.ndarray
    core_cols: np.ndarray
    cores_rowmajor: np.ndarray  # complex128, all pairs concatenated

    @property
    def Lc(self) -> int:
        return self.L // 2


class _Buf:
    def __init__(self, data: bytes):
        self.b, self.o = data, 0

    def take(self, n: int) -> bytes:
        if self.o + n > len(self.b):
            raise ValueError("tbf_load: truncated file")
        out = self.b[self.o:self.o + n]
        self.o += n
        return out

    def s(self, fmt: str):
        v = struct.unpack("<" + fmt, self.take(struct.calcsize("<" + fmt)))
        return v if len(v) > 1 else v[0]

    def arr(self, dtype, count: int) -> np.ndarray:
        dt = np.dtype(dtype).newbyteorder("<")
        return np.frombuffer(self.take(dt.itemsize * count), dtype=dt).copy()


def read_header(path: str):
    """(KernelSpec, L, tol, proxies, seed) from the first bytes only."""
    with open(path, "rb") as f:
        head = f.read(4 + 4 + 4 + 4 + 8 + 4 + 4 + 8 + 24 + 4 + 8 + 4 + 24 + 8)
    if head[:4] != MAGIC:
        raise ValueError("tbf_load: not a TBF1 file")
    r = _Buf(head)
    r.take(4)
    if r.s("I") != VERSION:
        raise ValueError("tbf_load: unsupported TBF1 version")
    kind, d, n, bitrev, kseed = r.s("i"), r.s("i"), r.s("q"), r.s("i"), r.s("I")
    kappa = r.s("d")
    offset = tuple(r.s("ddd"))
    L, tol = r.s("i"), r.s("d")
    proxies = (r.s("i"), r.s("q"), r.s("q"), r.s("q"))
    seed = r.s("Q")
    return KernelSpec(kind, d, n, kappa, offset, bool(bitrev), kseed), L, tol, proxies, seed


def read_tbf1(path: str, verify_checksum: bool = True) -> TBF1:
    data = open(path, "rb").read()
    if len(data) < 12 or data[:4] != MAGIC:
        raise ValueError("tbf_load: not a TBF1 file")
    body, tail = data[:-8], data[-8:]
    if verify_checksum and struct.unpack("<Q", tail)[0] != _fnv1a(body):
        raise ValueError("tbf_load: checksum mismatch")
    r = _Buf(body)
    r.take(4)
    if r.s("I") != VERSION:
        raise ValueError("tbf_load: unsupported TBF1 version")
    kind, d, n, bitrev, kseed = r.s("i"), r.s("i"), r.s("q"), r.s("i"), r.s("I")
    kappa = r.s("d")
    offset = tuple(r.s("ddd"))
    L, tol = r.s("i"), r.s("d")
    proxies = (r.s("i"), r.s("q"), r.s("q"), r.s("q"))
    seed = r.s("Q")
    spec = KernelSpec(kind, d, n, kappa, offset, bool(bitrev), kseed)
    levels = []
    for _side in range(2):
        for _l in range(L // 2 + 1):
            r_est, ns, rows, wmax, tsk, tip = (r.s("q") for _ in range(6))
            rank = r.arr(np.int32, ns)
            width = r.arr(np.int32, ns)
            perm = r.arr(np.int32, ns * wmax)
            skel = r.arr(np.int32, tsk)
            interp = r.arr(np.float64, 2 * tip).view(np.complex128)
            levels.append(dict(r_est=r_est, rows=rows, wmax=wmax, rank=rank, width=width, perm=perm, skel=skel,
                               interp=interp))
    npairs, tc = r.s("q"), r.s("q")
    rc = r.arr(np.int32, 2 * npairs).reshape(npairs, 2)
    cores = r.arr(np.float64, 2 * tc).view(np.complex128)
    if r.o != len(body):
        raise ValueError("tbf_load: trailing bytes")
    return TBF1(spec, L, tol, proxies, seed, levels, rc[:, 0].astype(np.int64), rc[:, 1].astype(np.int64), cores)
