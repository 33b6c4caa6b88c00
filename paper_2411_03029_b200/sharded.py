"""Sharded (multi-GPU) tensor butterfly — SURVEY.md §8(e), DESIGN.md §7.

One process per GPU.  Rank r owns the middle multi-sets o with owner(o) == r on
both sides (o % world by default, or an explicit ownership map -- e.g. the
byte-balanced `balanced_owners` of the measured per-s core bytes): the V/W IDs of its column multi-sets s and the cores of the
pairs (t, s) it owns, the U/P IDs of its row multi-sets t.  Collectives:

* construction: one all-reduce(max) of the local max rank per (side, level)
  (level-synchronous r_est), one sum-all-reduce of the U-side
  middle ranks (the rows of every block) and one all-to-all of the U-side
  middle skeletons (each rank receives those of the cores it generates);
* apply: V/W levels + core GEMV on the s-owner, ONE all-to-all of the blocks
  G_{t,s} to the t-owner, P/U levels on the t-owner.

The exchange layout (which block goes where, in which order) is pure integer
logic in this module (`exchange_layout`), shared by every backend: the GPU
library (`GpuShardBackend`, C ABI) in production, the CPU oracle in the gloo
tests.  `Comm` abstracts the collectives: `TorchComm` (torch.distributed,
NCCL on GPUs / gloo on CPU) and `run_lockstep` (emulated ranks in one process,
used by the single-GPU test).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib
from .configs import KernelSpec


def owns(outer: int, rank: int, world: int, owner=None) -> bool:
    if world <= 1:
        return True
    return (outer % world if owner is None else int(owner[outer])) == rank


def _owner_map(nmid: int, world: int, owner=None) -> np.ndarray:
    if owner is None:
        return round_robin_owners(nmid, world)
    owner = np.ascontiguousarray(owner, np.int32)
    if owner.shape != (nmid,) or owner.min(initial=0) < 0 or owner.max(initial=0) >= max(world, 1):
        raise ValueError("ownership map: need nmid entries in [0, world)")
    return owner


def round_robin_owners(nmid: int, world: int) -> np.ndarray:
    """The default ownership map: middle multi-set i belongs to rank i % world."""
    return (np.arange(nmid, dtype=np.int64) % max(world, 1)).astype(np.int32)


def balanced_owners(weights, world: int) -> np.ndarray:
    """Byte-balanced ownership map: longest-processing-time bin
    packing of per-multi-set weights (e.g. the core bytes of each s) over
    `world` ranks, every rank getting the same NUMBER of multi-sets where
    world divides it (the input / output slabs stay even).  Deterministic:
    ties go to the lower index / lower rank, so every rank computes the same
    map from the same weights; the round-robin map is returned when it is at
    least as good (tiny nmid)."""
    w = np.asarray(weights, np.float64)
    n = w.size
    if world <= 1:
        return np.zeros(n, np.int32)
    cap = -(-n // world)
    order = sorted(range(n), key=lambda i: (-w[i], i))
    load = [0.0] * world
    cnt = [0] * world
    own = np.zeros(n, np.int32)
    for i in order:
        q = min((r for r in range(world) if cnt[r] < cap), key=lambda r: (load[r], r))
        own[i] = q
        load[q] += w[i]
        cnt[q] += 1
    rr = round_robin_owners(n, world)  # never worse than the default map
    if np.bincount(rr, weights=w, minlength=world).max() <= max(load):
        return rr
    return own


@dataclass
class Layout:
    send_off: np.ndarray  # int64[nmid*nmid], element offsets at nv = 1, -1 = none
    recv_off: np.ndarray
    send_counts: np.ndarray  # int64[world], elements per destination
    recv_counts: np.ndarray  # int64[world], elements per source


def exchange_layout(R: np.ndarray, rank: int, world: int, owner=None) -> Layout:
    """R[t, s] = rows of G_{t,s} (prod of the U-side middle ranks).  The send
    buffer holds, per destination q (ascending), the blocks (t owned by q,
    s owned by me) in (t, s) order; the receive buffer holds, per source q, the
    blocks (t owned by me, s owned by q) in the same (t, s) order, so sender and
    receiver agree without any extra metadata.  `owner`: the ownership map
    (None = round-robin)."""
    R = np.asarray(R, np.int64)
    nmid = R.shape[0]
    own = _owner_map(nmid, world, owner)
    send_off = np.full((nmid, nmid), -1, np.int64)
    recv_off = np.full((nmid, nmid), -1, np.int64)
    send_counts = np.zeros(world, np.int64)
    recv_counts = np.zeros(world, np.int64)
    mine = np.flatnonzero(own == rank)
    cur = 0
    for q in range(world):
        theirs = np.flatnonzero(own == q)
        # send: (t of q, s of me), t-major
        blk = R[np.ix_(theirs, mine)]
        flat = blk.reshape(-1)
        send_off[np.ix_(theirs, mine)] = (cur + np.cumsum(flat) - flat).reshape(blk.shape)
        send_counts[q] = int(flat.sum())
        cur += send_counts[q]
    cur = 0
    for q in range(world):
        theirs = np.flatnonzero(own == q)
        # receive: (t of me, s of q), t-major
        blk = R[np.ix_(mine, theirs)]
        flat = blk.reshape(-1)
        recv_off[np.ix_(mine, theirs)] = (cur + np.cumsum(flat) - flat).reshape(blk.shape)
        recv_counts[q] = int(flat.sum())
        cur += recv_counts[q]
    return Layout(send_off.reshape(-1), recv_off.reshape(-1), send_counts, recv_counts)


class GpuShardBackend:
    """Product backend: the sm_100a library through the C ABI."""

    def __init__(self, spec: KernelSpec, L: int, tol: float, proxies, seed: int, rank: int, world: int):
        Lb = _lib.load()
        _declare(Lb)
        self.spec, self.L = spec, L
        self.d = spec.d
        self.Lc = L // 2
        self.nmid = 2 ** (spec.d * self.Lc)
        h = C.c_void_p()
        sc = _lib.spec_c(spec)
        ps = proxies.c()
        _lib.check(Lb.oiobf_tbf_shard_begin(C.byref(sc), L, tol, C.byref(ps), seed, rank, world, C.byref(h)))
        self.h = h

    def __del__(self):
        try:
            _lib.load().oiobf_tbf_destroy(self.h)
        except Exception:
            pass

    def set_owners(self, owner: np.ndarray):
        """Ownership map of the middle multi-sets (before the first level)."""
        owner = np.ascontiguousarray(owner, np.int32)
        _lib.check(_lib.load().oiobf_tbf_shard_set_owners(self.h, owner))

    def level(self, side: int, l: int, r_est: int) -> int:
        out = C.c_int64()
        _lib.check(_lib.load().oiobf_tbf_shard_level(self.h, side, l, r_est, C.byref(out)))
        return int(out.value)

    def umid_info(self):
        out = np.zeros(2, np.int64)
        _lib.check(_lib.load().oiobf_tbf_umid_info(self.h, out))
        return int(out[0]), int(out[1])

    def umid_export(self, wpad: int):
        n, _ = self.umid_info()
        ranks = np.zeros(n, np.int64)
        skel = np.zeros(n * max(wpad, 1), np.int32)
        _lib.check(_lib.load().oiobf_tbf_umid_export(self.h, ranks, skel, wpad))
        return ranks, skel

    def umid_import(self, ranks: np.ndarray, skel: np.ndarray, wpad: int):
        _lib.check(_lib.load().oiobf_tbf_umid_import(self.h, np.ascontiguousarray(ranks, np.int64),
                                                     np.ascontiguousarray(skel, np.int32), wpad))

    def set_exchange(self, lay: Layout):
        _lib.check(_lib.load().oiobf_tbf_set_exchange(self.h, lay.send_off, lay.recv_off,
                                                      int(lay.send_counts.sum()), int(lay.recv_counts.sum())))

    def copy_owned(self, direction: int, src_ptr: int, dst_ptr: int, nv: int, stream: int = 0):
        """Owned-slab copies (C ABI oiobf_tbf_copy_owned): direction 0 = the
        F(s) sub-tensors of the owned s, host -> device; 1 = the G(t)
        sub-tensors of the owned t, device -> host (strided DMA on `stream`)."""
        _lib.check(_lib.load().oiobf_tbf_copy_owned(self.h, direction, C.c_void_p(src_ptr), C.c_void_p(dst_ptr), nv,
                                                    C.c_void_p(stream)))

    def phase(self, phase: int, src_ptr: int, dst_ptr: int, nv: int, stream: int = 0):
        _lib.check(_lib.load().oiobf_tbf_contract_phase(self.h, phase, C.c_void_p(src_ptr), C.c_void_p(dst_ptr), nv,
                                                        C.c_void_p(stream)))


def _declare(Lb):
    if getattr(Lb, "_shard_declared", False):
        return
    i64p, i32p = _lib.i64p, _lib.i32p
    Lb.oiobf_tbf_shard_begin.argtypes = [C.POINTER(_lib.KernelSpecC), C.c_int32, C.c_double,
                                         C.POINTER(_lib.ProxyStrategyC), C.c_uint64, C.c_int32, C.c_int32,
                                         C.POINTER(C.c_void_p)]
    Lb.oiobf_tbf_shard_set_owners.argtypes = [C.c_void_p, i32p]
    Lb.oiobf_tbf_shard_level.argtypes = [C.c_void_p, C.c_int32, C.c_int32, C.c_int64, C.POINTER(C.c_int64)]
    Lb.oiobf_tbf_umid_info.argtypes = [C.c_void_p, i64p]
    Lb.oiobf_tbf_umid_export.argtypes = [C.c_void_p, i64p, i32p, C.c_int64]
    Lb.oiobf_tbf_umid_import.argtypes = [C.c_void_p, i64p, i32p, C.c_int64]
    Lb.oiobf_tbf_set_exchange.argtypes = [C.c_void_p, i64p, i64p, C.c_int64, C.c_int64]
    Lb.oiobf_tbf_contract_phase.argtypes = [C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p]
    Lb.oiobf_tbf_copy_owned.argtypes = [C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p]
    Lb.oiobf_tbf_set_peer_exchange.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32, C.c_int64]
    Lb.oiobf_device_alloc.argtypes = [C.c_int64, C.POINTER(C.c_void_p)]
    Lb.oiobf_device_free.argtypes = [C.c_void_p]
    Lb.oiobf_ipc_handle.argtypes = [C.c_void_p, C.c_char_p]
    Lb.oiobf_ipc_open.argtypes = [C.c_char_p, C.POINTER(C.c_void_p)]
    Lb.oiobf_ipc_close.argtypes = [C.c_void_p]
    Lb._shard_declared = True


class ShardedButterfly:
    """Step-wise sharded construction/apply for one rank.  Collectives are the
    caller's (`construct` / `contract` below do them with a Comm)."""

    def __init__(self, backend, rank: int, world: int, owner=None):
        self.be, self.rank, self.world = backend, rank, world
        self.nmid, self.d, self.Lc = backend.nmid, backend.d, backend.Lc
        self.layout: Layout | None = None
        self.R = None
        # ownership map of the middle multi-sets (None = round-robin); a map
        # must be the same on every rank and reaches the backend before the
        # first level is built
        self.owner = None if owner is None else _owner_map(self.nmid, world, owner)
        if self.owner is not None:
            backend.set_owners(self.owner)


def on_stream(stream: int, device=None):
    """torch stream context for a raw cudaStream_t (0 = legacy default)."""
    import torch
    if stream:
        return torch.cuda.stream(torch.cuda.ExternalStream(stream, device=device))
    return torch.cuda.stream(torch.cuda.default_stream(device))


class TorchComm:
    """Collectives over torch.distributed (NCCL for CUDA tensors, gloo on CPU)."""

    def __init__(self, group=None, device=None):
        import torch.distributed as dist
        self.dist, self.group, self.device = dist, group, device
        # gloo (validation runs, CPU tests): collectives on host tensors
        self.host = dist.get_backend(group) == "gloo"

    def _dev(self):
        return "cpu" if self.host else self.device

    def allreduce_max_int(self, v: int) -> int:
        import torch
        t = torch.tensor([v], dtype=torch.int64, device=self._dev())
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX, group=self.group)
        return int(t.item())

    def allreduce_sum_np(self, a: np.ndarray) -> np.ndarray:
        """Element-wise sum over ranks, in the array's own integer width
        (int32 skeletons move half the bytes of int64)."""
        import torch
        t = torch.from_numpy(np.ascontiguousarray(a)).to(self._dev())
        self.dist.all_reduce(t, op=self.dist.ReduceOp.SUM, group=self.group)
        return t.cpu().numpy()

    def alltoall_np(self, send: np.ndarray, send_counts, recv_counts) -> np.ndarray:
        """Variable all-to-all of a 1-D integer array (counts in elements)."""
        import torch
        st = torch.from_numpy(np.ascontiguousarray(send)).to(self._dev())
        rt = torch.empty(int(sum(recv_counts)), dtype=st.dtype, device=self._dev())
        self.dist.all_to_all_single(rt, st, [int(c) for c in recv_counts], [int(c) for c in send_counts],
                                    group=self.group)
        return rt.cpu().numpy()

    def allgather_bytes(self, b: bytes) -> list:
        out = [None] * self.dist.get_world_size(self.group)
        self.dist.all_gather_object(out, b, group=self.group)
        return out

    def barrier(self, stream: int = 0):
        """Stream-ordered on NCCL: a one-element all-reduce enqueued on
        `stream` (the raw cudaStream_t the phases run on; 0 = the legacy
        default stream), so it is ordered after this rank's phase-1 stores
        and before its phase 2.  Host-synchronous on gloo (validation runs on
        one GPU)."""
        import torch
        if self.host:
            torch.cuda.synchronize()
            self.dist.barrier(group=self.group)
        else:
            with on_stream(stream, self.device):
                t = torch.zeros(1, dtype=torch.float32, device=self.device)
                self.dist.all_reduce(t, group=self.group)

    def alltoall_on(self, send, recv, send_counts, recv_counts, stream: int = 0):
        """alltoall enqueued on `stream` (ordered between the two phases)."""
        if self.host:
            import torch
            torch.cuda.synchronize()
            self.alltoall(send, recv, send_counts, recv_counts)
            return
        with on_stream(stream, self.device):
            self.alltoall(send, recv, send_counts, recv_counts)

    def alltoall(self, send, recv, send_counts, recv_counts):
        """send/recv: float64 tensors (complex interleaved); counts in complex elements."""
        rs, ss = [2 * int(c) for c in recv_counts], [2 * int(c) for c in send_counts]
        if self.host and send.is_cuda:  # gloo has no CUDA all-to-all: stage through the host
            r = recv.cpu()
            self.dist.all_to_all_single(r, send.cpu(), rs, ss, group=self.group)
            recv.copy_(r)
        else:
            self.dist.all_to_all_single(recv, send, rs, ss, group=self.group)


def peer_offsets(R: np.ndarray, rank: int, world: int, owner=None) -> np.ndarray:
    """For the fused exchange: element offset (n_v = 1) of every block (t, s)
    this rank produces (s owned) inside the receive buffer of its destination
    (the owner of t) -- the destination's own `exchange_layout` receive
    offsets, so sender and receiver agree without exchanging metadata."""
    nmid = R.shape[0]
    own = _owner_map(nmid, world, owner)
    mine = np.flatnonzero(own == rank)
    off = np.full((nmid, nmid), -1, np.int64)
    for q in range(world):
        rq = exchange_layout(R, q, world, owner).recv_off.reshape(nmid, nmid)
        theirs = np.flatnonzero(own == q)
        off[np.ix_(theirs, mine)] = rq[np.ix_(theirs, mine)]
    return off.reshape(-1)


class PeerExchange:
    """Fused exchange (GpuShardBackend): the phase-1 core GEMV stores every
    block G_{t,s} straight into the receive buffer of the owner of t -- peer
    memory over NVLink, mapped through CUDA IPC -- instead of a send buffer
    followed by an all-to-all.  Two receive buffers per rank alternate between
    steps, so one barrier per step (after phase 1) orders everything: a step's
    stores never touch the buffer a peer's phase 2 may still be reading."""

    def __init__(self, sb: "ShardedButterfly", comm, nv_max: int = 1):
        Lb = _lib.load()
        _declare(Lb)
        self.sb, self.comm, self.nv_max = sb, comm, nv_max
        lay = sb.layout
        nbytes = 16 * max(1, int(lay.recv_counts.sum())) * nv_max
        self.own, self.opened = [], []
        for _ in range(2):
            p = C.c_void_p()
            _lib.check(Lb.oiobf_device_alloc(nbytes, C.byref(p)))
            self.own.append(int(p.value))
        hs = b""
        for p in self.own:
            buf = C.create_string_buffer(64)
            _lib.check(Lb.oiobf_ipc_handle(C.c_void_p(p), buf))
            hs += buf.raw
        allh = comm.allgather_bytes(hs)
        world, rank = sb.world, sb.rank
        base = np.zeros(2 * world, np.uint64)
        for q in range(world):
            for par in range(2):
                if q == rank:
                    base[par * world + q] = self.own[par]
                else:
                    p = C.c_void_p()
                    _lib.check(Lb.oiobf_ipc_open(allh[q][64 * par: 64 * (par + 1)], C.byref(p)))
                    self.opened.append(int(p.value))
                    base[par * world + q] = int(p.value)
        off = np.ascontiguousarray(peer_offsets(sb.R, rank, world, sb.owner), np.int64)
        _lib.check(Lb.oiobf_tbf_set_peer_exchange(sb.be.h, C.c_void_p(off.ctypes.data), C.c_void_p(base.ctypes.data),
                                                  world, nv_max))
        self.parity = 0

    def step(self, F_ptr: int, G_ptr: int, nv: int = 1, stream: int = 0):
        buf = self.own[self.parity]
        self.sb.be.phase(1, F_ptr, buf, nv, stream)
        self.comm.barrier(stream)  # on `stream`: every rank's GEMV stores have landed
        self.sb.be.phase(2, buf, G_ptr, nv, stream)
        self.parity ^= 1

    def close(self):
        Lb = _lib.load()
        if self.own:  # the handle goes back to the send buffer + all-to-all path
            _lib.check(Lb.oiobf_tbf_set_peer_exchange(self.sb.be.h, None, None, self.sb.world, 0))
        for p in self.opened:
            Lb.oiobf_ipc_close(C.c_void_p(p))
        for p in self.own:
            Lb.oiobf_device_free(C.c_void_p(p))
        self.opened, self.own = [], []


def construct(backend, rank: int, world: int, comm, owner=None) -> ShardedButterfly:
    """Sharded construction with real collectives (one rank per process).
    `owner`: ownership map of the middle multi-sets, identical on every rank
    (None = round-robin; `balanced_owners` of measured per-s core bytes for a
    byte-balanced apply, see `core_bytes_per_s`)."""
    sb = ShardedButterfly(backend, rank, world, owner)
    for side in (0, 1):
        r_est = 8
        for l in range(sb.Lc + 1):
            local = backend.level(side, l, r_est)
            r_est = max(r_est, comm.allreduce_max_int(local))
    _, local_max = backend.umid_info()
    wpad = max(1, comm.allreduce_max_int(local_max))
    ranks, skel = backend.umid_export(wpad)
    # every block's rows: the exchange layout needs all of them.  A slot is built by exactly one rank
    # (zero elsewhere) and a rank never exceeds wpad, so the sum moves bytes when they fit (the device IDs
    # hold at most 96 columns; config 4: 1e8 slots, 0.1 GB instead of 0.8 GB), 32-bit integers otherwise
    narrow = np.uint8 if wpad < 256 else np.int32
    ranks_all = comm.allreduce_sum_np(ranks.astype(narrow)).astype(np.int64)
    skel_all = exchange_umid_skeletons(skel, rank, world, sb.nmid, sb.d, wpad, comm, sb.owner)
    backend.umid_import(ranks_all, skel_all, wpad)
    _finish_layout(sb, ranks_all)
    return sb


def umid_slots(nmid: int, d: int, t_owner: int, s_owner: int, world: int, owner=None) -> np.ndarray:
    """U-side middle slots (Lc, t, nu = s, k) = (t nmid + s) d + k with t owned
    by `t_owner` and s by `s_owner`, ascending."""
    own = _owner_map(nmid, world, owner)
    t = np.flatnonzero(own == t_owner).astype(np.int64)
    s = np.flatnonzero(own == s_owner).astype(np.int64)
    pairs = (t[:, None] * nmid + s[None, :]).reshape(-1)
    return (pairs[:, None] * d + np.arange(d, dtype=np.int64)[None, :]).reshape(-1)


def exchange_umid_skeletons(skel: np.ndarray, rank: int, world: int, nmid: int, d: int, wpad: int, comm,
                            owner=None) -> np.ndarray:
    """The row skeletons a rank's cores need -- U-side middle slots (t, nu = s)
    for every t and the s it owns -- from their builders (the owners of t) by
    one variable all-to-all: rank q sends rank r the slots (t of q, s of r),
    so every rank receives nmid^2 d wpad / world ints instead of the
    all-reduce of the whole array.  Slots of other s stay zero (unused: the
    cores of pairs with s not owned are generated elsewhere)."""
    skel = np.asarray(skel, np.int32).reshape(-1, wpad)
    send_parts, send_counts = [], []
    for r in range(world):
        part = skel[umid_slots(nmid, d, rank, r, world, owner)].reshape(-1)
        send_parts.append(part)
        send_counts.append(part.size)
    recv_counts = [umid_slots(nmid, d, q, rank, world, owner).size * wpad for q in range(world)]
    recv = comm.alltoall_np(np.concatenate(send_parts) if send_parts else np.zeros(0, np.int32), send_counts,
                            recv_counts)
    out = np.zeros_like(skel)
    off = 0
    for q in range(world):
        sl = umid_slots(nmid, d, q, rank, world, owner)
        out[sl] = recv[off:off + sl.size * wpad].reshape(-1, wpad)
        off += sl.size * wpad
    return out.reshape(-1)


def _finish_layout(sb: ShardedButterfly, ranks_all: np.ndarray):
    nmid, d = sb.nmid, sb.d
    r = ranks_all.reshape(nmid, nmid, d)  # [t, s, k]  (U slot (Lc, t, nu=s, k))
    sb.R = np.prod(r, axis=2)
    sb.layout = exchange_layout(sb.R, sb.rank, sb.world, sb.owner)
    sb.be.set_exchange(sb.layout)


def contract(sb: ShardedButterfly, F, G, comm, nv: int = 1, stream: int = 0):
    """F, G: torch CUDA float64 tensors of 2*n^d*nv (complex interleaved,
    first mode fastest).  G receives this rank's row slabs."""
    import torch
    lay = sb.layout
    send = torch.empty(2 * max(1, int(lay.send_counts.sum())) * nv, dtype=torch.float64, device=F.device)
    recv = torch.empty(2 * max(1, int(lay.recv_counts.sum())) * nv, dtype=torch.float64, device=F.device)
    sb.be.phase(1, F.data_ptr(), send.data_ptr(), nv, stream)
    if hasattr(comm, "alltoall_on"):
        comm.alltoall_on(send, recv, lay.send_counts * nv, lay.recv_counts * nv, stream)
    else:
        comm.alltoall(send, recv, lay.send_counts * nv, lay.recv_counts * nv)
    sb.be.phase(2, recv.data_ptr(), G.data_ptr(), nv, stream)
    return send, recv


def core_bytes_per_s(R: np.ndarray, C: np.ndarray) -> np.ndarray:
    """Core bytes read by the owner of each s: 16 * sum_t R[t, s] * C[t, s]
    (R, C: rows / columns of every core, indexed [t, s]) -- the weights of the
    byte-balanced ownership map."""
    return 16 * (np.asarray(R, np.int64) * np.asarray(C, np.int64)).sum(axis=0)


def run_lockstep(backends: list, F, nv: int = 1, owner=None):
    """Emulate `world` ranks in one process (sequentially, one GPU): same
    steps and the same exchange layout, collectives done by hand.  Returns the
    assembled G (each rank contributes its own row slabs).  Used by the
    single-GPU test of the sharded path; ranks never wait on each other."""
    import torch
    world = len(backends)
    sbs = [ShardedButterfly(b, r, world, owner) for r, b in enumerate(backends)]
    Lc = sbs[0].Lc
    for side in (0, 1):
        r_est = 8
        for l in range(Lc + 1):
            r_est = max([r_est] + [b.level(side, l, r_est) for b in backends])
    wpad = max(1, max(b.umid_info()[1] for b in backends))
    ex = [b.umid_export(wpad) for b in backends]
    ranks_all = sum(e[0] for e in ex)
    skel_all = sum(e[1].astype(np.int64) for e in ex).astype(np.int32)
    for sb in sbs:
        sb.be.umid_import(ranks_all, skel_all, wpad)
        _finish_layout(sb, ranks_all)
    sends = []
    for sb in sbs:
        lay = sb.layout
        send = torch.zeros(2 * max(1, int(lay.send_counts.sum())) * nv, dtype=torch.float64, device=F.device)
        sb.be.phase(1, F.data_ptr(), send.data_ptr(), nv)
        sends.append(send)
    torch.cuda.synchronize()
    G = torch.zeros_like(F)
    for r, sb in enumerate(sbs):
        lay = sb.layout
        parts = []
        for q in range(world):  # block from source q: its send segment for destination r
            qlay = sbs[q].layout
            start = int(qlay.send_counts[:r].sum()) * nv
            parts.append(sends[q][2 * start: 2 * (start + int(qlay.send_counts[r]) * nv)])
        recv = torch.cat(parts) if parts else torch.zeros(2, dtype=torch.float64, device=F.device)
        if recv.numel() == 0:
            recv = torch.zeros(2, dtype=torch.float64, device=F.device)
        assert recv.numel() == 2 * int(lay.recv_counts.sum()) * nv or int(lay.recv_counts.sum()) == 0
        sb.be.phase(2, recv.data_ptr(), G.data_ptr(), nv)
    torch.cuda.synchronize()
    return G
