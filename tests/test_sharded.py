"""Sharded (multi-GPU) path, SURVEY §8(e).

* exchange layout invariants (pure integer logic, CPU)
* the full orchestration (sharded.construct: all-reduce max of r_est per level,
  sum-all-reduce of the U-side middle skeletons; one all-to-all of G_{t,s}) over
  torch.distributed gloo, world 2, with the CPU oracle as compute backend --
  must equal the unsharded oracle bit for bit
* the GPU phases with emulated ranks on one GPU (ranks run sequentially, never
  wait on each other) against the single-GPU contraction
"""
import os
import socket

import numpy as np
import pytest

from paper_2411_03029_b200.configs import green_cubes, green_plates, radon2d
from paper_2411_03029_b200.sharded import (ShardedButterfly, TorchComm, balanced_owners, construct, exchange_layout,
                                            owns)


@pytest.mark.parametrize("mapped", [False, True], ids=["round_robin", "owner_map"])
@pytest.mark.parametrize("world", [1, 2, 3, 4])
def test_exchange_layout_consistent(world, mapped):
    rng = np.random.default_rng(world)
    nmid = 8
    R = rng.integers(0, 30, size=(nmid, nmid))
    owner = rng.integers(0, world, nmid).astype(np.int32) if mapped else None  # uneven on purpose
    lays = [exchange_layout(R, r, world, owner) for r in range(world)]
    for r in range(world):
        for q in range(world):
            assert lays[q].send_counts[r] == lays[r].recv_counts[q]
    seen = np.zeros((nmid, nmid), int)
    for r, lay in enumerate(lays):
        for t in range(nmid):
            for s in range(nmid):
                so, ro = lay.send_off[t * nmid + s], lay.recv_off[t * nmid + s]
                assert (so >= 0) == owns(s, r, world, owner)
                assert (ro >= 0) == owns(t, r, world, owner)
                seen[t, s] += so >= 0
        # blocks are packed back to back in both buffers
        for off, counts in ((lay.send_off, lay.send_counts), (lay.recv_off, lay.recv_counts)):
            pairs = sorted((o, R.flat[i]) for i, o in enumerate(off) if o >= 0)
            cur = 0
            for o, sz in pairs:
                assert o == cur
                cur += sz
            assert cur == counts.sum()
    assert np.all(seen == 1)  # every block is sent exactly once
    # sender and receiver agree on the order inside each (source, destination) segment
    for r in range(world):
        for q in range(world):
            snd = sorted((lays[r].send_off[t * nmid + s], t, s) for t in range(nmid) for s in range(nmid)
                         if owns(s, r, world, owner) and owns(t, q, world, owner))
            rcv = sorted((lays[q].recv_off[t * nmid + s], t, s) for t in range(nmid) for s in range(nmid)
                         if owns(s, r, world, owner) and owns(t, q, world, owner))
            assert [x[1:] for x in snd] == [x[1:] for x in rcv]


def test_balanced_owners():
    """LPT bin packing: even counts, deterministic, no worse than round-robin
    and near the mean on a skewed weight profile."""
    rng = np.random.default_rng(1)
    for nmid, world in ((64, 8), (64, 4), (8, 2), (16, 3)):
        w = rng.integers(20, 80, nmid).astype(np.float64)
        w[: nmid // 4] *= 3  # a heavy corner, like the s nearest the target cube
        own = balanced_owners(w, world)
        assert np.array_equal(own, balanced_owners(w, world))
        cnt = np.bincount(own, minlength=world)
        assert cnt.max() <= -(-nmid // world) and cnt.sum() == nmid
        load = np.bincount(own, weights=w, minlength=world)
        rr = np.bincount(np.arange(nmid) % world, weights=w, minlength=world)
        assert load.max() <= rr.max() + 1e-9
        if nmid >= 8 * world:
            assert load.max() / load.mean() < 1.03


class OracleShardBackend:
    """Test backend: the CPU oracle behind the sharded backend interface."""

    def __init__(self, oracle, spec, L, tol, seed, rank, world):
        self.o, self.spec = oracle, spec
        self.owner = None
        self.tbf = oracle.tbf_construct(spec, L, tol, seed=seed, nthreads=2)
        self.fz = self.tbf.export()
        self.rank, self.world = rank, world
        self.d, self.Lc, self.nmid = spec.d, L // 2, self.fz.nmid
        self.base = {}
        b = 0
        for sd, l, cnt in self.fz.level_counts():
            self.base[(sd, l)] = (b, cnt)
            b += cnt

    def set_owners(self, owner):
        self.owner = np.ascontiguousarray(owner, np.int32)

    def level(self, side, l, r_est):
        assert r_est == self.fz.r_est[side * (self.Lc + 1) + l]
        b, cnt = self.base[(side, l)]
        nin, nj = 2 ** (self.d * l), 2 ** (self.Lc - l)
        outer = np.arange(cnt) // (nj * self.d * nin)
        mine = np.array([owns(int(o), self.rank, self.world, self.owner) for o in outer])
        return int(self.fz.ranks[b:b + cnt][mine].max(initial=0))

    def umid_info(self):
        b, cnt = self.base[(1, self.Lc)]
        t = np.arange(cnt) // (self.nmid * self.d)
        mine = np.array([owns(int(x), self.rank, self.world, self.owner) for x in t])
        return cnt, int(self.fz.ranks[b:b + cnt][mine].max(initial=0))

    def umid_export(self, wpad):
        b, cnt = self.base[(1, self.Lc)]
        so = np.concatenate([[0], np.cumsum(self.fz.ranks)])
        ranks = np.zeros(cnt, np.int64)
        skel = np.zeros(cnt * wpad, np.int32)
        for q in range(cnt):
            if owns(q // (self.nmid * self.d), self.rank, self.world, self.owner):
                r = int(self.fz.ranks[b + q])
                ranks[q] = r
                skel[q * wpad:q * wpad + r] = self.fz.skel[so[b + q]:so[b + q] + r]
        return ranks, skel

    def umid_import(self, ranks, skel, wpad):
        b, cnt = self.base[(1, self.Lc)]
        np.testing.assert_array_equal(ranks, self.fz.ranks[b:b + cnt])

    def set_exchange(self, lay):
        self.lay = lay

    def phase(self, phase, src, nv):
        import ctypes as C
        from oracle.bindings import cx
        L = self.o.lib
        L.oracle_tbf_contract_phase_owned.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_void_p,
                                                      C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_int64,
                                                      C.c_int64, C.c_int]
        N = self.spec.n ** self.spec.d * nv
        se, re = int(self.lay.send_counts.sum()), int(self.lay.recv_counts.sum())
        if phase == 1:
            inp = cx(src)
            out = np.zeros(2 * max(se * nv, 1))
        else:
            inp = src.astype(np.float64) if src.size else np.zeros(2)
            out = np.zeros(2 * N)
        rc = L.oracle_tbf_contract_phase_owned(self.tbf.h, phase, self.rank, self.world,
                                               None if self.owner is None else self.owner.ctypes.data,
                                               inp.ctypes.data, out.ctypes.data, self.lay.send_off.ctypes.data,
                                               self.lay.recv_off.ctypes.data, se, re, nv, 2)
        assert rc == 0, L.oracle_last_error()
        return out


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _gloo_worker(rank, world, port, spec_args, q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import Oracle
        o = Oracle()
        spec, L, tol, seed = spec_args[:4]
        be = OracleShardBackend(o, spec, L, tol, seed, rank, world)
        comm = TorchComm()
        owner = None
        if len(spec_args) > 4 and spec_args[4]:  # byte-balanced map from the core shapes (same on every rank)
            from paper_2411_03029_b200.sharded import core_bytes_per_s
            nm = be.nmid
            cr = np.asarray(be.fz.core_rows).reshape(nm, nm).T  # pair p = s * nmid + t -> [t, s]
            cc = np.asarray(be.fz.core_cols).reshape(nm, nm).T
            owner = balanced_owners(core_bytes_per_s(cr, cc), world)
            assert not np.array_equal(owner, np.arange(nm) % world)
        sb = construct(be, rank, world, comm, owner)
        rng = np.random.default_rng(11)
        F = (rng.standard_normal((spec.n,) * spec.d) + 1j * rng.standard_normal((spec.n,) * spec.d))
        send = torch.from_numpy(be.phase(1, F.reshape(-1, order="F"), 1))
        recv = torch.zeros(2 * max(1, int(sb.layout.recv_counts.sum())), dtype=torch.float64)
        comm.alltoall(send, recv, sb.layout.send_counts, sb.layout.recv_counts)
        G = be.phase(2, recv.numpy()[: 2 * int(sb.layout.recv_counts.sum())], 1)
        Gt = torch.from_numpy(G)
        dist.all_reduce(Gt)  # each rank wrote only its own row slabs (others zero)
        if rank == 0:
            ref = be.tbf.contract(F).reshape(-1, order="F")
            got = Gt.numpy().view(np.complex128)
            q.put(("ok", bool(np.array_equal(got, ref)), float(np.abs(got - ref).max())))
    except Exception as e:  # pragma: no cover - surfaced by the parent
        q.put(("err", repr(e), 0.0))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("spec,L,tol,balanced",
                         [(green_plates(32), 2, 1e-6, False), (green_cubes(16), 2, 1e-4, False),
                          (radon2d(32), 2, 1e-6, False), (green_cubes(16), 2, 1e-4, True)],
                         ids=["plates32", "cubes16", "radon32", "cubes16_balanced"])
def test_sharded_gloo_world2_bitexact(oracle, spec, L, tol, balanced):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gloo_worker, args=(r, 2, port, (spec, L, tol, 5, balanced), q)) for r in range(2)]
    for p in procs:
        p.start()
    res = q.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
    assert res[0] == "ok", res
    assert res[1], f"sharded result differs from the unsharded oracle (max {res[2]})"


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 4])
def test_sharded_gpu_lockstep_balanced(world):
    """Byte-balanced ownership (an LPT map of the per-s core bytes instead of
    s % world) through the device construction, the exchange layout and both
    apply phases: G within 1e-12 of the single-GPU contraction."""
    import torch

    import paper_2411_03029_b200 as tb
    from paper_2411_03029_b200.sharded import GpuShardBackend, core_bytes_per_s, run_lockstep
    spec, L, tol = green_cubes(32), 2, 1e-4
    single = tb.tbf_construct(spec, L, tol, seed=5)
    fz = single.export()
    nm = fz.nmid
    w = core_bytes_per_s(np.asarray(fz.core_rows).reshape(nm, nm).T, np.asarray(fz.core_cols).reshape(nm, nm).T)
    owner = balanced_owners(w, world)
    assert not np.array_equal(owner, np.arange(nm) % world)
    rr = np.bincount(np.arange(nm) % world, weights=w, minlength=world)
    bal = np.bincount(owner, weights=w, minlength=world)
    assert bal.max() <= rr.max()
    rng = np.random.default_rng(3)
    F = rng.standard_normal((32,) * 3) + 1j * rng.standard_normal((32,) * 3)
    G1 = single.contract(F).reshape(-1, order="F")
    Ft = torch.from_numpy(np.ascontiguousarray(F.reshape(-1, order="F")).view(np.float64).copy()).cuda()
    backends = [GpuShardBackend(spec, L, tol, tb.ProxyStrategy(), 5, r, world) for r in range(world)]
    G = run_lockstep(backends, Ft, owner=owner).cpu().numpy().view(np.complex128)
    err = np.linalg.norm(G - G1) / np.linalg.norm(G1)
    assert err < 1e-12, err


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 3])
def test_sharded_gpu_lockstep(world):
    import torch

    import paper_2411_03029_b200 as tb
    from paper_2411_03029_b200.sharded import GpuShardBackend, run_lockstep
    spec, L, tol = green_cubes(16), 2, 1e-4
    single = tb.tbf_construct(spec, L, tol, seed=5)
    rng = np.random.default_rng(3)
    F = rng.standard_normal((16,) * 3) + 1j * rng.standard_normal((16,) * 3)
    G1 = single.contract(F).reshape(-1, order="F")
    Ft = torch.from_numpy(np.ascontiguousarray(F.reshape(-1, order="F")).view(np.float64).copy()).cuda()
    backends = [GpuShardBackend(spec, L, tol, tb.ProxyStrategy(), 5, r, world) for r in range(world)]
    G = run_lockstep(backends, Ft).cpu().numpy().view(np.complex128)
    err = np.linalg.norm(G - G1) / np.linalg.norm(G1)
    assert err < 1e-12, err


@pytest.mark.gpu
@pytest.mark.parametrize("world,balanced", [(2, False), (4, False), (4, True), (3, False)])
def test_sharded_gpu_lockstep_rank_one(world, balanced):
    """d = 6 DFT (every ID of rank 1): the sharded phases run on the rank-one
    engine (local outer indices, pack / unpack around the exchange) when every
    rank owns the same power-of-two number of middle multi-sets -- world 2, 4,
    round-robin or a permuted ownership map -- and fall back to the box engine
    otherwise (world 3); G within 1e-12 of the single-GPU rank-one apply,
    nv = 1 and 2."""
    import ctypes as C

    import torch

    import paper_2411_03029_b200 as tb
    from paper_2411_03029_b200 import _lib
    from paper_2411_03029_b200.configs import dft
    from paper_2411_03029_b200.sharded import GpuShardBackend, run_lockstep
    spec, L, tol = dft(6, 4), 2, 1e-8
    single = tb.tbf_construct(spec, L, tol, seed=5)
    assert single.apply_engine() == "rank1"
    owner = None
    if balanced:  # any equal-count map: a fixed permutation of the round-robin one
        nm = 2 ** (spec.d * (L // 2))
        owner = np.random.default_rng(7).permutation(np.arange(nm) % world).astype(np.int32)
    rng = np.random.default_rng(3)
    for nv in (1, 2):
        shape = (4,) * 6 + ((nv,) if nv > 1 else ())
        F = rng.standard_normal(shape) + 1j * rng.standard_normal(shape)
        G1 = single.contract(F).reshape(-1, order="F")
        Ft = torch.from_numpy(np.ascontiguousarray(F.reshape(-1, order="F")).view(np.float64).copy()).cuda()
        backends = [GpuShardBackend(spec, L, tol, tb.ProxyStrategy(), 5, r, world) for r in range(world)]
        G = run_lockstep(backends, Ft, nv=nv, owner=owner).cpu().numpy().view(np.complex128)
        eng = C.c_int32()
        _lib.check(_lib.load().oiobf_tbf_apply_engine(backends[0].h, C.byref(eng)))
        assert eng.value == (4 if world in (2, 4) else 1), eng.value
        err = np.linalg.norm(G - G1) / np.linalg.norm(G1)
        assert err < 1e-12, (nv, err)


@pytest.mark.gpu
def test_bench_sharded_torchrun_validation():
    """bench.py's N > 1 path end to end under torchrun (world 2), in its
    validation mode: gloo collectives staged through the host and both ranks on
    device 0, so the ranks never wait on each other on the GPU.  Guards the
    collective call order of construction, timed steps and e2e (a per-rank
    time-based warm-up once desynchronised the all-to-all and hung)."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, OIOBF_BENCH_DIST="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), "bench.py", "--gpus", "2",
           "--steps", "2", "--warmup", "3", "--config", "green_cubes_n64"]
    r = subprocess.run(cmd, cwd=root, env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["n_gpus"] == 2 and line["dist_backend"] == "gloo"
    assert line["sampled_rel_err_vs_dense"] < 1e-4
    assert line["gpu_launches"] > 0


def test_peer_offsets_match_receivers():
    """Fused exchange: the offset at which a producer stores block (t, s) in
    the owner of t's receive buffer is that owner's own receive offset."""
    from paper_2411_03029_b200.sharded import exchange_layout, owns, peer_offsets
    rng = np.random.default_rng(0)
    for world in (2, 3, 4, 8):
        nmid = 8
        R = rng.integers(1, 6, (nmid, nmid))
        lays = [exchange_layout(R, q, world) for q in range(world)]
        for r in range(world):
            off = peer_offsets(R, r, world)
            for t in range(nmid):
                for s in range(nmid):
                    if owns(s, r, world):
                        assert off[t * nmid + s] == lays[t % world].recv_off[t * nmid + s] >= 0
                    else:
                        assert off[t * nmid + s] == -1


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 3])
def test_fused_exchange_equals_alltoall(world):
    """The fused exchange (phase-1 GEMV storing G_{t,s} into the owners'
    receive buffers through CUDA IPC, two alternating buffers) gives the same
    G bit for bit as the send buffer + all-to-all path, nv = 1, 2, three
    consecutive steps (both parities).  Validation mode: all ranks on device 0,
    gloo host barriers -- no kernel waits on another rank."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, OIOBF_BENCH_DIST="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(world),
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), "tools/peer_check.py"]
    r = subprocess.run(cmd, cwd=root, env=env, capture_output=True, text=True, timeout=400)
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["world"] == world and line["fused_equals_alltoall"], line


def _umid_worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2411_03029_b200.sharded import exchange_umid_skeletons
        nmid, d, wpad = 8, 3, 4
        nslots = nmid * nmid * d
        full = (np.arange(nslots * wpad, dtype=np.int32) + 7).reshape(nslots, wpad)  # the whole truth
        t_of = np.arange(nslots) // (nmid * d)
        s_of = (np.arange(nslots) // d) % nmid
        mine_built = full.copy()
        mine_built[t_of % world != rank] = 0  # this rank built only its t (umid_export zeroes the rest)
        got = exchange_umid_skeletons(mine_built.reshape(-1), rank, world, nmid, d, wpad, TorchComm()).reshape(nslots,
                                                                                                            wpad)
        need = s_of % world == rank
        ok = bool(np.array_equal(got[need], full[need]) and not got[~need].any())
        q.put(("ok", ok, 0.0))
    except Exception as e:  # pragma: no cover
        q.put(("err", repr(e), 0.0))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_umid_skeleton_alltoall(world):
    """The U-side middle skeletons reach exactly the ranks whose cores need them
    (slots (t, nu = s) with s owned), over a real gloo all-to-all."""
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_umid_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in ps:
        p.join(timeout=60)
    assert all(r[0] == "ok" and r[1] for r in res), res
