"""Fused exchange (GEMV peer stores) vs the all-to-all path, under torchrun.
Validation mode on one GPU: OIOBF_BENCH_DIST=gloo puts every rank on device 0
(CUDA IPC between processes on one device; the ranks only meet at host
barriers, no kernel waits on another rank).  Prints one JSON line on rank 0."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, torch.distributed as dist
import paper_2411_03029_b200 as tb
from paper_2411_03029_b200 import _lib
from paper_2411_03029_b200.configs import BY_NAME, green_cubes, radon2d
from paper_2411_03029_b200.sharded import GpuShardBackend, PeerExchange, TorchComm, construct

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
gloo = os.environ.get("OIOBF_BENCH_DIST", "nccl") == "gloo"
local = 0 if gloo else int(os.environ.get("LOCAL_RANK", "0"))
torch.cuda.set_device(local)
if gloo:
    dist.init_process_group("gloo")
else:
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
_lib.check(_lib.load().oiobf_set_device(local))
dev = torch.device("cuda", local)
comm = TorchComm(device=dev)
res = {}
for name, spec, L, tol in (("cubes16", green_cubes(16), 2, 1e-4), ("cubes64", BY_NAME["green_cubes_n64"].spec, 2, 1e-6),
                           ("radon64", radon2d(64), 2, 1e-6)):
    be = GpuShardBackend(spec, L, tol, tb.ProxyStrategy(), 3, rank, world)
    sb = construct(be, rank, world, comm)
    for nv in (1, 2):
        rng = np.random.default_rng(5 + nv)
        N = spec.n ** spec.d
        F = torch.from_numpy(rng.standard_normal(2 * N * nv)).to(dev)
        lay = sb.layout
        send = torch.zeros(2 * max(1, int(lay.send_counts.sum())) * nv, dtype=torch.float64, device=dev)
        recv = torch.zeros(2 * max(1, int(lay.recv_counts.sum())) * nv, dtype=torch.float64, device=dev)
        G1 = torch.zeros_like(F)
        s = torch.cuda.current_stream().cuda_stream
        be.phase(1, F.data_ptr(), send.data_ptr(), nv, s)
        comm.alltoall(send, recv, lay.send_counts * nv, lay.recv_counts * nv)
        be.phase(2, recv.data_ptr(), G1.data_ptr(), nv, s)
        px = PeerExchange(sb, comm, nv_max=2)
        G2 = torch.zeros_like(F)
        for _ in range(3):  # both parities, then the first again
            G2.zero_()
            px.step(F.data_ptr(), G2.data_ptr(), nv, s)
            torch.cuda.synchronize()
            ok = bool(torch.equal(G1, G2))
            res.setdefault(f"{name}_nv{nv}", []).append(ok)
        comm.barrier()
        px.close()
oks = torch.tensor([int(all(all(v) for v in res.values()))], dtype=torch.int64)
dist.all_reduce(oks, op=dist.ReduceOp.MIN)
if rank == 0:
    print(json.dumps({"world": world, "fused_equals_alltoall": bool(oks.item()), "cases": res}), flush=True)
dist.destroy_process_group()
