"""The one-process-per-GPU setup of the fused PCG (PeerPCG with a
torch.distributed group): two processes exchange their infos with
all_gather_object, export / open CUDA IPC handles of their CG buffers and
mailboxes (ebb_ipc_*), bind (ebb_cg_peer_bind with IPC-mapped peer
addresses) and launch ebb_cg_peer_step with 0 iterations (nothing waits on
the other process: kernels that wait on one another must not share one GPU,
B200_PROFILING.md).  Both processes use the one GPU of this box; each writes
a marker through its mapping of the peer's u2 buffer and the peer reads it
back from its own field -- the P2P path the kernel's ghost-row stores take."""
import os
import socket
import tempfile

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu


def _view(addr, n):
    import torch

    class _CAI:
        __cuda_array_interface__ = {"shape": (n,), "typestr": "<f8", "data": (addr, False), "version": 3,
                                    "strides": None}
    return torch.as_tensor(_CAI(), device="cuda:0")


def _worker(rank, world, port, outdir):
    import sys
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import torch
    import torch.distributed as tdist

    from helpers import Case
    from paper_1506_07577_b200 import dist, ebb
    torch.cuda.set_device(0)
    tdist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    ctx = ebb.Context(0)
    case = Case(n=5, model="nh")
    part = dist.partition_rank(ctx, case.X, case.tets, world, rank, name=f"ipc{rank}")
    R = dist.GpuRank(ctx, rank, part, case.X, case.free, case.u, case.vel, case.mu, case.lam, name=f"ipcr{rank}",
                     nranks=world)
    peer = dist.PeerPCG([R], comm=tdist.group.WORLD)
    opened = len(peer._opened)
    for q in range(world):
        if q != rank:
            _view(peer.peer_addr[(rank, q, "u2")], 4).copy_(
                torch.tensor([100.0 * rank + q, 1.0, 2.0, 3.0], device="cuda:0"))
    torch.cuda.synchronize()
    tdist.barrier()
    got = R.halo_fields["u2"].read()[0].tolist()
    peer.step(0)                                     # the kernel with IPC-mapped peer addresses, no waits
    torch.cuda.synchronize()
    errs = ctx.error_counts()
    tdist.barrier()
    peer.close()
    np.savez(os.path.join(outdir, f"r{rank}.npz"), got=np.array(got), opened=opened,
             timeouts=errs["peer_timeouts"])
    tdist.barrier()
    ctx.close()
    tdist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_peer_pcg_ipc_setup_two_processes():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import torch.multiprocessing as mp
    world = 2
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_worker, args=(world, _free_port(), d), nprocs=world, join=True)
        for r in range(world):
            z = np.load(os.path.join(d, f"r{r}.npz"))
            q = 1 - r
            assert z["got"].tolist() == [100.0 * q + r, 1.0, 2.0, 3.0]
            assert int(z["opened"]) == 5                      # u, u2, x, z, mailbox of the one peer
            assert int(z["timeouts"]) == 0
