"""Host bookkeeping of the fused multi-GPU PCG (dist.peer_tables, the input
of ebb_cg_peer_bind) on CPU: from the ranks' exported infos -- recv rows per
peer, local sizes, buffer entries -- every rank's remote rows must name, on
the peer, the same global vertices its send rows name locally (oracle O4
lists, overlapping mode), in the same order.  The one-process-per-GPU path
moves the infos with torch.distributed.all_gather_object: checked on gloo,
world size 2 and 3."""
import os
import socket
import tempfile

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _infos(P, n=4):
    import sys
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from helpers import Case, oracle_renumbered

    import oracle
    case = Case(n=n, model="nh")
    m, _, _, _ = oracle_renumbered(case)
    part = oracle.partition(m.nv, m.tets, P, mode="overlap")
    infos, local = {}, {}
    for r in range(P):
        lv = np.asarray(part["local"][r])
        local[r] = lv
        row = {int(g): i for i, g in enumerate(lv)}
        send = {q: np.array([row[int(g)] for g in part["send"][r][q]], np.int64)
                for q in range(P) if len(part["send"][r][q])}
        recv = {q: np.array([row[int(g)] for g in part["send"][q][r]], np.int64)
                for q in range(P) if len(part["send"][q][r])}
        infos[r] = dict(rank=r, nv=int(lv.size), send={q: int(s.size) for q, s in send.items()}, recv=recv,
                        buf={name: 1000 * r + k for k, name in enumerate(("u", "u2", "x", "z", "mbox"))},
                        _send_rows=send)
    return infos, local


@pytest.mark.parametrize("P", [2, 3, 4])
def test_peer_tables_name_the_same_vertices(P):
    from paper_1506_07577_b200 import dist
    infos, local = _infos(P)
    tables = dist.peer_tables(infos, list(range(P)), P)
    for r in range(P):
        t = tables[r]
        assert t["peers"] == sorted(infos[r]["send"])
        for q, rem, nvq in zip(t["peers"], t["remote"], t["peer_nv"]):
            send_rows = infos[r]["_send_rows"][q]
            assert np.array_equal(local[q][rem], local[r][send_rows])   # same global vertices, same order
            assert nvq == local[q].size and rem.max() < nvq
        for name in dist.PEER_BUFFERS:
            assert t["bufs"][name][r] is None
            assert [t["bufs"][name][q] for q in range(P) if q != r] == [infos[q]["buf"][name] for q in range(P)
                                                                        if q != r]


def test_peer_tables_refuse_mismatched_lists():
    from paper_1506_07577_b200 import dist
    infos, _ = _infos(2)
    q = sorted(infos[0]["send"])[0]
    infos[q]["recv"][0] = infos[q]["recv"][0][:-1]          # the peer expects one row fewer
    with pytest.raises(ValueError, match="expects"):
        dist.peer_tables(infos, [0], 2)


def _worker(rank, world, port, outdir):
    import sys
    sys.path.insert(0, ROOT)
    import torch.distributed as tdist

    from paper_1506_07577_b200 import dist
    tdist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    infos, _ = _infos(world)
    mine = {k: v for k, v in infos[rank].items() if not k.startswith("_")}
    gathered = [None] * world
    tdist.all_gather_object(gathered, mine)                 # what PeerPCG(comm=...) does
    got = {d["rank"]: d for d in gathered}
    t = dist.peer_tables(got, [rank], world)[rank]
    np.savez(os.path.join(outdir, f"r{rank}.npz"), peers=np.array(t["peers"]),
             remote=np.concatenate(t["remote"]) if t["remote"] else np.zeros(0, np.int64),
             peer_nv=np.array(t["peer_nv"]))
    tdist.barrier()
    tdist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("world", [2, 3])
def test_peer_tables_over_gloo_all_gather(world):
    import torch.multiprocessing as mp

    from paper_1506_07577_b200 import dist
    infos, _ = _infos(world)
    ref = dist.peer_tables(infos, list(range(world)), world)
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_worker, args=(world, _free_port(), d), nprocs=world, join=True)
        for r in range(world):
            z = np.load(os.path.join(d, f"r{r}.npz"))
            assert z["peers"].tolist() == ref[r]["peers"]
            assert np.array_equal(z["remote"], np.concatenate(ref[r]["remote"]))
            assert z["peer_nv"].tolist() == ref[r]["peer_nv"]
