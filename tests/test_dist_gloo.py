"""Multi-rank host logic on CPU (gloo, world size 2 and 3): partition plans,
ghost consistency, halo exchange and scalar allreduces of the distributed
implicit step (paper_1506_07577_b200.dist) reproduce the single-domain oracle.

The local compute of each rank is the oracle (test code below mirrors the
semantics of the GPU phases: MATVEC with the fused direction update, UPDATE,
scalar slots rho / p.q / r.z); the driver, the plans and the torch.distributed
transport are the product's."""
import os
import socket
import tempfile

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


class OracleRank:
    def __init__(self, rank, X, tets, owner_v, plan, free, u, vel, mu, lam, rho=1e3):
        import torch

        import oracle
        problems, send, recv = plan
        lt, verts, ltets, owned = problems[rank]
        self.rank, self.verts, self.owned = rank, verts, owned
        self.mesh = oracle.Mesh(X[verts], ltets, rho=rho)
        self.mask = (free[verts] & owned).astype(np.float64)
        self.u, self.vel = u[verts].copy(), vel[verts].copy()
        self.mu, self.lam = mu[lt], lam[lt]
        self.scal = torch.zeros(8, dtype=torch.float64)
        local = {g: i for i, g in enumerate(verts)}
        self.send = {o: np.array([local[g] for g in lst], dtype=np.int64)
                     for o, lst in enumerate(send[rank]) if len(lst)}
        self.recv = {o: np.array([local[g] for g in lst], dtype=np.int64)
                     for o, lst in enumerate(recv[rank]) if len(lst)}

    def map_assemble(self, model, h, alpha, beta, g):
        import oracle
        m = self.mesh
        f, K, en, inv = oracle.element_map(model, m.X, self.u, m.tets, m.Dminv, m.W, self.mu, self.lam,
                                           e=m.e, ne=m.ne)
        self.A, self.b = oracle.implicit_assemble(m.row_ptr, m.head, K, m.mass, f, self.vel, h, alpha, beta, g)

    def cg_init(self):
        m = self.mesh
        d = np.zeros((m.nv, 3))
        for v in range(m.nv):
            for e in range(m.row_ptr[v], m.row_ptr[v + 1]):
                if m.head[e] == v:
                    d[v] = np.diag(self.A[e])
        self.dinv = np.where(self.mask[:, None] > 0, 1.0 / d, 0.0)
        self.x = np.zeros((m.nv, 3))
        self.r = self.b * self.mask[:, None]
        self.z = self.r * self.dinv
        self.p = self.z.copy()
        rz = float(np.sum(self.r * self.z))
        self.scal[:] = 0.0
        self.scal[0], self.scal[2], self.scal[3] = rz, rz, 1.0

    def cg_phase(self, k):
        import oracle
        s = self.scal
        if k == 1:
            rho, rz = float(s[0]), float(s[2])
            beta = 0.0 if (s[3] != 0 or rho == 0) else rz / rho
            self.p = self.z + beta * self.p
            self.q = oracle.edge_matvec(self.mesh.row_ptr, self.mesh.head, self.A, self.p) * self.mask[:, None]
            s[1] = float(np.sum(self.p * self.q))
            s[0], s[3] = s[2], 0.0
        elif k == 2:
            pq = float(s[1])
            alpha = float(s[0]) / pq if pq != 0 else 0.0
            self.x += alpha * self.p
            self.r -= alpha * self.q
            self.z = self.r * self.dinv
            s[2] = float(np.sum(self.r * self.z))

    def finish(self, h):
        self.vel += self.x
        self.u += h * self.vel

    def scal_tensor(self):
        return self.scal

    def peers(self):
        return sorted(set(self.send) | set(self.recv))

    def pack(self, peer):
        import torch
        return torch.from_numpy(np.ascontiguousarray(self.z[self.send[peer]]))

    def recv_buffer(self, peer):
        import torch
        return torch.empty((len(self.recv[peer]), 3), dtype=torch.float64)

    def unpack(self, peer, data):
        self.z[self.recv[peer]] = data.numpy()


def _case():
    import sys
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from helpers import Case, oracle_renumbered
    import oracle
    case = Case(n=4, model="nh", vel_amp=0.05)
    m, new_of_old, tet_src, order = oracle_renumbered(case)
    return case, m, tet_src, order, oracle


def _worker(rank, world, port, outdir):
    import sys
    sys.path.insert(0, ROOT)
    import torch.distributed as tdist

    from paper_1506_07577_b200 import dist
    tdist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    case, m, tet_src, order, oracle = _case()
    part = oracle.partition(m.nv, m.tets, world)
    plan = dist.halo_plan(m.tets, part["owner_v"], world)
    R = OracleRank(rank, m.X, m.tets, part["owner_v"], plan, case.free[order], case.u[order], case.vel[order],
                   case.mu[tet_src], case.lam[tet_src])
    dist.implicit_step([R], dist.TorchTransport(), "nh", h=1e-2, iters=50)
    np.savez(os.path.join(outdir, f"r{rank}.npz"), ids=R.verts[R.owned], dv=R.x[R.owned], u=R.u[R.owned])
    tdist.barrier()
    tdist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_distributed_implicit_step(world):
    import torch.multiprocessing as mp
    case, m, tet_src, order, oracle = _case()
    ref = oracle.implicit_step(m, "nh", case.u[order], case.vel[order], case.mu[tet_src], case.lam[tet_src],
                               case.free[order], 1e-2, iters=50)
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_worker, args=(world, _free_port(), d), nprocs=world, join=True)
        dv = np.full((m.nv, 3), np.nan)
        u = np.full((m.nv, 3), np.nan)
        for r in range(world):
            z = np.load(os.path.join(d, f"r{r}.npz"))
            assert np.all(np.isnan(dv[z["ids"]]))          # each vertex owned once
            dv[z["ids"]] = z["dv"]
            u[z["ids"]] = z["u"]
    assert not np.isnan(dv).any()
    assert np.linalg.norm(dv - ref["dv"]) <= 1e-10 * np.linalg.norm(ref["dv"])
    assert np.linalg.norm(u - ref["u"]) <= 1e-10 * np.linalg.norm(ref["u"])
