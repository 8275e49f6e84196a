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
        self.scal = torch.zeros(12, dtype=torch.float64)
        self.halo = "z"
        local = {g: i for i, g in enumerate(verts)}
        self.send = {o: np.array([local[g] for g in lst], dtype=np.int64)
                     for o, lst in enumerate(send[rank]) if len(lst)}
        self.recv = {o: np.array([local[g] for g in lst], dtype=np.int64)
                     for o, lst in enumerate(recv[rank]) if len(lst)}

    def map_forces(self, model):
        import oracle
        m = self.mesh
        self.f, self.K, en, inv = oracle.element_map(model, m.X, self.u, m.tets, m.Dminv, m.W, self.mu, self.lam,
                                                     e=m.e, ne=m.ne)

    def assemble(self, h, alpha, beta, g):
        import oracle
        m = self.mesh
        self.A, self.b = oracle.implicit_assemble(m.row_ptr, m.head, self.K, m.mass, self.f, self.vel, h, alpha,
                                                  beta, g)

    def cg_init(self, single=False):
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
        self.scal[0], self.scal[2], self.scal[3], self.scal[7] = rz, rz, 1.0, rz
        z0 = np.zeros_like(self.x)
        self.s, self.y, self.w, self.ub = z0.copy(), z0.copy(), z0.copy(), [z0.copy(), z0.copy()]

    def _sr_phase(self):
        """One single-reduction (Chronopoulos-Gear) phase in the GPU's phase
        mode (solver.cu k_cg1_persistent, dist=1): finish the previous
        phase's recurrences from the allreduced sums, then one matvec of the
        operand and the owner recurrences, leaving the local (w.z, r.z)."""
        import oracle
        s = self.scal
        gam, alpha, beta = float(s[0]), float(s[5]), float(s[1])
        first, par = s[3] != 0, int(s[4])
        if s[6] == 1:
            dsum = float(s[10])
            alpha, beta, first = (gam / dsum if dsum != 0 else 0.0), 0.0, False
        elif s[6] == 2:
            dsum, gnew = float(s[10]), float(s[11])
            bn = gnew / gam if gam != 0 else 0.0
            den = dsum - (bn * gnew / alpha if alpha != 0 else 0.0)
            alpha, beta, gam, par = (gnew / den if den != 0 else 0.0), bn, gnew, par ^ 1
        op = self.z if first else self.ub[par]
        un = par if first else 1 - par
        a = oracle.edge_matvec(self.mesh.row_ptr, self.mesh.head, self.A, op) * self.mask[:, None]
        if first:
            self.w = a
            self.ub[un] = a * self.dinv
            pd, pg = float(np.sum(a * self.z)), 0.0
        else:
            zi = self.r * self.dinv
            self.s = self.w + beta * self.s
            self.y = a + beta * self.y
            self.p = zi + beta * self.p
            self.x += alpha * self.p
            self.r -= alpha * self.s
            self.w -= alpha * self.y
            self.ub[un] = self.w * self.dinv
            self.z = self.r * self.dinv
            pg, pd = float(np.sum(self.r * self.z)), float(np.sum(self.w * self.z))
        s[10], s[11], s[6] = pd, pg, (1.0 if first else 2.0)
        s[0], s[2], s[5], s[1], s[3], s[4] = gam, gam, alpha, beta, (1.0 if first else 0.0), par

    def set_halo(self, which):
        self.halo = which

    def _arr(self):
        return {"z": self.z, "x": self.x, "u": self.ub[0], "u2": self.ub[1]}[self.halo]

    def cg_phase(self, k):
        import oracle
        s = self.scal
        if k == 3:
            return self._sr_phase()
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

    def send_peers(self):
        return sorted(self.send)

    def recv_peers(self):
        return sorted(self.recv)

    def pack(self, peer):
        import torch
        return torch.from_numpy(np.ascontiguousarray(self._arr()[self.send[peer]]))

    def recv_buffer(self, peer):
        import torch
        return torch.empty((len(self.recv[peer]), 3), dtype=torch.float64)

    def unpack(self, peer, data):
        self._arr()[self.recv[peer]] = data.numpy()


def _case():
    import sys
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from helpers import Case, oracle_renumbered
    import oracle
    case = Case(n=4, model="nh", vel_amp=0.05)
    m, new_of_old, tet_src, order = oracle_renumbered(case)
    return case, m, tet_src, order, oracle


STEPS = 3


def _plan(part, tets, P):
    """(problems, send, recv) of every rank from the oracle's overlapping O4
    (the GPU ranks get theirs from ebb_partition_local): problems[r] = (local
    tets, local vertices ascending, local tet keys, owned mask)."""
    ov = part["owner_v"]
    problems = []
    for r in range(P):
        lt = part["ltets"][r]
        verts = np.sort(part["local"][r])
        problems.append((lt, verts, np.searchsorted(verts, tets[lt]), ov[verts] == r))
    send = [[part["send"][o][r] for r in range(P)] for o in range(P)]
    recv = [[part["send"][o][r] for o in range(P)] for r in range(P)]
    return problems, send, recv


def _worker(rank, world, port, outdir, variant):
    import sys
    sys.path.insert(0, ROOT)
    import torch.distributed as tdist

    from paper_1506_07577_b200 import dist
    tdist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    case, m, tet_src, order, oracle = _case()
    part = oracle.partition(m.nv, m.tets, world, mode="overlap")
    plan = _plan(part, m.tets, world)
    R = OracleRank(rank, m.X, m.tets, part["owner_v"], plan, case.free[order], case.u[order], case.vel[order],
                   case.mu[tet_src], case.lam[tet_src])
    for _ in range(STEPS):
        dist.implicit_step([R], dist.TorchTransport(), "nh", h=1e-2, iters=50, variant=variant)
    np.savez(os.path.join(outdir, f"r{rank}.npz"), ids=R.verts, owned=R.owned, u=R.u, v=R.vel)
    tdist.barrier()
    tdist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("variant,world", [("saad", 2), ("saad", 3), ("single", 2), ("single", 3)])
def test_gloo_distributed_implicit_steps(world, variant):
    """STEPS consecutive distributed implicit steps on `world` gloo ranks
    (both PCG drivers) reproduce STEPS single-domain oracle steps on every
    local row -- owned AND ghost: a ghost that went stale after step 1 would
    corrupt the next map on ghost tets."""
    import torch.multiprocessing as mp
    case, m, tet_src, order, oracle = _case()
    u, v = case.u[order], case.vel[order]
    for _ in range(STEPS):
        ref = oracle.implicit_step(m, "nh", u, v, case.mu[tet_src], case.lam[tet_src], case.free[order], 1e-2,
                                   iters=50)
        u, v = ref["u"], ref["v"]
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_worker, args=(world, _free_port(), d, variant), nprocs=world, join=True)
        seen = np.zeros(m.nv, dtype=np.int64)
        for r in range(world):
            z = np.load(os.path.join(d, f"r{r}.npz"))
            seen[z["ids"][z["owned"]]] += 1
            for got, want in ((z["u"], u[z["ids"]]), (z["v"], v[z["ids"]])):
                assert np.linalg.norm(got - want) <= 1e-10 * np.linalg.norm(want)
    assert np.all(seen == 1)                      # every vertex owned exactly once
