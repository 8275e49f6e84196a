#!/usr/bin/env python
"""Exercise every hot kernel once on small meshes, for compute-sanitizer
(memcheck / racecheck / synccheck / initcheck):

    compute-sanitizer --tool racecheck python tools/sanitize_run.py [--sizes 4,12]

Kuhn-6 n=4 (C1, 384 tets) and n=12 (10,368 tets): the element map with every
scatter strategy (fp64 and fp32, StVK and NH), assembly, the edge-relation
matvec, every persistent PCG variant (Saad, single-reduction, symmetric) and
the phase kernels of the multi-GPU driver, the explicit update, the matrix-free
EBE matvec, the Fig. 2 spring-mass step (fused and paper form) and the 2-D grid
stencil / PointLocate / particle interpolation, and the multi-GPU setup and
exchange kernels on 2 virtual ranks.  Prints one line per stage;
the sanitizer's own report is the evidence (profiles/r02_sanitizer_*.txt).
"""
from __future__ import annotations

import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", default="4,12")
    ap.add_argument("--quick", action="store_true", help="fp64 NH only (racecheck is slow)")
    ap.add_argument("--peer-only", action="store_true", help="only the multi-GPU setup and the fused peer PCG")
    a = ap.parse_args()
    import numpy as np
    import torch

    from paper_1506_07577_b200 import _abi as A
    from paper_1506_07577_b200 import ebb
    from paper_1506_07577_b200.grid import Grid2
    from paper_1506_07577_b200.springmass import SpringMass
    from paper_1506_07577_b200.tetfem import TetFEM
    from synth import mesh as M
    from synth import state as S

    scat = {"atomic": A.SCATTER_ATOMIC, "segmented": A.SCATTER_SEGMENTED, "color": A.SCATTER_COLOR,
            "chunk": A.SCATTER_CHUNK, "chunk_red": A.SCATTER_CHUNK_RED}
    ctx = ebb.Context(0)
    for n in ([] if a.peer_only else [int(x) for x in a.sizes.split(",")]):
        X, tets = M.kuhn6(n)
        X, tets = M.permute_vertices(X, tets, 2)
        free = S.fixed_mask(X, n)
        u = S.stretch_noise_u(X, n, 1, free=free)
        mu, lam = S.materials(tets.shape[0], 2e5, 0.3)
        for dt in (("f64",) if a.quick else ("f64", "f32")):
            fem = TetFEM(ctx, X, tets, dtype=dt, mu=mu, lam=lam, free=free, u=u, name=f"s{n}{dt}")
            for model in (("nh",) if a.quick else ("nh", "stvk")):
                for name, sid in scat.items():
                    fem.map_forces(model, scatter=sid)
                    torch.cuda.synchronize()
                    print(f"n={n} {dt} {model} map {name} ok", flush=True)
            fem.map_forces("nh")
            fem.assemble(1e-2)
            P = fem.verts.field("p_s", dt, (3, 1), init=np.ones((fem.nv, 3)))
            Q = fem.verts.field("q_s", dt, (3, 1))
            fem.matvec(fem.K, P, Q)
            torch.cuda.synchronize()
            print(f"n={n} {dt} assemble + matvec ok", flush=True)
            for var in (A.CG_SAAD, A.CG_SINGLE_REDUCTION, A.CG_SYMMETRIC):
                fem.map_forces("nh")
                fem.assemble(1e-2)
                fem.cg_init(variant=var)
                fem.cg_step(5)
                torch.cuda.synchronize()
                print(f"n={n} {dt} pcg variant {var} ok", flush=True)
            fem.cg_init(variant=A.CG_AUTO, tol=1e-6)
            fem.cg_step(20)
            fem.cg_iterations()
            fem.cg.tol = 0.0
            # phase kernels of the multi-GPU driver (Saad phases and the single-reduction phase)
            fem.cg_init(variant=A.CG_SAAD)
            for ph in (A.CG_DIR, A.CG_MATVEC, A.CG_UPDATE):
                ctx.check(ctx.L.ebb_cg_phase(ctx.h, __import__("ctypes").byref(fem.cg), ph, None))
            fem.cg_init(variant=A.CG_SINGLE_REDUCTION)
            for _ in range(3):
                ctx.check(ctx.L.ebb_cg_phase(ctx.h, __import__("ctypes").byref(fem.cg), A.CG_SR_PHASE, None))
            torch.cuda.synchronize()
            print(f"n={n} {dt} cg phases ok", flush=True)
            fem.explicit_step("stvk")
            st = fem.ebe_state("nh")
            fem.ebe_matvec(st, P, Q, "nh")
            torch.cuda.synchronize()
            print(f"n={n} {dt} explicit + ebe ok", flush=True)
            sm = SpringMass(fem, K=-1.0, name=f"sp{n}{dt}")
            sm.init_len()
            sm.step()
            sm.step_paper()
            sm.kinetic_energy()
            torch.cuda.synchronize()
            print(f"n={n} {dt} spring ok", flush=True)
            del fem
    # the multi-GPU setup and exchange kernels on 2 virtual ranks: device
    # partition (overlap and own modes), reverse-add lists, SOA row gather,
    # scatter-add, the distributed map step and one distributed implicit step
    from paper_1506_07577_b200 import dist
    X, tets = M.kuhn6(6)
    X, tets = M.permute_vertices(X, tets, 2)
    free = S.fixed_mask(X, 6)
    u = S.stretch_noise_u(X, 6, 1, free=free)
    mu, lam = S.materials(tets.shape[0], 2e5, 0.3)
    for variant in ("overlap", "reverse"):
        ranks = []
        for r in range(2):
            dist.partition_rank(ctx, X, tets, 2, r, name=f"sp_own{variant}{r}", mode="own")
            part = dist.partition_rank(ctx, X, tets, 2, r, name=f"sp{variant}{r}")
            ranks.append(dist.GpuRank(ctx, r, part, X, free, u, np.zeros_like(u), mu, lam, name=f"sr{variant}{r}",
                                      map_variant=variant, nranks=2))
        if not a.peer_only:
            dist.map_step(ranks, dist.LocalTransport(), "nh")
            dist.implicit_step(ranks, dist.LocalTransport(), "nh", iters=5, variant="single")
            torch.cuda.synchronize()
            print(f"dist {variant} ok", flush=True)
        # the fused multi-GPU PCG over peer memory, both bodies, the 2 ranks
        # in one cooperative launch (the P2P stores and mailbox exchanges)
        for body in ("single", "saad"):
            peer = dist.PeerPCG(ranks, variant=body)
            for _ in range(2):
                dist.implicit_step(ranks, dist.LocalTransport(), "nh", iters=5, variant="peer", peer=peer)
            torch.cuda.synchronize()
            assert ctx.error_counts()["peer_timeouts"] == 0
            print(f"dist {variant} peer pcg {body} ok", flush=True)
        del ranks
    if a.peer_only:
        ctx.close()
        print("SANITIZE RUN DONE", flush=True)
        return
    import gc
    gc.collect()
    torch.cuda.empty_cache()   # the halo staging tensors come from torch's caching allocator
    g = Grid2(ctx, 37, 29, name="sgrid")
    rng = np.random.default_rng(3)
    fin = g.cells.field("fin", "f64", (2, 1), init=rng.uniform(-1, 1, size=(37 * 29, 2)))
    fout = g.cells.field("fout", "f64", (2, 1))
    g.stencil(fin, fout, [(0, 0), (1, 0), (-1, 0), (0, 1), (0, -1)], [-4, 1, 1, 1, 1])
    Pp, pos, key = g.particles("sparts", rng.uniform(0, 37, size=(2000, 3)))
    vel = Pp.field("pvel", "f64", (2, 1))
    g.particle_vel(key, fin, pos, vel)
    torch.cuda.synchronize()
    print("grid ok", flush=True)
    ctx.close()
    print("SANITIZE RUN DONE", flush=True)


if __name__ == "__main__":
    main()
