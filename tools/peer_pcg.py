#!/usr/bin/env python
"""The fused multi-GPU PCG (ebb_cg_peer_step) on ranks emulated on one B200,
against the single-domain persistent PCG on the same global mesh and the
per-phase "single" driver (one launch + one allreduce + one halo per
iteration, host-driven).

For each P the global mesh is the same (strong scaling, the T10M recipe by
default): P ranks from the device partition share the GPU's SMs in ONE
cooperative launch of the peer kernel, so its time against the single-domain
kernel is the cost of the decomposition itself (ghost rows gathered, per-rank
grid barriers, the mailbox exchange, P2P stores of u, x) -- on P real GPUs
each rank would have the whole device.  CUDA events, L2 flushed, 50
iterations after ebb_cg_init.  One JSON line per P.

    python tools/peer_pcg.py [--n 119] [--P 1,2,4,8] [--reps 5] [--phase]
"""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def _time(fn, reps, flush):
    import torch
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    fn()                                          # warm-up
    tot = []
    for _ in range(reps):
        flush.zero_()
        torch.cuda.synchronize()
        ev[0].record()
        fn()
        ev[1].record()
        ev[1].synchronize()
        tot.append(ev[0].elapsed_time(ev[1]))
    return sorted(tot)[len(tot) // 2]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=119)
    ap.add_argument("--P", default="1,2,4,8")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--iters", type=int, default=50)
    ap.add_argument("--phase", action="store_true", help="also time the per-phase single-reduction driver")
    a = ap.parse_args()
    import numpy as np
    import torch

    from paper_1506_07577_b200 import _abi as A
    from paper_1506_07577_b200 import build, dist, ebb
    from paper_1506_07577_b200.tetfem import TetFEM
    build.build()
    w = dict(bench.WORKLOAD)
    n = a.n
    E_n = w["E"] * (w["n"] / n) ** 2
    X, tets, free, u0, mu, lam = bench.make_case(n, w["order_seed"], w["u_seed"], E_n, w["nu"], wall_ramp=0.1)
    v0 = np.zeros_like(u0)
    flush = torch.empty(bench.FLUSH_BYTES, dtype=torch.uint8, device="cuda")
    g = (0.0, -9.81, 0.0)
    # single-domain reference: the same system, one persistent kernel (the
    # solve alone: ebb_cg_init timed separately and subtracted, as for the ranks)
    ctx = ebb.Context(0)
    fem = TetFEM(ctx, X, tets, dtype="f64", mu=mu, lam=lam, rho=w["rho"], free=free, u=u0, vel=v0, name="sd")
    fem.map_forces(w["model"])
    fem.assemble(w["h"], 0.0, 0.0, g)
    single = {}
    for var, code in (("saad", A.CG_SAAD), ("single_reduction", A.CG_SINGLE_REDUCTION)):
        def run(code=code):
            fem.cg_init(variant=code)
            fem.cg_step(a.iters)
        single[var] = _time(run, a.reps, flush) - _time(lambda code=code: fem.cg_init(variant=code), a.reps, flush)
    nv_g = fem.nv
    ctx.close()
    del fem
    for P in [int(x) for x in a.P.split(",")]:
        ctx = ebb.Context(0)
        ranks = []
        for r in range(P):
            part = dist.partition_rank(ctx, X, tets, P, r, name=f"pp{P}p{r}")
            ranks.append(dist.GpuRank(ctx, r, part, X, free, u0, v0, mu, lam, rho=w["rho"], name=f"pp{P}r{r}",
                                      nranks=P))
        for R in ranks:
            R.map_assemble(w["model"], w["h"], 0.0, 0.0, g)
        peer_ms = {}
        for var in ("single", "saad"):
            peer = dist.PeerPCG(ranks, variant=var)
            sr = var == "single"

            def run_peer():
                for R in ranks:
                    R.cg_init(single=sr)
                peer.step(a.iters)
            t_init = _time(lambda: [R.cg_init(single=sr) for R in ranks], a.reps, flush)
            peer_ms[var] = _time(run_peer, a.reps, flush) - t_init
            peer.close()
        # the position halo of the displacements: one peer push kernel for all
        # ranks vs the transport's pack / copy / unpack per peer
        halo = dist.PeerHalo(ranks, "disp")
        T = dist.LocalTransport()

        def run_transport():
            for R in ranks:
                R.set_halo("disp")
            T.exchange(ranks)
        halo_us = {"peer_push": 1e3 * _time(halo.push, a.reps, flush),
                   "transport": 1e3 * _time(run_transport, a.reps, flush)}
        halo.close()
        line = {"P": P, "n": n, "global_tets": int(tets.shape[0]), "global_verts": int(nv_g),
                "position_halo_us_all_ranks": halo_us,
                "owned_verts": [int(R.n_owned) for R in ranks], "local_verts": [int(R.fem.nv) for R in ranks],
                "send_rows": [int(sum(len(r_) for r_ in R.part_send.values())) for R in ranks],
                "iters": a.iters, "peer_ms": peer_ms,
                "peer_us_per_iter": {k: 1e3 * v / a.iters for k, v in peer_ms.items()},
                "single_domain_ms": single, "errors": ctx.error_counts()}
        if P == 1:
            # the single-GPU persistent kernel on this rank's own (partition-ordered) mesh
            F = ranks[0].fem
            line["rank_single_reduction_ms"] = (_time(lambda: (F.cg_init(variant=A.CG_SINGLE_REDUCTION),
                                                               F.cg_step(a.iters)), a.reps, flush)
                                                - _time(lambda: F.cg_init(variant=A.CG_SINGLE_REDUCTION), a.reps,
                                                        flush))
        line["peer_over_single_domain"] = {"single": peer_ms["single"] / single["single_reduction"],
                                           "saad": peer_ms["saad"] / single["saad"]}
        if a.phase:
            T = dist.LocalTransport()

            def run_phase():
                for R in ranks:
                    R.cg_init(single=True)
                T.allreduce(ranks, (dist.SLOT_RHO, dist.SLOT_RZ + 1))
                T.allreduce(ranks, (dist.SLOT_RZ0, dist.SLOT_RZ0 + 1))
                for R in ranks:
                    R.set_halo("z")
                T.exchange(ranks)
                for k in range(a.iters + 1):
                    for R in ranks:
                        R.cg_phase(dist.CG_SR_PHASE)
                    T.allreduce(ranks, (dist.SLOT_DSUM, dist.SLOT_GSUM + 1))
                    if k < a.iters:
                        for R in ranks:
                            R.set_halo("u" if k % 2 == 0 else "u2")
                        T.exchange(ranks)
                for R in ranks:
                    R.set_halo("x")
                T.exchange(ranks)
            t_init = _time(lambda: [R.cg_init(single=True) for R in ranks], a.reps, flush)
            line["phase_driver_ms"] = _time(run_phase, max(2, a.reps // 2), flush) - t_init
        line["note"] = ("ranks emulated on one B200: ONE cooperative launch of the peer kernel runs all P ranks, "
                        "each on 1/P of the SMs; single_domain = the same global system in one rank")
        print(json.dumps(line), flush=True)
        ctx.close()
        del ranks


if __name__ == "__main__":
    main()
