#!/usr/bin/env python
"""Multi-GPU map designs on virtual ranks (one B200): ghost-tet overlap vs the
north_star reverse add of partial f / K rows.

For P ranks of a weak-scaled Kuhn-6 cube (~`--per-rank` tets each, the T10M
recipe) every rank's local problem comes from the device partition; per rank
and variant the element map (CUDA events, L2 flushed) and, for the reverse
variant, the reverse exchange (pack on the sender, copy, scatter-add on the
receiver: the bytes NCCL would move) are timed; the halo bytes per PCG
iteration (the forward u halo) are counted.  One JSON line per (P, variant).

    python tools/dist_variants.py [--P 2,4,8] [--per-rank 1000000] [--reps 5]
"""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--P", default="1,2,4,8")
    ap.add_argument("--per-rank", type=int, default=1_000_000)
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    import numpy as np
    import torch

    from paper_1506_07577_b200 import _abi as A
    from paper_1506_07577_b200 import build, dist, ebb
    build.build()
    w = bench.WORKLOAD
    flush = torch.empty(bench.FLUSH_BYTES, dtype=torch.uint8, device="cuda")
    for P in [int(x) for x in a.P.split(",")]:
        n = int(round((P * a.per_rank / 6) ** (1 / 3)))
        E_n = w["E"] * (w["n"] / n) ** 2
        X, tets, free, u0, mu, lam = bench.make_case(n, w["order_seed"], w["u_seed"], E_n, w["nu"], wall_ramp=0.1)
        v0 = np.zeros_like(u0)
        for variant in ("overlap", "reverse"):
            ctx = ebb.Context(0)
            ranks = []
            for r in range(P):
                part = dist.partition_rank(ctx, X, tets, P, r, name=f"dv{P}{variant}{r}")
                ranks.append(dist.GpuRank(ctx, r, part, X, free, u0, v0, mu, lam, rho=w["rho"],
                                          name=f"dv{P}{variant}r{r}", map_variant=variant, nranks=P))
            T = dist.LocalTransport()
            for R in ranks:                       # warm-up (plans built here)
                R.map_forces(w["model"])
            torch.cuda.synchronize()
            ctx.timing(True)
            map_us, ex_us, peer_rev_us = [], 0.0, None
            for R in ranks:
                ctx.timing_read(A.K_TET_MAP, reset=True)
                for _ in range(a.reps):
                    flush.zero_()
                    R.map_forces(w["model"])
                ms, nl = ctx.timing_read(A.K_TET_MAP, reset=True)
                map_us.append(1e3 * ms / max(nl, 1))
            if variant == "reverse":
                for which in ("rf", "rK"):
                    for R in ranks:
                        R.set_halo(which)
                    T.exchange(ranks)             # warm-up
                ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
                tot = 0.0
                for _ in range(a.reps):
                    flush.zero_()
                    ev[0].record()
                    for which in ("rf", "rK"):
                        for R in ranks:
                            R.set_halo(which)
                        T.exchange(ranks)
                    ev[1].record()
                    ev[1].synchronize()
                    tot += ev[0].elapsed_time(ev[1])
                ex_us = 1e3 * tot / a.reps / P      # all P ranks' exchanges run one after the other here
                # the same reverse add as peer-memory REDs (PeerHalo ADD, all ranks in one launch per list)
                prev = (dist.PeerHalo(ranks, "rf"), dist.PeerHalo(ranks, "rK"))
                for hp in prev:
                    hp.push()                     # warm-up
                tot = 0.0
                for _ in range(a.reps):
                    flush.zero_()
                    ev[0].record()
                    for hp in prev:
                        hp.push()
                    ev[1].record()
                    ev[1].synchronize()
                    tot += ev[0].elapsed_time(ev[1])
                peer_rev_us = 1e3 * tot / a.reps
            ctx.timing(False)
            # one whole distributed implicit step (map, reverse add, assembly,
            # 50 PCG iterations, halos, allreduces) per PCG driver; all P ranks
            # run one after the other on this GPU, so per rank = total / P
            step_ms = {}
            for cg in ("single", "saad"):
                dist.implicit_step(ranks, T, w["model"], h=w["h"], iters=w["cg_iters"], variant=cg)   # warm-up
                ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
                tot = 0.0
                for _ in range(2):
                    flush.zero_()
                    ev[0].record()
                    dist.implicit_step(ranks, T, w["model"], h=w["h"], iters=w["cg_iters"], variant=cg)
                    ev[1].record()
                    ev[1].synchronize()
                    tot += ev[0].elapsed_time(ev[1])
                step_ms[cg] = tot / 2 / P
            # the transport-free step: the fused peer PCG (+ the peer RED
            # reverse add); the PCG of all ranks is ONE launch here
            pcg = dist.PeerPCG(ranks)
            prv = (dist.PeerHalo(ranks, "rf"), dist.PeerHalo(ranks, "rK")) if variant == "reverse" else None

            def peer_step():
                dist.implicit_step(ranks, None, w["model"], h=w["h"], iters=w["cg_iters"], variant="peer", peer=pcg,
                                   peer_rev=prv)
            peer_step()
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
            tot = 0.0
            for _ in range(2):
                flush.zero_()
                ev[0].record()
                peer_step()
                ev[1].record()
                ev[1].synchronize()
                tot += ev[0].elapsed_time(ev[1])
            peer_step_ms_total = tot / 2
            bf = 8
            halo_rows = [sum(b[1][3][1].shape[0] for b in R._lists["fwd"]["send"].values()) for R in ranks]
            line = {"P": P, "variant": variant, "global_tets": int(tets.shape[0]), "n": n,
                    "local_tets": [int(R.fem.nt) for R in ranks],
                    "mapped_tets": [int(R.n_map_tets) if variant == "reverse" else int(R.fem.nt) for R in ranks],
                    "map_us": map_us, "map_us_max": max(map_us),
                    "reverse_bytes_per_rank": [int(R.rev_bytes["rf"] + R.rev_bytes["rK"]) for R in ranks]
                    if variant == "reverse" else None,
                    "reverse_exchange_us_per_rank": ex_us if variant == "reverse" else None,
                    "reverse_add_peer_red_us_all_ranks": peer_rev_us if variant == "reverse" else None,
                    "step_ms_per_rank": step_ms,
                    "peer_step_ms_all_ranks": peer_step_ms_total, "peer_pcg_body": pcg.variant,
                    "pcg_iter_us_per_rank_incl_halo": {k: 1e3 * v / w["cg_iters"] for k, v in step_ms.items()},
                    "fwd_halo_rows_per_rank": halo_rows,
                    "fwd_halo_bytes_per_iteration_per_rank": [r_ * 4 * bf for r_ in halo_rows],
                    "note": "virtual ranks on one B200; exchange = pack + device copy + scatter(-add), the bytes "
                            "an NCCL send/recv would move"}
            print(json.dumps(line), flush=True)
            ctx.close()
            del ranks


if __name__ == "__main__":
    main()
