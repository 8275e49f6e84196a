#!/usr/bin/env python
"""Run the C2 element map a few times with one strategy (for ncu captures).

    python tools/map_once.py --dtype f64 --model nh --scatter gather --reps 3
"""
from __future__ import annotations

import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--dtype", default="f64")
    ap.add_argument("--model", default="nh")
    ap.add_argument("--scatter", default="segmented")
    ap.add_argument("--n", type=int, default=55)
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    import torch

    from paper_1506_07577_b200 import _abi as A
    from paper_1506_07577_b200 import build, ebb
    from paper_1506_07577_b200.tetfem import TetFEM
    from synth import mesh as M
    from synth import state as S
    build.build()
    X, tets = M.kuhn6(a.n)
    free = S.fixed_mask(X, a.n)
    mu, lam = S.materials(tets.shape[0], 1e6, 0.3, spread=0.1)
    ctx = ebb.Context(0)
    fem = TetFEM(ctx, X, tets, dtype=a.dtype, mu=mu, lam=lam, free=free, u=S.twist_u(X, a.n, 6, free=free))
    sid = {"atomic": A.SCATTER_ATOMIC, "segmented": A.SCATTER_SEGMENTED, "chunk": A.SCATTER_CHUNK,
           "color": A.SCATTER_COLOR}[a.scatter]
    for _ in range(a.reps):
        fem.map_forces(a.model, scatter=sid)
    torch.cuda.synchronize()
    ctx.close()


if __name__ == "__main__":
    main()
