#!/usr/bin/env python
"""C5 (BASELINE configs[4]) on ONE B200: the 100M-tet neo-Hookean implicit
step (Kuhn-6 n=255: 99,488,250 tets, fp64, 50 PCG iterations) -- the single-GPU
point of the 8-GPU config (this run has one GPU).  Times the element map, the
assembly, the PCG iteration and the whole step with the library's CUDA events
(L2 is irrelevant at this size: 45+ GB of state).  No oracle (too large);
parity at this scale is covered by the sampled-row tests.

    python tools/c5.py [--n 255] [--steps 2]
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=255)
    ap.add_argument("--steps", type=int, default=2)
    a = ap.parse_args()
    import torch

    from paper_1506_07577_b200 import _abi as A
    from paper_1506_07577_b200 import build, ebb
    from paper_1506_07577_b200.tetfem import TetFEM

    build.build()
    w = bench.WORKLOAD
    t0 = time.perf_counter()
    # the C2 recipe keeps h^2 E n^2 / rho ~ 60: E scales as 1/n^2
    E_n = w["E"] * (w["n"] / a.n) ** 2
    # stretch ramped off the wall (synth.state.stretch_noise_u): the plain C2
    # recipe's wall shear ~0.05 n inverts 186 tets at n = 255
    X, tets, free, u0, mu, lam = bench.make_case(a.n, w["order_seed"], w["u_seed"], E_n, w["nu"], wall_ramp=0.1)
    t_mesh = time.perf_counter() - t0
    free_b, total_b = torch.cuda.mem_get_info()
    ctx = ebb.Context(0)
    t0 = time.perf_counter()
    fem = TetFEM(ctx, X, tets, dtype="f64", mu=mu, lam=lam, rho=w["rho"], free=free, u=u0, name="c5")
    torch.cuda.synchronize()
    t_setup = time.perf_counter() - t0
    del X, tets, u0, mu, lam
    T, V, E = fem.nt, fem.nv, fem.ne
    t0 = time.perf_counter()
    fem.implicit_step(w["model"], h=w["h"], iters=w["cg_iters"])          # plans + warm-up
    torch.cuda.synchronize()
    t_first = time.perf_counter() - t0
    err_first = ctx.error_counts(reset=True)
    used = free_b - torch.cuda.mem_get_info()[0]
    ctx.timing(True)
    ctx.timing_read(A.K_TET_MAP, reset=True)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(a.steps)]
    for s in range(a.steps):
        ev[s][0].record()
        fem.implicit_step(w["model"], h=w["h"], iters=w["cg_iters"])
        ev[s][1].record()
    torch.cuda.synchronize()
    step_ms = sum(x.elapsed_time(y) for x, y in ev) / a.steps
    # (timing_read(reset=True) clears every kernel's records: read all, then reset)
    t = {name: ctx.timing_read(k) for name, k in
         (("map", A.K_TET_MAP), ("assemble", A.K_ASSEMBLE), ("cg_solve", A.K_CG_SOLVE),
          ("matvec", A.K_EDGE_MATVEC))}
    ctx.timing_read(A.K_TET_MAP, reset=True)
    avg = {k: (1e3 * ms / n if n else None) for k, (ms, n) in t.items()}
    peak, src = bench._peaks()
    it_us = avg["cg_solve"] / w["cg_iters"]
    b_map, b_it = bench.bytes_map(T, V, E), bench.bytes_cg_iter(V, E)
    out = {"workload": f"C5 at P=1: Kuhn-6 n={a.n} ({T} tets, {V} verts, {E} edge rows), NH implicit step + "
                       f"{w['cg_iters']} PCG iterations, fp64, one B200",
           "tets": T, "verts": V, "edge_rows": E, "step_ms": step_ms, "tet_steps_per_s": T / (step_ms * 1e-3),
           "map_us": avg["map"], "map_tets_per_s": T / (avg["map"] * 1e-6),
           "map_hbm_frac": b_map / (avg["map"] * 1e-6) / 1e9 / peak,
           "cg_iter_us": it_us, "cg_iters_per_s": 1e6 / it_us, "cg_hbm_frac": b_it / (it_us * 1e-6) / 1e9 / peak,
           "assemble_us": avg["assemble"], "matvec_us": avg["matvec"], "peak_gbs": peak, "peak_source": src,
           "device_bytes_used": used, "device_bytes_total": total_b, "host_mesh_s": t_mesh,
           "setup_s": t_setup, "first_step_s_incl_plan": t_first, "plan": fem.plan_stats(),
           "E_young": E_n, "errors_first_step": err_first, "errors_timed_steps": ctx.error_counts(reset=True)}
    print(json.dumps(out))
    ctx.close()


if __name__ == "__main__":
    main()
