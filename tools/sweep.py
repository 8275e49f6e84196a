#!/usr/bin/env python
"""Secondary measurements of SURVEY §8(d) (not the bench line): one JSON line each.

  C3  StVK (and NH) force+stiffness map on a ~1e7-tet blob mesh, fp32 and fp64,
      segmented vs chunk vs atomic scatter -- tets/s and fraction of measured HBM peak.
  C4  edge-relation matvec sweep over Kuhn-6 meshes (1e5 .. 1e8 tets), fp32 vs
      fp64 -- GB/s and fraction of peak (algorithmic bytes of §8(d)).

Timing: CUDA events on the launching stream around each launch (library
instrumentation), warm-up first, L2 flushed before every timed launch.

    python tools/sweep.py [--c3] [--c4] [--sizes 26,55,119] [--reps 5]
"""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402  (peaks, byte models)


def _flush(buf):
    buf.zero_()


def _prewarm(seconds=0.5):
    """Busy the GPU so clocks leave idle before anything is timed."""
    import time

    import torch
    a = torch.empty(1 << 26, device="cuda")
    t = time.perf_counter()
    while time.perf_counter() - t < seconds:
        a.mul_(1.0)
        torch.cuda.synchronize()


def run_c3(reps, dtypes=("f32", "f64"), models=("stvk", "nh"), target=10_000_000, kuhn_n=0,
           scatters=("segmented", "chunk", "atomic")):
    import numpy as np
    import torch

    from paper_1506_07577_b200 import _abi as A
    from paper_1506_07577_b200 import ebb
    from paper_1506_07577_b200.tetfem import TetFEM
    from synth import mesh as M
    from synth import state as S

    if kuhn_n:
        n = kuhn_n
        X, tets = M.kuhn6(n)
        wl, mname = ("C2" if n == 55 else "C4"), f"kuhn6 n={n}"
    else:
        X, tets, n = M.blob(target)
        wl, mname = "C3", f"blob n={n}"
    free = S.fixed_mask(X, n)
    u = S.twist_u(X, n, 6, free=free)
    mu, lam = S.materials(tets.shape[0], 1e6, 0.3, spread=0.1)
    peak, src = bench._peaks()
    flush = torch.empty(bench.FLUSH_BYTES, dtype=torch.uint8, device="cuda")
    for dt in dtypes:
        ctx = ebb.Context(0)
        fem = TetFEM(ctx, X, tets, dtype=dt, mu=mu, lam=lam, free=free, u=u, name="c3")
        T, V, E = fem.nt, fem.nv, fem.ne
        bf = 4 if dt == "f32" else 8
        for model in models:
            ids = {"segmented": A.SCATTER_SEGMENTED, "atomic": A.SCATTER_ATOMIC, "color": A.SCATTER_COLOR,
                   "chunk": A.SCATTER_CHUNK, "chunk_red": A.SCATTER_CHUNK_RED}
            for scat in scatters:
                sid = ids[scat]
                fem.map_forces(model, scatter=sid)
                torch.cuda.synchronize()
                ctx.timing(True)
                ctx.timing_read(A.K_TET_MAP, reset=True)
                for _ in range(reps):
                    _flush(flush)
                    fem.map_forces(model, scatter=sid)
                ms, nl = ctx.timing_read(A.K_TET_MAP, reset=True)
                ctx.timing(False)
                us = 1e3 * ms / nl
                b = bench.bytes_map(T, V, E, bf)
                plan = fem.plan_stats() if scat == "segmented" else None
                print(json.dumps({"plan": plan, "workload": wl, "mesh": mname, "tets": T, "verts": V, "edge_rows": E,
                                  "dtype": dt, "model": model, "scatter": scat, "avg_us": us,
                                  "tets_per_s": T / (us * 1e-6), "algorithmic_bytes": b,
                                  "hbm_frac": b / (us * 1e-6) / 1e9 / peak, "peak_gbs": peak, "peak_source": src}),
                      flush=True)
        ctx.close()
        del fem
    del np


def run_c4(sizes, reps):
    import numpy as np
    import torch

    from paper_1506_07577_b200 import _abi as A
    from paper_1506_07577_b200 import ebb
    from paper_1506_07577_b200.tetfem import TetFEM
    from synth import mesh as M

    peak, src = bench._peaks()
    flush = torch.empty(bench.FLUSH_BYTES, dtype=torch.uint8, device="cuda")
    for n in sizes:
        X, tets = M.kuhn6(n)
        for dt in ("f32", "f64"):
            ctx = ebb.Context(0)
            fem = TetFEM(ctx, X, tets, dtype=dt, name=f"c4_{n}_{dt}")
            rng = np.random.default_rng(6)
            fem.K.write(rng.uniform(-1, 1, size=(fem.ne, 9)))
            P = fem.verts.field("p", dt, (3, 1), init=rng.uniform(-1, 1, size=(fem.nv, 3)))
            Q = fem.verts.field("q", dt, (3, 1))
            fem.matvec(fem.K, P, Q)
            torch.cuda.synchronize()
            ctx.timing(True)
            ctx.timing_read(A.K_EDGE_MATVEC, reset=True)
            for _ in range(reps):
                _flush(flush)
                fem.matvec(fem.K, P, Q)
            ms, nl = ctx.timing_read(A.K_EDGE_MATVEC, reset=True)
            ctx.timing(False)
            us = 1e3 * ms / nl
            bf = 4 if dt == "f32" else 8
            b = bench.bytes_matvec(fem.nv, fem.ne, bf)
            print(json.dumps({"workload": "C4", "mesh": f"kuhn6 n={n}", "tets": fem.nt, "verts": fem.nv,
                              "edge_rows": fem.ne, "dtype": dt, "avg_us": us, "gbs": b / (us * 1e-6) / 1e9,
                              "hbm_frac": b / (us * 1e-6) / 1e9 / peak, "algorithmic_bytes": b, "peak_gbs": peak,
                              "peak_source": src}), flush=True)
            ctx.close()
            del fem


def run_c4cg(sizes, reps, dtypes=("f64", "f32")):
    """C4: the full PCG iteration (persistent single-launch solve) per size."""
    import torch

    from paper_1506_07577_b200 import _abi as A
    from paper_1506_07577_b200 import ebb
    from paper_1506_07577_b200.tetfem import TetFEM

    peak, src = bench._peaks()
    flush = torch.empty(bench.FLUSH_BYTES, dtype=torch.uint8, device="cuda")
    w = bench.WORKLOAD
    for n in sizes:
        X, tets, free, u0, mu, lam = bench.make_case(n, w["order_seed"], w["u_seed"], w["E"], w["nu"])
        for dt in dtypes:
            ctx = ebb.Context(0)
            fem = TetFEM(ctx, X, tets, dtype=dt, mu=mu, lam=lam, rho=w["rho"], free=free, u=u0, name=f"cg{n}{dt}")
            fem.implicit_step(w["model"], h=w["h"], iters=w["cg_iters"])
            torch.cuda.synchronize()
            ctx.timing(True)
            ctx.timing_read(A.K_CG_SOLVE, reset=True)
            for _ in range(reps):
                _flush(flush)
                fem.implicit_step(w["model"], h=w["h"], iters=w["cg_iters"])
            ms, nl = ctx.timing_read(A.K_CG_SOLVE, reset=True)
            ctx.timing(False)
            it_us = 1e3 * ms / nl / w["cg_iters"]
            bf = 4 if dt == "f32" else 8
            b = bench.bytes_cg_iter(fem.nv, fem.ne, bf)
            print(json.dumps({"workload": "C4-cg", "mesh": f"kuhn6 n={n}", "tets": fem.nt, "verts": fem.nv,
                              "edge_rows": fem.ne, "dtype": dt, "iter_us": it_us, "iters_per_s": 1e6 / it_us,
                              "gbs": b / (it_us * 1e-6) / 1e9, "hbm_frac": b / (it_us * 1e-6) / 1e9 / peak,
                              "algorithmic_bytes_per_iter": b, "peak_gbs": peak, "peak_source": src}), flush=True)
            ctx.close()
            del fem


def run_spring(sizes, reps, dtypes=("f64", "f32"), steps=50):
    """the Fig. 2 spring-mass iteration (fused one-kernel step
    and the paper's two kernels) per Kuhn-6 size; steps back to back (the
    workload's own loop), CUDA events around `steps` iterations."""
    import numpy as np
    import torch

    from paper_1506_07577_b200 import ebb
    from paper_1506_07577_b200.springmass import SpringMass
    from paper_1506_07577_b200.tetfem import TetFEM
    from synth import mesh as M

    peak, src = bench._peaks()
    flush = torch.empty(bench.FLUSH_BYTES, dtype=torch.uint8, device="cuda")
    for n in sizes:
        X, tets = M.kuhn6(n)
        X, tets = M.permute_vertices(X, tets, 2)
        q0 = X + np.random.default_rng(1).uniform(-0.05 / n, 0.05 / n, X.shape)
        for dt in dtypes:
            ctx = ebb.Context(0)
            fem = TetFEM(ctx, X, tets, dtype=dt, name=f"sp{n}{dt}")
            sm = SpringMass(fem, K=-1.0, dt=1e-4, q=q0, name=f"sp{n}{dt}")
            bf = 8 if dt == "f64" else 4
            V, E = fem.nv, fem.ne
            b_fused = E * (4 + bf) + V * 13 * bf            # head, rest_len; q r + q' w, qd r/w, mass
            b_paper = (E * (4 + bf) + V * 6 * bf) + V * 16 * bf
            gst = torch.cuda.Stream()
            for mode in ("fused", "paper", "fused_graph"):
                fn = {"fused": sm.step, "paper": sm.step_paper,
                      "fused_graph": (lambda: sm.run(2, gst))}[mode]
                for _ in range(5):
                    fn()
                torch.cuda.synchronize()
                res = {}
                for warm in (True, False):
                    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    tot = 0.0
                    per = (2 if mode == "fused_graph" else 1)          # steps per fn() call
                    for _ in range(reps):
                        if not warm:
                            _flush(flush)
                        cs = gst if mode == "fused_graph" else torch.cuda.current_stream()
                        cs.wait_stream(torch.cuda.current_stream())
                        a.record(cs)
                        for _ in range(steps if warm else 1):
                            fn()
                        b.record(cs)
                        torch.cuda.synchronize()
                        tot += a.elapsed_time(b)
                    res["l2_warm" if warm else "l2_flushed"] = 1e3 * tot / (reps * (steps if warm else 1) * per)
                bb = b_paper if mode == "paper" else b_fused
                print(json.dumps({"workload": "spring-mass (Fig. 2)", "mode": mode, "mesh": f"kuhn6 n={n}",
                                  "verts": V, "edge_rows": E, "dtype": dt,
                                  "step_us_back_to_back": res["l2_warm"], "step_us_l2_flushed": res["l2_flushed"],
                                  "algorithmic_bytes": bb,
                                  "hbm_frac_flushed": bb / (res["l2_flushed"] * 1e-6) / 1e9 / peak,
                                  "gbs_back_to_back": bb / (res["l2_warm"] * 1e-6) / 1e9,
                                  "peak_gbs": peak, "peak_source": src}), flush=True)
            ctx.close()
            del fem, sm


def run_ebe(sizes, reps, dtypes=("f64", "f32"), model="nh"):
    """matrix-free element-by-element matvec vs the assembled
    edge-relation matvec on the same mesh and state (L2 flushed)."""
    import numpy as np
    import torch

    from paper_1506_07577_b200 import _abi as A
    from paper_1506_07577_b200 import ebb
    from paper_1506_07577_b200.tetfem import TetFEM

    peak, src = bench._peaks()
    flush = torch.empty(bench.FLUSH_BYTES, dtype=torch.uint8, device="cuda")
    w = bench.WORKLOAD
    for n in sizes:
        X, tets, free, u0, mu, lam = bench.make_case(n, w["order_seed"], w["u_seed"], w["E"], w["nu"])
        for dt in dtypes:
            ctx = ebb.Context(0)
            fem = TetFEM(ctx, X, tets, dtype=dt, mu=mu, lam=lam, rho=w["rho"], free=free, u=u0, name=f"ebe{n}{dt}")
            fem.map_forces(model)
            st = fem.ebe_state(model)
            rng = np.random.default_rng(6)
            P = fem.verts.field("p", dt, (3, 1), init=rng.uniform(-1, 1, size=(fem.nv, 3)))
            Q = fem.verts.field("q", dt, (3, 1))
            res = {}
            for name, fn, kid in (("ebe", lambda: fem.ebe_matvec(st, P, Q, model=model), A.K_EBE_MATVEC),
                                  ("assembled", lambda: fem.matvec(fem.K, P, Q), A.K_EDGE_MATVEC)):
                fn()
                torch.cuda.synchronize()
                ctx.timing(True)
                ctx.timing_read(kid, reset=True)
                for _ in range(reps):
                    _flush(flush)
                    fn()
                ms, nl = ctx.timing_read(kid, reset=True)
                ctx.timing(False)
                res[name] = 1e3 * ms / nl
            bf = 4 if dt == "f32" else 8
            words = 15 if model == "nh" else 26
            b_ebe = fem.nt * (16 + (9 + words) * bf) + fem.nv * 6 * bf
            b_asm = bench.bytes_matvec(fem.nv, fem.ne, bf)
            print(json.dumps({"workload": "EBE vs assembled matvec", "model": model, "mesh": f"kuhn6 n={n}",
                              "tets": fem.nt, "verts": fem.nv, "edge_rows": fem.ne, "dtype": dt,
                              "ebe_us": res["ebe"], "assembled_us": res["assembled"],
                              "ebe_algorithmic_bytes": b_ebe, "assembled_algorithmic_bytes": b_asm,
                              "ebe_hbm_frac": b_ebe / (res["ebe"] * 1e-6) / 1e9 / peak,
                              "assembled_hbm_frac": b_asm / (res["assembled"] * 1e-6) / 1e9 / peak,
                              "peak_gbs": peak, "peak_source": src}), flush=True)
            ctx.close()
            del fem


def run_grid(reps, dtypes=("f32", "f64")):
    """the 5-point periodic stencil on a 8192 x 8192 grid (vec2)
    and Fig. 3 particle interpolation (16M particles), L2 flushed."""
    import numpy as np
    import torch

    from paper_1506_07577_b200 import _abi as A
    from paper_1506_07577_b200 import ebb
    from paper_1506_07577_b200.grid import Grid2

    peak, src = bench._peaks()
    flush = torch.empty(bench.FLUSH_BYTES, dtype=torch.uint8, device="cuda")
    nx = ny = 8192
    npart = 1 << 24
    for dt in dtypes:
        ctx = ebb.Context(0)
        g = Grid2(ctx, nx, ny, name=f"g{dt}")
        rng = np.random.default_rng(0)
        fin = g.cells.field("in", dt, (2, 1), init=rng.standard_normal((nx * ny, 2)))
        fout = g.cells.field("out", dt, (2, 1))
        pos = np.zeros((npart, 3))
        pos[:, 0] = rng.uniform(0, nx, npart)
        pos[:, 1] = rng.uniform(0, ny, npart)
        P, pf, key = g.particles(f"p{dt}", pos, dtype=dt)
        vf = P.field("vel", dt, (2, 1))
        bf = 4 if dt == "f32" else 8
        runs = (("stencil5", lambda: g.stencil(fin, fout, [(0, 0), (1, 0), (-1, 0), (0, 1), (0, -1)],
                                               [-4.0, 1.0, 1.0, 1.0, 1.0]), nx * ny * 2 * bf * 2),
                ("particle_vel", lambda: g.particle_vel(key, fin, pf, vf),
                 npart * (3 * bf + 4 + 2 * bf) + nx * ny * 2 * bf))
        def sorted_vel():
            g.particle_vel(key, fin, pf, vf)
        runs = runs + (("particle_vel_sorted", sorted_vel, npart * (3 * bf + 4 + 2 * bf) + nx * ny * 2 * bf),)
        for name, fn, b in runs:
            if name == "particle_vel_sorted":
                g.sort_particles(P, key)            # particles in dual-cell order
            fn()
            torch.cuda.synchronize()
            ctx.timing(True)
            ctx.timing_read(A.K_GRID, reset=True)
            for _ in range(reps):
                _flush(flush)
                fn()
            ms, nl = ctx.timing_read(A.K_GRID, reset=True)
            ctx.timing(False)
            us = 1e3 * ms / nl
            print(json.dumps({"workload": f"grid2 {name}", "grid": f"{nx}x{ny}", "particles": npart,
                              "dtype": dt, "us": us, "algorithmic_bytes": b,
                              "hbm_frac": b / (us * 1e-6) / 1e9 / peak, "peak_gbs": peak,
                              "peak_source": src}), flush=True)
        ctx.close()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--c3", action="store_true")
    ap.add_argument("--c4", action="store_true")
    ap.add_argument("--sizes", default="26,37,55,79,119")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--c3-tets", type=int, default=10_000_000)
    ap.add_argument("--c2", action="store_true", help="the map sweep on the C2 Kuhn n=55 mesh")
    ap.add_argument("--c4map", action="store_true", help="the map strategies on every --sizes Kuhn mesh")
    ap.add_argument("--c4cg", action="store_true", help="the PCG iteration on every --sizes Kuhn mesh")
    ap.add_argument("--spring", action="store_true", help="the Fig. 2 spring-mass step on every --sizes Kuhn mesh")
    ap.add_argument("--ebe", action="store_true", help="matrix-free vs assembled matvec on every --sizes Kuhn mesh")
    ap.add_argument("--grid", action="store_true", help="2-D grid stencil and particle interpolation")
    ap.add_argument("--scatters", default="segmented,chunk,atomic")
    ap.add_argument("--dtypes", default="f32,f64")
    ap.add_argument("--models", default="stvk,nh")
    a = ap.parse_args()
    from paper_1506_07577_b200 import build
    build.build()
    _prewarm()
    if a.c2:
        run_c3(a.reps, kuhn_n=55, scatters=a.scatters.split(","), dtypes=a.dtypes.split(","),
               models=a.models.split(","))
    if a.c3:
        run_c3(a.reps, target=a.c3_tets, scatters=a.scatters.split(","), dtypes=a.dtypes.split(","),
               models=a.models.split(","))
    if a.c4:
        run_c4([int(x) for x in a.sizes.split(",")], a.reps)
    if a.c4map:
        for n in [int(x) for x in a.sizes.split(",")]:
            run_c3(a.reps, kuhn_n=n, scatters=a.scatters.split(","), dtypes=a.dtypes.split(","),
                   models=a.models.split(","))
    if a.c4cg:
        run_c4cg([int(x) for x in a.sizes.split(",")], a.reps)
    if a.grid:
        run_grid(a.reps, dtypes=a.dtypes.split(","))
    if a.ebe:
        run_ebe([int(x) for x in a.sizes.split(",")], a.reps, dtypes=a.dtypes.split(","))
    if a.spring:
        run_spring([int(x) for x in a.sizes.split(",")], a.reps, dtypes=a.dtypes.split(","))


if __name__ == "__main__":
    main()
