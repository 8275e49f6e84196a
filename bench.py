#!/usr/bin/env python
"""bench.py -- throughput of the Ebb tet-FEM hot path on B200 (one JSON line).

Workload (BASELINE.json north_star "Target": a 10^7-tet neo-Hookean mesh, the
map and the CG of its implicit solve): neo-Hookean implicit backward-Euler
step with 50 Jacobi-PCG iterations on the Kuhn-6 subdivided cube n=119
(10,110,954 tets, 1,728,000 vertices, 25,575,838 edge rows), fp64.  A "step"
is one pass of the whole hot path: element
force+stiffness map, system assembly, PCG init + 50 iterations, state update.
The C2 workload (BASELINE configs[1], n=55, 998,250 tets) is measured in the
same run as a component.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

value = tets advanced through one full step per second (tet-steps/s), summed
over ranks; the metric's two quantities are top-level too: "map" (tets/s of
the force+stiffness map, fraction of HBM peak) and "cg" (PCG iterations/s,
fraction of HBM peak on the algorithmic and on the ncu-measured DRAM bytes).
--impl reference times the CPU oracle (the reference arm of this tier) on a
bounded sample of the workload.  Under torchrun (N > 1) the global mesh is a
Kuhn cube with round(119 N^(1/3)) cells per side (~10M tets per GPU, weak
scaling), partitioned by the O4 owner maps; each rank runs the distributed
implicit step (paper_1506_07577_b200.dist: ghost tets, u halo and one fused
2-scalar allreduce per PCG iteration over NCCL) -- DESIGN.md §7.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "tets/sec (force+stiffness map) and CG iters/sec at 1/2/4/8 B200; % HBM roofline"
# E scaled as 1/n^2 keeps h^2 E n^2 / rho ~ 60 (the C2 conditioning, DESIGN §3 reading 14); the
# stretch is ramped off the fixed wall (wall_ramp): the plain C2 recipe's wall shear (~0.05 n)
# would invert tets at n = 119 (C5 note)
WORKLOAD = dict(name="T10M", n=119, model="nh", E=2e5 * (55 / 119) ** 2, nu=0.3, rho=1e3, h=1e-2, cg_iters=50,
                order_seed=2, u_seed=1, wall_ramp=0.1)
C2 = dict(name="C2", n=55, model="nh", E=2e5, nu=0.3, rho=1e3, h=1e-2, cg_iters=50, order_seed=2, u_seed=1,
          wall_ramp=0.0)
SAMPLE_N = 55          # oracle sample: the same recipe on the 1/10-size n=55 cube (3-6 s per step, one core)
CPU_BASELINE_STEPS = 3 # ~10-20 s of oracle work for the cpu_baseline field
FLUSH_BYTES = 256 << 20


def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md: 6.65 TB/s)"


def _ncu_entry(kernel, workload):
    """The committed ncu --set full capture of `kernel` at this bench's
    workload (profiles/ncu_traffic.json, tools/ncu_traffic.py), else None."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(p) as f:
            d = json.load(f)
        e = d.get(f"{workload}:{kernel}") or d[kernel]
        if e.get("workload") == workload:
            return e
    except Exception:
        pass
    return None


def _ncu_traffic(kernel, workload):
    """DRAM bytes per launch of `kernel` from that capture, else None."""
    e = _ncu_entry(kernel, workload)
    return float(e["dram_bytes_per_launch"]) if e else None


def _ncu_extra(kernel, workload):
    """SURVEY §8(d)'s other ncu figures of the same capture: L2 hit rate, L2
    red / atom sectors, fp64-pipe utilisation (whatever the capture has)."""
    e = _ncu_entry(kernel, workload)
    if not e:
        return None
    keys = ("l2_hit_rate_pct", "l2_red_sectors", "l2_atom_sectors", "fp64_pipe_pct", "fp64_pipe_inst_pct")
    out = {k: e[k] for k in keys if k in e}
    if out:
        out["capture"] = e.get("capture")
    return out or None


class ClockSampler:
    """Samples SM clock + throttle reasons during the timed region (NVML)."""

    REASONS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown", 0x4: "sw_power_cap",
               0x80: "hw_power_brake_slowdown"}

    def __init__(self, device):
        self.device = device
        self.samples, self.reasons = [], set()
        self.max_mhz = None
        self._stop = threading.Event()
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.hdl = pynvml.nvmlDeviceGetHandleByIndex(device)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.hdl, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.ok = False

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.hdl, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.hdl)
                for bit, name in self.REASONS.items():
                    if r & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.002)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": 0}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def make_case(n, order_seed, u_seed, E, nu, wall_ramp=0.0):
    from synth import mesh as M
    from synth import state as S
    X, tets = M.kuhn6(n)
    if order_seed is not None:
        X, tets = M.permute_vertices(X, tets, order_seed)
    free = S.fixed_mask(X, n)
    u = S.stretch_noise_u(X, n, u_seed, free=free, wall_ramp=wall_ramp)
    mu, lam = S.materials(tets.shape[0], E, nu)
    return X, tets, free, u, mu, lam


def bytes_map(T, V, E, bf=8):
    """compulsory bytes of the force+stiffness map."""
    return T * (4 + 16) * 4 + T * 12 * bf + V * 6 * bf + E * 9 * bf


def bytes_matvec(V, E, bf=8):
    return E * (9 * bf + 4) + V * (4 + 6 * bf)


_OUT = None


def _claim_stdout():
    """The contract is ONE JSON line on stdout: libraries that print to fd 1
    (NCCL's version banner, CUDA/driver notices) are moved to stderr; the
    JSON line goes to the original stdout."""
    global _OUT
    if _OUT is None:
        sys.stdout.flush()
        _OUT = os.fdopen(os.dup(1), "w")
        os.dup2(2, 1)


def emit(line):
    out = _OUT if _OUT is not None else sys.stdout
    out.write(json.dumps(line) + "\n")
    out.flush()


def bytes_cg_iter(V, E, bf=8):
    return bytes_matvec(V, E, bf) + V * 3 * bf * 11


def _e2e_pipelined(ctx, fem, stream, flush, run_step, u_h, v_h, steps, dev):
    """Device time (ms, CUDA events on the compute stream) of `steps`
    end-to-end steps with the host copies overlapped (see run_ours)."""
    import numpy as np
    import torch
    V = fem.nv
    nb = V * 3 * 8
    S = ctx.relation("e2e.stage", V)
    sin = [(S.field(f"u_in{i}", "f64", (3, 1)), S.field(f"v_in{i}", "f64", (3, 1))) for i in range(2)]
    sout = [(S.field(f"u_out{i}", "f64", (3, 1)), S.field(f"v_out{i}", "f64", (3, 1))) for i in range(2)]
    host_out = [(torch.empty((V, 3), dtype=torch.float64, pin_memory=True),
                 torch.empty((V, 3), dtype=torch.float64, pin_memory=True)) for _ in range(2)]
    copy = torch.cuda.Stream(device=dev)
    ev = lambda: torch.cuda.Event()                          # noqa: E731
    staged, used, ready, drained = [ev(), ev()], [ev(), ev()], [ev(), ev()], [ev(), ev()]
    used_rec, drained_rec = [False, False], [False, False]
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

    def h2d(slot):
        su, sv = sin[slot]
        if used_rec[slot]:
            copy.wait_event(used[slot])                      # the step that read this slot has copied it out
        su.write_async(u_h.data_ptr(), nb, copy)
        sv.write_async(v_h.data_ptr(), nb, copy)
        staged[slot].record(copy)

    torch.cuda.synchronize()
    t0.record(stream)
    copy.wait_event(t0)
    h2d(0)
    for k in range(steps):
        s_ = k % 2
        with torch.cuda.stream(stream):
            flush.zero_()
        stream.wait_event(staged[s_])
        fem.u.copy_from(sin[s_][0], stream)
        fem.vel.copy_from(sin[s_][1], stream)
        used[s_].record(stream)
        used_rec[s_] = True
        if k + 1 < steps:
            h2d((k + 1) % 2)
        run_step()
        if drained_rec[s_]:
            stream.wait_event(drained[s_])                   # step k-2's result left this slot
        sout[s_][0].copy_from(fem.u, stream)
        sout[s_][1].copy_from(fem.vel, stream)
        ready[s_].record(stream)
        copy.wait_event(ready[s_])
        sout[s_][0].read_async(host_out[s_][0].data_ptr(), nb, copy)
        sout[s_][1].read_async(host_out[s_][1].data_ptr(), nb, copy)
        drained[s_].record(copy)
        drained_rec[s_] = True
    stream.wait_stream(copy)                                 # the last result is on the host
    t1.record(stream)
    t1.synchronize()
    # every step starts from (u0, v0): the last result on the host is the state
    last = host_out[(steps - 1) % 2]
    assert np.array_equal(last[0].numpy(), fem.u.read()) and np.array_equal(last[1].numpy(), fem.vel.read())
    S.free()
    return t0.elapsed_time(t1)


def _host_cpu():
    """The host the oracle ran on (report nproc and the CPU model)."""
    model = "?"
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"cpu_model": model, "nproc": os.cpu_count()}


def cpu_baseline(steps=CPU_BASELINE_STEPS):
    """The oracle, as it stands, on a bounded sample of the workload (1 thread)."""
    import numpy as np

    import oracle
    w = C2
    X, tets, free, u, mu, lam = make_case(SAMPLE_N, w["order_seed"], w["u_seed"], w["E"], w["nu"])
    m = oracle.Mesh(X, tets, rho=w["rho"])
    v = np.zeros_like(u)
    t0 = time.perf_counter()
    for _ in range(steps):        # every step from the seeded state, as in the timed GPU steps
        oracle.implicit_step(m, w["model"], u, v, mu, lam, free, w["h"], iters=w["cg_iters"])
    dt = time.perf_counter() - t0
    T = tets.shape[0]
    return {"value": T * steps / dt, "unit": "tets/s", "cores": 1, "kind": "oracle",
            "sample": f"{steps} full implicit NH step(s) (map + assembly + 50 PCG iterations) of the same "
                      f"recipe on the 1/10-size Kuhn-6 n={SAMPLE_N} cube ({T} tets: the C2 workload); "
                      f"single-threaded C oracle (gcc -O2, generic 4th-order stiffness tensor)",
            "seconds": dt, **_host_cpu()}


def run_reference(args, rank, world):
    if rank != 0:
        return
    # warm-up: one untimed sample step (if W > 0), then K timed sample steps
    import numpy as np

    import oracle
    w = C2
    X, tets, free, u, mu, lam = make_case(SAMPLE_N, w["order_seed"], w["u_seed"], w["E"], w["nu"])
    m = oracle.Mesh(X, tets, rho=w["rho"])
    v = np.zeros_like(u)
    for _ in range(min(args.warmup, 1)):
        oracle.implicit_step(m, w["model"], u, v, mu, lam, free, w["h"], iters=w["cg_iters"])
    t0 = time.perf_counter()
    for _ in range(args.steps):   # every step from the seeded state, as in our arm (state_reset)
        oracle.implicit_step(m, w["model"], u, v, mu, lam, free, w["h"], iters=w["cg_iters"])
    dt = time.perf_counter() - t0
    T = tets.shape[0]
    val = T * args.steps / dt
    cb = {"value": val, "unit": "tets/s", "cores": 1, "kind": "oracle",
          "sample": f"each step = one implicit NH step (map + assembly + 50 PCG its) of the same recipe on the "
                    f"1/10-size Kuhn-6 n={SAMPLE_N} cube ({T} tets); single-threaded C oracle", **_host_cpu()}
    line = {"impl": "reference", "metric": METRIC, "value": val, "unit": "tets/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * dt / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": _config(world),
            "cpu_baseline": cb, "e2e": {"value": val, "unit": "tets/s", "h2d_bytes_per_step": 0,
                                        "d2h_bytes_per_step": 0}}
    emit(line)


def _config(world, sample=False, n=None):
    from synth import mesh as M
    n = SAMPLE_N if sample else (n or WORKLOAD["n"])
    T, V, U, E = M.kuhn_counts(n)
    return {"workload": f"{WORKLOAD['name']} (BASELINE north_star target): neo-Hookean implicit backward-Euler "
                        f"step + 50 Jacobi-PCG iterations, Kuhn-6 subdivided cube n={n} ({T} tets, {V} verts, "
                        f"{E} edge rows), fp64"
                        + (f" [CPU oracle on the 1/10-size n={SAMPLE_N} sample]" if sample else ""),
            "tets": T, "verts": V, "edge_rows": E, "h": WORKLOAD["h"], "cg_iters": WORKLOAD["cg_iters"],
            "E_young": WORKLOAD["E"], "nu": WORKLOAD["nu"], "wall_ramp": WORKLOAD["wall_ramp"],
            "l2": "flushed between timed steps (256 MiB write); per-step working set ~5 GB > 126 MB L2",
            "state": "every step starts from the seeded initial state (u0, v0): the same physical step each time, "
                     "reset outside the timed events",
            "parallelism": "single GPU" if world == 1 else f"{world} GPUs, domain decomposition (weak)"}


def state_reset(fem, stream):
    """Every step starts from the seeded initial state (u0, v0): the same
    physical step -- one batch of synthetic input -- each time.  Left to
    evolve, the soft T10M body sags under gravity and inverts tets after ~20
    unconverged 50-iteration steps (NaN from step 22), and a step timed on
    that state would be physically meaningless.  The copy runs on `stream`,
    outside the timed events (inputs resident in HBM, like the L2 flush)."""
    import torch
    u0, v0 = fem.u.tensor().clone(), fem.vel.tensor().clone()

    def reset():
        with torch.cuda.stream(stream):
            fem.u.tensor().copy_(u0)
            fem.vel.tensor().copy_(v0)
    return reset


def _measure(ctx, fem, w, stream, flush, steps, warmup, use_graph, world=1, clocks_device=None):
    """W warm-up steps, then K timed steps (one CUDA graph per step), L2 flushed
    and the state reset to (u0, v0) between steps outside the events;
    per-kernel times from the library's event records (graph event nodes)."""
    import torch
    import torch.distributed as dist

    from paper_1506_07577_b200 import _abi as A
    reset = state_reset(fem, stream)

    def step():
        reset()
        fem.implicit_step(w["model"], h=w["h"], iters=w["cg_iters"], stream=stream)

    # clocks ramp from idle: untimed steps for >= 0.5 s before the W warm-up steps
    t_pre = time.perf_counter()
    while time.perf_counter() - t_pre < 0.5:
        step()
        torch.cuda.synchronize()
    for _ in range(warmup):
        step()
    torch.cuda.synchronize()
    ctx.error_counts(reset=True)
    ctx.timing(True)
    ctx.timing_read(0, reset=True)
    graph = None
    if use_graph:
        # one implicit step captured as a CUDA graph (kernel timers become graph
        # event nodes: each replay re-records them)
        reset()
        ctx.graph_begin(stream)
        fem.implicit_step(w["model"], h=w["h"], iters=w["cg_iters"], stream=stream)
        graph = ctx.graph_end(stream)
        reset()
        ctx.graph_launch(graph, stream)          # untimed replay
        torch.cuda.synchronize()

    def run_step():
        # the state reset is part of step() (eager) and outside the graph
        if graph is None:
            fem.implicit_step(w["model"], h=w["h"], iters=w["cg_iters"], stream=stream)
        else:
            ctx.graph_launch(graph, stream)

    kids = (("tet_map", A.K_TET_MAP), ("edge_matvec", A.K_EDGE_MATVEC), ("cg_update", A.K_CG_UPDATE),
            ("cg_dir", A.K_CG_DIR), ("assemble", A.K_ASSEMBLE), ("cg_solve", A.K_CG_SOLVE))
    kt = {name: {"total_ms": 0.0, "launches": 0} for name, _ in kids}
    if graph is None:
        ctx.timing_read(0, reset=True)
    ctx.launch_count(reset=True)
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(clocks_device if clocks_device is not None else 0) as clk:
        for k in range(steps):
            with torch.cuda.stream(stream):
                flush.zero_()                          # L2 flush, outside the timed events
            reset()                                    # state (u0, v0), outside the timed events
            evs[k][0].record(stream)
            run_step()
            evs[k][1].record(stream)
            if graph is not None:
                # read this replay's kernel events before the next replay re-records them
                evs[k][1].synchronize()
                for name, kid in kids:
                    ms, n = ctx.timing_read(kid)
                    kt[name]["total_ms"] += ms
                    kt[name]["launches"] += n
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    launches = ctx.launch_count(reset=True)
    t_ms = sum(a.elapsed_time(b) for a, b in evs)
    if graph is None:
        for name, kid in kids:
            ms, n = ctx.timing_read(kid)
            kt[name] = {"total_ms": ms, "launches": n}
    for v in kt.values():
        v["avg_us"] = 1e3 * v["total_ms"] / max(v["launches"], 1)
    ctx.timing(False)
    return {"t_ms": t_ms, "kt": kt, "launches": launches, "clocks": clk.summary(),
            "errors": ctx.error_counts(reset=True), "graph": graph, "run_step": run_step, "reset": reset}


def _components(fem, w, kt, t_ms, peak, workload_name):
    """The metric's two quantities (map tets/s, CG iterations/s) with their
    fractions of HBM peak (SURVEY §8(d) algorithmic bytes; the CG also on the
    DRAM bytes ncu measured for this workload, when captured)."""
    T, V, E = fem.nt, fem.nv, fem.ne
    mv, mp, cs = kt["edge_matvec"], kt["tet_map"], kt["cg_solve"]
    iters = w["cg_iters"]
    b_map, b_it = bytes_map(T, V, E), bytes_cg_iter(V, E)
    if cs["launches"]:
        cg_it_us = cs["avg_us"] / iters
    else:
        cg_it_us = mv["avg_us"] + kt["cg_update"]["avg_us"] + kt["cg_dir"]["avg_us"]
    dram = _ncu_traffic("cg_solve", workload_name)
    cg = {"iters_per_s": 1e6 / cg_it_us, "iter_us": cg_it_us,
          "hbm_frac": b_it / (cg_it_us * 1e-6) / 1e9 / peak, "bytes_per_iter": b_it,
          "variant": {1: "saad (k_cg_persistent)", 2: "single-reduction (k_cg1_persistent)",
                      3: "symmetric (k_cg_sym_persistent)"}.get(fem.cg_variant(), "?")}
    if dram is not None and cs["launches"]:
        cg["dram_bytes_per_iter"] = dram / iters
        cg["hbm_frac_dram"] = dram / (cs["avg_us"] * 1e-6) / 1e9 / peak
    cg_ncu = _ncu_extra("cg_solve", workload_name)
    if cg_ncu:
        cg["ncu"] = cg_ncu
    map_ncu = _ncu_extra("tet_map", workload_name)
    return {
        "map": {"tets_per_s": T / (mp["avg_us"] * 1e-6), "avg_us": mp["avg_us"],
                "hbm_frac": b_map / (mp["avg_us"] * 1e-6) / 1e9 / peak, "bytes": b_map,
                "kernel": "k_tet_map_seg (SEGMENTED)", **({"ncu": map_ncu} if map_ncu else {})},
        "cg": cg,
        "ms_per_step": t_ms,
    }


def run_ours(args, rank, world, local_rank):
    import torch

    from paper_1506_07577_b200 import build as B
    from paper_1506_07577_b200 import ebb
    from paper_1506_07577_b200.tetfem import TetFEM

    B.build()
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    w = WORKLOAD
    X, tets, free, u0, mu, lam = make_case(w["n"], w["order_seed"], w["u_seed"], w["E"], w["nu"],
                                           wall_ramp=w["wall_ramp"])
    ctx = ebb.Context(local_rank)
    fem = TetFEM(ctx, X, tets, dtype="f64", mu=mu, lam=lam, rho=w["rho"], free=free, u=u0, name="bench")
    del X, tets
    T, V, E = fem.nt, fem.nv, fem.ne
    stream = torch.cuda.Stream(device=dev)
    flush = torch.empty(FLUSH_BYTES, dtype=torch.uint8, device=dev)
    M_ = _measure(ctx, fem, w, stream, flush, args.steps, args.warmup, not args.no_graph, world, local_rank)
    t_ms, kt, graph, run_step = M_["t_ms"], M_["kt"], M_["graph"], M_["run_step"]
    value = world * T * args.steps / (t_ms / 1e3)

    # ---- end to end through the public API: the step's input state (u0, v0)
    # from pinned host memory, the step, the new state (u, v) back to the host
    M_["reset"]()
    torch.cuda.synchronize()
    u_h = torch.empty((V, 3), dtype=torch.float64, pin_memory=True)
    v_h = torch.empty((V, 3), dtype=torch.float64, pin_memory=True)
    u_h.copy_(torch.from_numpy(fem.u.read()))
    v_h.copy_(torch.from_numpy(fem.vel.read()))
    u_o = torch.empty_like(u_h).pin_memory()
    v_o = torch.empty_like(v_h).pin_memory()
    nb = V * 3 * 8
    e2e_ms = 0.0
    for k in range(args.steps):
        with torch.cuda.stream(stream):
            flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        fem.u.write_async(u_h.data_ptr(), nb, stream)
        fem.vel.write_async(v_h.data_ptr(), nb, stream)
        run_step()
        fem.u.read_into(u_o.data_ptr(), nb, stream)      # synchronous
        fem.vel.read_into(v_o.data_ptr(), nb, stream)
        b.record(stream)
        b.synchronize()
        e2e_ms += a.elapsed_time(b)
    serial = world * T * args.steps / (e2e_ms / 1e3)
    # pipelined (how a serving loop runs it): every step's inputs still come
    # from pinned host memory and every step's result goes back to it inside
    # the timed region, but the copies of step k+1's inputs and of step k-1's
    # result run on a copy stream while step k computes.  Device staging
    # fields (two slots each way) decouple the copies from the step's own
    # u, v, which the step reads and writes; the stage <-> state moves are
    # device copies (ebb_field_copy) on the compute stream.
    pe_ms = _e2e_pipelined(ctx, fem, stream, flush, run_step, u_h, v_h, args.steps, dev)
    e2e = {"value": world * T * args.steps / (pe_ms / 1e3), "unit": "tets/s",
           "h2d_bytes_per_step": 2 * nb, "d2h_bytes_per_step": 2 * nb, "pipelined": True,
           "serial_value": serial,
           "api": "per step: ebb_field_write (pinned host u0, v0 -> device stage, copy stream) -> ebb_field_copy "
                  "(stage -> u, v) -> implicit step (TetFEM.implicit_step as captured graph) -> ebb_field_copy "
                  "(u, v -> stage) -> ebb_field_read_async (stage -> pinned host, copy stream); the copies of "
                  "steps k+1 / k-1 overlap step k; serial_value: the same with nothing overlapped"}

    # ---- roofline of the dominant kernel (largest share of the timed step)
    peak, peak_src = _peaks()
    iters = w["cg_iters"]
    b_mv, b_map, b_it = bytes_matvec(V, E), bytes_map(T, V, E), bytes_cg_iter(V, E)
    shares = {k: v["total_ms"] / t_ms for k, v in kt.items()}
    dom = max(shares, key=shares.get)
    per_launch = {"edge_matvec": b_mv, "tet_map": b_map, "cg_solve": iters * b_it}
    if dom not in per_launch:
        dom = "edge_matvec"
    d = kt[dom]
    ach = per_launch[dom] / (d["avg_us"] * 1e-6) / 1e9
    cgk = "k_cg1_persistent (single-reduction PCG" if fem.cg_variant() == 2 else "k_cg_persistent (Saad PCG"
    traffic = _ncu_traffic(dom, w["name"])
    roof = {"kernel": {"cg_solve": cgk + ", all 50 iterations in one launch)",
                       "edge_matvec": "k_spmv_tma", "tet_map": "k_tet_map_seg"}[dom],
            "bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak,
            "peak_source": peak_src, "traffic": traffic, "algorithmic_bytes_per_launch": per_launch[dom],
            "bytes_model": "SURVEY 8(d): PCG iteration = E(9 b_f + 4) + V(4 + 6 b_f) + 33 V b_f, x 50 iterations"
                           if dom == "cg_solve" else "SURVEY 8(d)",
            "avg_launch_us": d["avg_us"], "share_of_step": shares[dom]}
    if traffic is not None:
        roof["frac_dram_measured"] = traffic / (d["avg_us"] * 1e-6) / 1e9 / peak
        roof["traffic_source"] = "profiles/ncu_traffic.json (ncu --set full capture of this workload)"
    comps = _components(fem, w, kt, t_ms / args.steps, peak, w["name"])
    comps.update({"kernel_times": kt, "shares": shares})
    launches, clocks, errs = M_["launches"], M_["clocks"], M_["errors"]
    ctx.close()
    del fem

    # ---- C2 (BASELINE configs[1], 1M tets) as a component, same method
    c2 = None
    if not args.no_c2:
        wc = C2
        Xc, tc, fc, uc, muc, lamc = make_case(wc["n"], wc["order_seed"], wc["u_seed"], wc["E"], wc["nu"])
        ctx2 = ebb.Context(local_rank)
        fem2 = TetFEM(ctx2, Xc, tc, dtype="f64", mu=muc, lam=lamc, rho=wc["rho"], free=fc, u=uc, name="benchc2")
        steps2 = max(3, min(args.steps, 10))
        M2 = _measure(ctx2, fem2, wc, stream, flush, steps2, max(3, args.warmup), not args.no_graph, 1, local_rank)
        c2 = _components(fem2, wc, M2["kt"], M2["t_ms"] / steps2, peak, "C2")
        c2.update({"workload": "C2 (BASELINE configs[1]): Kuhn-6 n=55, 998,250 tets, NH implicit step + 50 PCG "
                               "iterations, fp64", "steps": steps2,
                   "tets_per_s": fem2.nt * steps2 / (M2["t_ms"] / 1e3)})
        ctx2.close()
        del fem2

    line = {"metric": METRIC, "value": value, "unit": "tets/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t_ms / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded Kuhn-6 cube, stretch+noise displacement, no external meshes)",
            "config": dict(_config(world), launch="one CUDA graph per step" if graph is not None else "eager"),
            "map": comps["map"], "cg": comps["cg"],
            "roofline": roof, "e2e": e2e, "gpu_launches": launches,
            "clocks": clocks, "components": {"kernel_times": kt, "shares": shares, "c2": c2},
            "device_errors": errs}
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline()
    if rank == 0:
        emit(line)


def run_dist(args, rank, world, local_rank):
    """N > 1: one partition of a global weak-scaled mesh per rank (NCCL transport)."""
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_1506_07577_b200 import _abi as A
    from paper_1506_07577_b200 import build as B
    from paper_1506_07577_b200 import dist as D
    from paper_1506_07577_b200 import ebb

    B.build()
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    w = WORKLOAD
    n = int(round(w["n"] * world ** (1.0 / 3.0)))
    E_n = w["E"] * (w["n"] / n) ** 2    # keep h^2 E n^2 / rho ~ 60 (SURVEY §8(c) recipe)
    # stretch ramped off the wall: the plain recipe's wall shear (~0.05 n) inverts tets at large n
    X, tets, free, u0, mu, lam = make_case(n, w["order_seed"], w["u_seed"], E_n, w["nu"], wall_ramp=0.1)
    ctx = ebb.Context(local_rank)
    # this rank's local problem from the device partition (the global mesh is
    # freed again; only local-size arrays come back to the host)
    t_part = time.perf_counter()
    part = D.partition_rank(ctx, X, tets, world, rank, name="global")
    stream = torch.cuda.Stream(device=dev)
    R = D.GpuRank(ctx, rank, part, X, free, u0, np.zeros_like(u0), mu, lam, rho=w["rho"], stream=stream,
                  name=f"rank{rank}")
    t_part = time.perf_counter() - t_part
    cg_var = args.dist_cg
    peer = None
    if cg_var == "peer":
        # the fused multi-GPU PCG: one kernel per solve; u / x / z_0 halos as
        # P2P stores into the peers' (CUDA-IPC mapped) ghost rows and the CG
        # scalars through peer mailboxes -- no NCCL on the step; no fallback
        T = None
        peer = D.PeerPCG([R], comm=dist.group.WORLD if world > 1 else None, stream=stream)
        transport = "peer memory (CUDA IPC over NVLink; ebb_cg_peer_step)"
    else:
        # NCCL inside the library (ebb_comm_*); no fallback: a failure here ends the run
        T = D.NcclTransport(ctx, rank, world, stream=stream)
        transport = "nccl (in-library, ebb_comm_*)"
    T_global = tets.shape[0]
    flush = torch.empty(FLUSH_BYTES, dtype=torch.uint8, device=dev)

    kmv = A.K_EDGE_MATVEC if cg_var == "saad" else A.K_CG_SOLVE   # the streamed-matrix kernel

    reset = state_reset(R.fem, stream)       # local u, v (owned + ghost rows) back to (u0, v0)

    def step():
        D.implicit_step([R], T, w["model"], h=w["h"], iters=w["cg_iters"], variant=cg_var, peer=peer)

    t_pre = time.perf_counter()              # clocks ramp from idle (see run_ours)
    while time.perf_counter() - t_pre < 0.5:
        reset()
        step()
        torch.cuda.synchronize()
    for _ in range(args.warmup):
        reset()
        step()
    torch.cuda.synchronize()
    ctx.timing(True)
    ctx.timing_read(0, reset=True)
    graph = None
    if not args.no_graph:
        # the whole distributed step -- kernels and the in-library NCCL calls on
        # one stream -- captured once and replayed (no host loop per iteration)
        reset()
        ctx.graph_begin(stream)
        step()
        graph = ctx.graph_end(stream)
        reset()
        ctx.graph_launch(graph, stream)       # untimed replay (keeps the captured timer records)
        torch.cuda.synchronize()
    ctx.launch_count(reset=True)
    ctx.error_counts(reset=True)
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    mp_tot, mp_cnt, mv_tot, mv_cnt = 0.0, 0, 0.0, 0
    dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local_rank) as clk:
        for k in range(args.steps):
            with torch.cuda.stream(stream):
                flush.zero_()
            reset()
            evs[k][0].record(stream)
            if graph is None:
                step()
            else:
                ctx.graph_launch(graph, stream)
            evs[k][1].record(stream)
            if graph is not None:
                evs[k][1].synchronize()               # read this replay's kernel events
                ms_, n_ = ctx.timing_read(A.K_TET_MAP)
                mp_tot += ms_
                mp_cnt += n_
                ms_, n_ = ctx.timing_read(kmv)
                mv_tot += ms_
                mv_cnt += n_
        torch.cuda.synchronize()
    dist.barrier()
    launches = ctx.launch_count(reset=True)
    errs = ctx.error_counts(reset=True)
    if errs.get("peer_timeouts"):
        # a peer never arrived at a mailbox exchange: the numbers would be
        # those of an abandoned solve -- fail loudly instead of reporting them
        raise RuntimeError(f"rank {rank}: {errs['peer_timeouts']} peer waits abandoned (error word [3])")
    t_ms = sum(a.elapsed_time(b) for a, b in evs)
    mv_ms, mv_n = ctx.timing_read(kmv)
    mp_ms, mp_n = ctx.timing_read(A.K_TET_MAP, reset=True)
    if graph is not None:
        mp_ms, mp_n, mv_ms, mv_n = mp_tot, mp_cnt, mv_tot, mv_cnt
    tt = torch.tensor([t_ms], device=dev, dtype=torch.float64)
    dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    t_ms = float(tt.item())
    value = T_global * args.steps / (t_ms / 1e3)
    # ---- end to end: every rank uploads its local u, v from pinned host memory,
    # runs the step (graph replay incl. the NCCL calls) and reads u, v back
    V_loc = R.fem.nv
    reset()
    torch.cuda.synchronize()
    u_h = torch.empty((V_loc, 3), dtype=torch.float64, pin_memory=True)
    v_h = torch.empty((V_loc, 3), dtype=torch.float64, pin_memory=True)
    u_h.copy_(torch.from_numpy(R.fem.u.read()))
    v_h.copy_(torch.from_numpy(R.fem.vel.read()))
    u_o = torch.empty_like(u_h).pin_memory()
    v_o = torch.empty_like(v_h).pin_memory()
    nb = V_loc * 3 * 8
    e2e_ms = 0.0
    dist.barrier()
    for k in range(args.steps):
        with torch.cuda.stream(stream):
            flush.zero_()
        a_, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a_.record(stream)
        R.fem.u.write_async(u_h.data_ptr(), nb, stream)
        R.fem.vel.write_async(v_h.data_ptr(), nb, stream)
        if graph is None:
            step()
        else:
            ctx.graph_launch(graph, stream)
        R.fem.u.read_into(u_o.data_ptr(), nb, stream)
        R.fem.vel.read_into(v_o.data_ptr(), nb, stream)
        b_.record(stream)
        b_.synchronize()
        e2e_ms += a_.elapsed_time(b_)
    dist.barrier()
    pe_ms = _e2e_pipelined(ctx, R.fem, stream, flush, lambda: step() if graph is None else
                           ctx.graph_launch(graph, stream), u_h, v_h, args.steps, dev)
    tt = torch.tensor([e2e_ms, pe_ms], device=dev, dtype=torch.float64)
    dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    e2e_ms, pe_ms = float(tt[0].item()), float(tt[1].item())
    e2e = {"value": T_global * args.steps / (pe_ms / 1e3), "unit": "tets/s", "h2d_bytes_per_step": 2 * nb,
           "d2h_bytes_per_step": 2 * nb, "pipelined": True,
           "serial_value": T_global * args.steps / (e2e_ms / 1e3),
           "api": "per rank: ebb_field_write (pinned host local u0, v0 -> stage, copy stream) -> ebb_field_copy -> "
                  "distributed implicit step (graph replay) -> ebb_field_copy -> ebb_field_read_async (copy "
                  "stream), the copies of steps k+1 / k-1 overlapping step k; bytes of this rank; max over ranks"}
    peak, peak_src = _peaks()
    E_loc = R.fem.ne
    # single: one launch = one PCG iteration of the local rows (the prologue
    # launch moves about the same bytes); peer: one launch = all iterations
    # (+ the prologue matvec); saad: the MATVEC phase kernel
    if cg_var == "single":
        b_mv = bytes_cg_iter(V_loc, E_loc)
        kname = "k_cg1_persistent (one single-reduction phase per launch)"
    elif cg_var == "peer":
        b_mv = (w["cg_iters"] + (1 if peer.variant == "single" else 0)) * bytes_cg_iter(V_loc, E_loc)
        kname = (f"k_cg_peer1 ({peer.variant} body; fused multi-GPU PCG, all iterations in one launch, halos and "
                 f"scalar exchanges over peer memory)")
    else:
        b_mv = bytes_matvec(V_loc, E_loc)
        kname = "edge_matvec (Saad MATVEC phase)"
    avg_mv = 1e3 * mv_ms / max(mv_n, 1)
    roof = {"kernel": kname, "bound": "hbm", "achieved": b_mv / (avg_mv * 1e-6) / 1e9, "peak": peak,
            "unit": "GB/s", "frac": b_mv / (avg_mv * 1e-6) / 1e9 / peak, "peak_source": peak_src, "traffic": None,
            "algorithmic_bytes_per_launch": b_mv, "avg_launch_us": avg_mv, "rank": rank}
    cfg = _config(world)
    cfg.update({"workload": f"{WORKLOAD['name']} recipe weak-scaled: Kuhn-6 n={n} ({T_global} tets, {X.shape[0]} verts) split over "
                            f"{world} GPUs by the O4 owner maps (ghost tets; per PCG iteration "
                            + {"single": "one fused 2-scalar allreduce + u halo, single-reduction phases over NCCL",
                               "saad": "z halo + 2 scalar allreduces, Saad phases over NCCL",
                               "peer": "u / x halo as P2P stores + a 2-scalar mailbox exchange inside ONE fused "
                                       "single-reduction PCG kernel"}[cg_var]
                            + "), fp64", "transport": transport, "pcg": cg_var if peer is None else f"peer ({peer.variant})",
                "tets": T_global,
                "parallelism": f"domain decomposition x{world} ("
                               + ("peer-memory halo + scalar exchange in the PCG kernel" if cg_var == "peer"
                                  else "NCCL halo + allreduce") + ")"})
    line = {"metric": METRIC, "value": value, "unit": "tets/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t_ms / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded Kuhn-6 cube, stretch+noise displacement)",
            "config": cfg, "roofline": roof, "gpu_launches": launches, "clocks": clk.summary(),
            "e2e": e2e, "device_errors": errs,
            "components": {"map_avg_us": 1e3 * mp_ms / max(mp_n, 1), "matvec_avg_us": avg_mv,
                           "local_tets": int(R.fem.nt), "local_verts": int(V_loc),
                           "owned_verts": int(part["n_owned"]), "partition_setup_s": t_part}}
    if rank == 0:
        emit(line)
    if peer is not None:
        dist.barrier()                        # no peer still reads a buffer this rank is about to unmap / free
        peer.close()
    ctx.close()


def run_dist_map(args, rank, world, local_rank):
    """BASELINE configs[2] (C3): the StVK force + stiffness map on the ~1e7-tet
    synthetic blob, fp32, over N GPUs with the position halo (strong scaling:
    the same global mesh at every N).  A step = the u halo exchange (owners ->
    ghosts, NCCL) + the map of every local (owned + ghost) tet."""
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_1506_07577_b200 import _abi as A
    from paper_1506_07577_b200 import build as B
    from paper_1506_07577_b200 import dist as D
    from paper_1506_07577_b200 import ebb
    from synth import mesh as M
    from synth import state as S

    B.build()
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    X, tets, n = M.blob(10_000_000)
    free = S.fixed_mask(X, n)
    u0 = S.twist_u(X, n, 6, free=free)
    mu, lam = S.materials(tets.shape[0], 1e6, 0.3, spread=0.1)
    ctx = ebb.Context(local_rank)
    t_part = time.perf_counter()
    part = D.partition_rank(ctx, X, tets, world, rank, name="c3")
    stream = torch.cuda.Stream(device=dev)
    R = D.GpuRank(ctx, rank, part, X, free, u0, np.zeros_like(u0), mu, lam, dtype="f32", stream=stream,
                  name=f"c3r{rank}")
    t_part = time.perf_counter() - t_part
    if args.dist_halo == "peer":
        # the position halo as one peer-memory push kernel (CUDA IPC of the
        # peers' u; no NCCL on the step)
        T = None
        halo = D.PeerHalo([R], "disp", comm=dist.group.WORLD if world > 1 else None, stream=stream)
        transport = "peer memory (CUDA IPC over NVLink; ebb_peer_halo_push)"
    else:
        T = D.NcclTransport(ctx, rank, world, stream=stream)
        halo = None
        transport = "nccl (in-library, ebb_comm_*)"
    T_global = tets.shape[0]
    flush = torch.empty(FLUSH_BYTES, dtype=torch.uint8, device=dev)

    def step():
        D.map_step([R], T, "stvk", halo=halo)

    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize()
    ctx.timing(True)                  # before the capture: the graph carries the timer event nodes
    ctx.timing_read(A.K_TET_MAP, reset=True)
    graph = None
    if not args.no_graph:
        ctx.graph_begin(stream)
        step()
        graph = ctx.graph_end(stream)
        ctx.graph_launch(graph, stream)       # untimed replay (keeps the captured timer records)
        torch.cuda.synchronize()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    mp_tot, mp_n = 0.0, 0
    dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local_rank) as clk:
        for k in range(args.steps):
            with torch.cuda.stream(stream):
                flush.zero_()
            evs[k][0].record(stream)
            if graph is None:
                step()
            else:
                ctx.graph_launch(graph, stream)
            evs[k][1].record(stream)
            evs[k][1].synchronize()
            ms_, n_ = ctx.timing_read(A.K_TET_MAP)
            mp_tot += ms_
            mp_n += n_
        torch.cuda.synchronize()
    dist.barrier()
    if ctx.error_counts()["peer_timeouts"]:
        raise RuntimeError(f"rank {rank}: peer waits of the position halo abandoned (error word [3])")
    t_ms = sum(a_.elapsed_time(b_) for a_, b_ in evs)
    tt = torch.tensor([t_ms], device=dev, dtype=torch.float64)
    dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    t_ms = float(tt.item())
    peak, peak_src = _peaks()
    map_us = 1e3 * mp_tot / max(mp_n, 1)
    b_map = bytes_map(R.fem.nt, R.fem.nv, R.fem.ne, 4)
    line = {"metric": METRIC, "value": T_global * args.steps / (t_ms / 1e3), "unit": "tets/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_ms / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (seeded metaball blob of Kuhn cubes, twist displacement)",
            "config": {"workload": f"C3 (BASELINE configs[2]): StVK force+stiffness map, blob of {T_global} tets "
                                   f"(n={n}), fp32, split over {world} GPU(s) by the O4 owner maps with ghost tets; "
                                   f"a step = the u halo ({args.dist_halo}) + the map of the local tets",
                       "tets": T_global, "transport": transport,
                       "parallelism": f"domain decomposition x{world} ({args.dist_halo} position halo)",
                       "l2": "flushed between timed steps (256 MiB write)"},
            "roofline": {"kernel": "k_tet_map_seg (local tets of this rank)", "bound": "hbm",
                         "achieved": b_map / (map_us * 1e-6) / 1e9, "peak": peak, "unit": "GB/s",
                         "frac": b_map / (map_us * 1e-6) / 1e9 / peak, "peak_source": peak_src, "traffic": None,
                         "algorithmic_bytes_per_launch": b_map, "avg_launch_us": map_us, "rank": rank},
            "gpu_launches": None, "clocks": clk.summary(),
            "e2e": {"value": T_global * args.steps / (t_ms / 1e3), "unit": "tets/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0, "note": "map-only line: the state stays on the devices"},
            "components": {"local_tets": int(R.fem.nt), "owned_verts": int(part["n_owned"]),
                           "partition_setup_s": t_part}}
    if rank == 0:
        emit(line)
    if halo is not None:
        dist.barrier()
        halo.close()
    ctx.close()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-graph", action="store_true", help="launch kernels eagerly instead of a CUDA graph")
    ap.add_argument("--no-c2", action="store_true", help="skip the C2 (1M-tet) component measurement")
    ap.add_argument("--map-only", action="store_true",
                    help="BASELINE configs[2]: the fp32 StVK map on the 1e7-tet blob with the position halo "
                         "(domain decomposition; with one rank add --dist)")
    ap.add_argument("--dist-cg", default="peer", choices=["peer", "single", "saad"],
                    help="PCG driver of the multi-GPU path (peer: ONE fused kernel per solve, halos and scalar "
                         "sums over peer memory; single: per-iteration phases with one fused NCCL allreduce; "
                         "saad: two allreduces per iteration)")
    ap.add_argument("--dist-halo", default="peer", choices=["peer", "nccl"],
                    help="position halo of the --map-only multi-GPU path (peer: one push kernel over peer memory)")
    ap.add_argument("--dist", action="store_true",
                    help="run the multi-GPU (domain decomposition) path even with one rank (smoke test)")
    args = ap.parse_args()
    _claim_stdout()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    use_dist = world > 1 or args.dist
    if use_dist:
        import torch
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29517")
        os.environ.setdefault("RANK", str(rank))
        os.environ.setdefault("WORLD_SIZE", str(world))
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    try:
        if use_dist and args.map_only:
            run_dist_map(args, rank, world, local_rank)
        elif use_dist:
            run_dist(args, rank, world, local_rank)
        else:
            run_ours(args, rank, world, local_rank)
    finally:
        if use_dist:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
