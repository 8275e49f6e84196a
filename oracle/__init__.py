"""Sequential fp64 CPU ORACLE for the Ebb tet-FEM hot path -- TEST INFRASTRUCTURE.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and ``--impl reference``) may import this package.  The
product path (``paper_1506_07577_b200``) never imports it and shares no code
with it; the only shared module is ``synth`` (seeded inputs, no method
arithmetic).

The arithmetic lives in ``ebb_oracle.c`` (plain C, ``-O2 -ffp-contract=off``),
one function per step O1..O10 of SURVEY.md §8(c) / DESIGN.md §3; this module
is ctypes marshalling plus O4 (partition bookkeeping, plain numpy) and the
composition of steps in the paper's order.

Parity status of every function is listed in DESIGN.md §4; every function
is pinned (the multi-step trajectory since late round 2: the closed-form
free fall over 10 implicit steps and the energy dissipation of converged
backward Euler, tests/test_oracle_solver.py).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "ebb_oracle.c")
_LIB = os.path.join(_HERE, "libebb_oracle.so")

STVK, NH = 0, 1
MODELS = {"stvk": STVK, "nh": NH}


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (no FMA contraction, no fast-math)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-std=c11",
                               "-fPIC", "-shared", "-o", _LIB, _SRC, "-lm"])
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        P = C.c_void_p
        I = C.c_int64
        D = C.c_double
        sig = {
            "orc_orient": (I, [I, P, I, P]),
            "orc_edges": (I, [I, I, P, I, P, P, P, P]),
            "orc_morton": (None, [I, P, P]),
            "orc_renumber": (None, [I, P, I, P, P, P, P]),
            "orc_rest": (I, [I, P, I, P, D, P, P, P]),
            "orc_element_map": (I, [C.c_int, I, P, P, I, P, P, P, P, P, P, I, P, P, P]),
            "orc_edge_matvec": (None, [I, P, P, P, P, P]),
            "orc_dot": (D, [I, P, P]),
            "orc_explicit_update": (None, [I, P, P, P, P, D, P, P]),
            "orc_implicit_assemble": (None, [I, P, P, P, P, P, P, D, D, D, P, P, P]),
            "orc_consistent_mass": (None, [I, P, P, D, I, P]),
            "orc_newton_rhs": (None, [I, P, P, P, P, P, P, P, D, D, D, P, P]),
            "orc_spring_init_len": (None, [I, P, P, P, P]),
            "orc_spring_forces": (None, [I, P, P, P, P, D, P]),
            "orc_spring_apply": (None, [I, P, D, P, P, P]),
            "orc_kinetic_energy": (D, [I, P, P]),
            "orc_grid2_stencil": (None, [I, I, C.c_int, P, P, C.c_int, P, P]),
            "orc_grid2_point_locate": (None, [I, I, I, P, P]),
            "orc_grid2_particle_vel": (None, [I, I, C.c_int, P, I, P, P, P]),
            "orc_implicit_assemble_consistent": (None, [I, P, P, P, P, P, P, D, D, D, P, P, P]),
            "orc_pcg": (C.c_int, [I, P, P, P, P, P, C.c_int, P, P]),
            "orc_implicit_update": (None, [I, P, D, P, P]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(_lib, name)
            fn.restype = res
            fn.argtypes = args
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _i64(a):
    return np.ascontiguousarray(a, dtype=np.int64)


# ---------------------------------------------------------------- O1
def orient(X, tets):
    """O1: returns (oriented tets copy, number of swaps); raises on degenerate."""
    t = _i64(tets).copy()
    r = lib().orc_orient(X.shape[0], _p(_f64(X)), t.shape[0], _p(t))
    if r < 0:
        raise ValueError(f"degenerate tet {-r - 1}")
    return t, int(r)


# ---------------------------------------------------------------- O2
def edges(nv, tets):
    """O2: (tail, head, row_ptr, e[T,4,4]) of the edge relation grouped by tail."""
    t = _i64(tets)
    nt = t.shape[0]
    cap = 16 * nt + nv
    tail = np.empty(cap, np.int64)
    head = np.empty(cap, np.int64)
    row_ptr = np.empty(nv + 1, np.int64)
    e = np.empty((nt, 4, 4), np.int64)
    E = lib().orc_edges(nv, nt, _p(t), cap, _p(tail), _p(head), _p(row_ptr), _p(e))
    assert E >= 0
    return tail[:E].copy(), head[:E].copy(), row_ptr, e


# ---------------------------------------------------------------- O3
def morton(X):
    c = np.empty(X.shape[0], np.uint64)
    lib().orc_morton(X.shape[0], _p(_f64(X)), _p(c))
    return c


def renumber(X, tets):
    """O3: (new_of_old[V], tet_src[T], tets_new[T,4])."""
    X = _f64(X)
    t = _i64(tets)
    nv, nt = X.shape[0], t.shape[0]
    new_of_old = np.empty(nv, np.int64)
    tet_src = np.empty(nt, np.int64)
    tets_out = np.empty((nt, 4), np.int64)
    lib().orc_renumber(nv, _p(X), nt, _p(t), _p(new_of_old), _p(tet_src), _p(tets_out))
    return new_of_old, tet_src, tets_out


# ---------------------------------------------------------------- O4
def partition(nv, tets, P, tail=None, mode="own"):
    """O4 tet-first SFC partition into P parts (plain numpy bookkeeping).

    owner_t(t) = floor(t P / T); owner_v(v) = owner_t(min{t : v in t}) or
    floor(v P / V) for isolated vertices.  Local tets of part p:
      mode="own"      the tets p owns (owner_t == p) -- SURVEY §8(e) O4;
      mode="overlap"  every tet with a vertex owned by p (the ghost-tet
                      decomposition: every row of an owned
                      vertex is then complete on p without a reverse add).
    ghosts of p = vertices of p's local tets not owned by p (ascending);
    send[p][q] = vertices owned by p that are ghosts on q (ascending); edge
    rows owned by owner_v(tail); local numbering = owned ascending then ghosts
    ascending; ltets[p] = p's local tets (ascending).
    """
    if mode not in ("own", "overlap"):
        raise ValueError(mode)
    tets = _i64(tets)
    T = tets.shape[0]
    owner_t = (np.arange(T, dtype=np.int64) * P) // max(T, 1)
    first = np.full(nv, T, dtype=np.int64)
    for t in range(T):                      # plain loop: min tet per vertex
        for v in tets[t]:
            if t < first[v]:
                first[v] = t
    owner_v = np.empty(nv, np.int64)
    iso = first == T
    owner_v[~iso] = owner_t[first[~iso]]
    owner_v[iso] = (np.nonzero(iso)[0] * P) // max(nv, 1)
    ghosts, local, ltets = [], [], []
    for p in range(P):
        if mode == "own":
            lt = np.nonzero(owner_t == p)[0]
        else:
            lt = np.array([t for t in range(T) if any(owner_v[v] == p for v in tets[t])], dtype=np.int64)
        vs = np.unique(tets[lt].ravel())
        g = vs[owner_v[vs] != p]
        ghosts.append(g)
        ltets.append(lt)
        local.append(np.concatenate([np.nonzero(owner_v == p)[0], g]))
    send = [[None] * P for _ in range(P)]
    for p in range(P):
        for q in range(P):
            gq = ghosts[q]
            send[p][q] = gq[owner_v[gq] == p] if p != q else np.zeros(0, np.int64)
    out = dict(owner_t=owner_t, owner_v=owner_v, ghosts=ghosts, send=send, local=local, ltets=ltets)
    if tail is not None:
        out["owner_e"] = owner_v[_i64(tail)]
    return out


def partition_reverse(nv, tets, P, key=None):
    """O4, reverse-add reading (SURVEY §8(e) "halo exchange ...
    of the partial force sums"): every tet is computed by ONE rank, the
    owner (O4 owner_v) of its vertex of lowest key (key = a global vertex
    numbering every rank shares, default the vertex id); a rank sends the
    partial rows whose tail it does not own to the tail's owner.  Plain loops:
      comp[t]        computing rank of tet t
      fsend[r][q]    the vertices owned by q that r's tets touch (the force
                     rows r adds into q), ascending by key
      ksend[r][q]    (tail, head) of the edge rows -- every ordered pair of
                     vertices of one of r's tets, self pairs included --
                     whose tail q owns, ascending by (key[tail], key[head])
    r receives from q exactly what q sends to r (frecv[r][q] = fsend[q][r])."""
    tets = _i64(tets)
    key = np.arange(nv, dtype=np.int64) if key is None else _i64(key)
    owner_v = partition(nv, tets, P, mode="overlap")["owner_v"]
    T = tets.shape[0]
    comp = np.empty(T, np.int64)
    fs = [[set() for _ in range(P)] for _ in range(P)]
    ks = [[set() for _ in range(P)] for _ in range(P)]
    for t in range(T):
        lo = min(tets[t], key=lambda v: key[v])
        r = int(owner_v[lo])
        comp[t] = r
        for a in tets[t]:
            q = int(owner_v[a])
            if q == r:
                continue
            fs[r][q].add(int(a))
            for b in tets[t]:
                ks[r][q].add((int(a), int(b)))
    fsend = [[np.array(sorted(fs[r][q], key=lambda v: key[v]), np.int64) for q in range(P)] for r in range(P)]
    ksend = [[np.array(sorted(ks[r][q], key=lambda e: (key[e[0]], key[e[1]])), np.int64).reshape(-1, 2)
              for q in range(P)] for r in range(P)]
    return dict(owner_v=owner_v, comp=comp, fsend=fsend, ksend=ksend)


# ---------------------------------------------------------------- O5
def rest(X, tets, rho):
    """O5: (Dminv[T,3,3], W[T], mass[V]); raises if some W <= 0."""
    X = _f64(X)
    t = _i64(tets)
    nt = t.shape[0]
    Dminv = np.empty((nt, 3, 3))
    W = np.empty(nt)
    m = np.empty(X.shape[0])
    bad = lib().orc_rest(X.shape[0], _p(X), nt, _p(t), rho, _p(Dminv), _p(W), _p(m))
    if bad:
        raise ValueError(f"{bad} tets with W <= 0")
    return Dminv, W, m


# ---------------------------------------------------------------- O6/O7
def element_map(model, X, u, tets, Dminv, W, mu, lam, e=None, ne=0, want_K=True):
    """O6+O7: (f[V,3], K[E,3,3] or None, energy, n_inverted)."""
    model = MODELS.get(model, model)
    X = _f64(X)
    u = _f64(u)
    t = _i64(tets)
    nv, nt = X.shape[0], t.shape[0]
    f = np.empty((nv, 3))
    K = np.empty((ne, 3, 3)) if want_K else None
    en = C.c_double(0.0)
    inv = lib().orc_element_map(model, nv, _p(X), _p(u), nt, _p(t), _p(_f64(Dminv)), _p(_f64(W)),
                                _p(_f64(mu)), _p(_f64(lam)), _p(_i64(e)) if want_K else None, ne,
                                _p(f), _p(K), C.byref(en))
    return f, K, en.value, int(inv)


def edge_matvec(row_ptr, head, A, p):
    nv = row_ptr.shape[0] - 1
    q = np.empty((nv, 3))
    lib().orc_edge_matvec(nv, _p(_i64(row_ptr)), _p(_i64(head)), _p(_f64(A)), _p(_f64(p)), _p(q))
    return q


def dot(a, b):
    a = _f64(a).ravel()
    b = _f64(b).ravel()
    return lib().orc_dot(a.size, _p(a), _p(b))


# ---------------------------------------------------------------- O8
def explicit_update(f, mass, free, g, h, u, v):
    u = _f64(u).copy()
    v = _f64(v).copy()
    g = _f64(g)
    lib().orc_explicit_update(mass.shape[0], _p(_f64(f)), _p(_f64(mass)),
                              _p(np.ascontiguousarray(free, np.uint8)) if free is not None else None,
                              _p(g), h, _p(u), _p(v))
    return u, v


# ---------------------------------------------------------------- O9
def implicit_assemble(row_ptr, head, K, mass, f, vel, h, alpha=0.0, beta=0.0, g=(0.0, -9.81, 0.0)):
    nv = row_ptr.shape[0] - 1
    A = np.empty_like(_f64(K))
    b = np.empty((nv, 3))
    lib().orc_implicit_assemble(nv, _p(_i64(row_ptr)), _p(_i64(head)), _p(_f64(K)), _p(_f64(mass)),
                                _p(_f64(f)), _p(_f64(vel)), h, alpha, beta, _p(_f64(np.asarray(g))),
                                _p(A), _p(b))
    return A, b


def consistent_mass(tets_e, W, rho, ne):
    """Consistent (Galerkin) mass on the edge relation: mass_e[E] with
    M_r = mass_e[r] I_3, mass_e[e[i][j]] += rho W (1 + d_ij) / 20."""
    e = _i64(tets_e).reshape(-1, 16)
    m = np.empty(ne)
    lib().orc_consistent_mass(e.shape[0], _p(e), _p(_f64(W)), rho, ne, _p(m))
    return m


def implicit_assemble_consistent(row_ptr, head, K, mass_e, f, vel, h, alpha=0.0, beta=0.0,
                                 g=(0.0, -9.81, 0.0)):
    """O9 with the consistent edge mass (M v, M g as edge query-loops)."""
    nv = row_ptr.shape[0] - 1
    A = np.empty_like(_f64(K))
    b = np.empty((nv, 3))
    lib().orc_implicit_assemble_consistent(nv, _p(_i64(row_ptr)), _p(_i64(head)), _p(_f64(K)),
                                           _p(_f64(mass_e)), _p(_f64(f)), _p(_f64(vel)), h, alpha, beta,
                                           _p(_f64(np.asarray(g))), _p(A), _p(b))
    return A, b


# ---------------------------------------------------------------- O10
def pcg(row_ptr, head, A, b, free, iters):
    """O10: (x[V,3], rho_hist[iters+1], not_spd)."""
    nv = row_ptr.shape[0] - 1
    x = np.empty((nv, 3))
    hist = np.empty(iters + 1)
    ns = lib().orc_pcg(nv, _p(_i64(row_ptr)), _p(_i64(head)), _p(_f64(A)), _p(_f64(b)),
                       _p(np.ascontiguousarray(free, np.uint8)) if free is not None else None,
                       iters, _p(x), _p(hist))
    return x, hist, bool(ns)


def implicit_update(dv, h, u, v):
    u = _f64(u).copy()
    v = _f64(v).copy()
    lib().orc_implicit_update(u.shape[0], _p(_f64(dv)), h, _p(u), _p(v))
    return u, v


# ---------------------------------------------------------------- composed steps
class Mesh:
    """Oracle-side mesh: O1 orientation, O2 edges, O5 rest data."""

    def __init__(self, X, tets, rho=1e3, renumbered=False):
        self.X = _f64(X)
        self.tets, self.swaps = orient(self.X, tets)
        self.nv, self.nt = self.X.shape[0], self.tets.shape[0]
        self.tail, self.head, self.row_ptr, self.e = edges(self.nv, self.tets)
        self.ne = self.tail.shape[0]
        self.rho = rho
        self.Dminv, self.W, self.mass = rest(self.X, self.tets, rho)


def explicit_step(mesh, model, u, v, mu, lam, free, h, g=(0.0, -9.81, 0.0)):
    """O8: force-only map then the Fig. 2 update."""
    f, _, en, inv = element_map(model, mesh.X, u, mesh.tets, mesh.Dminv, mesh.W, mu, lam, want_K=False)
    u2, v2 = explicit_update(f, mesh.mass, free, np.asarray(g), h, u, v)
    return u2, v2, f, en


def lumped_as_edges(mesh):
    """The lumped vertex mass as an edge-row mass (self rows only)."""
    me = np.zeros(mesh.ne)
    me[mesh.tail == mesh.head] = mesh.mass[mesh.tail[mesh.tail == mesh.head]]
    return me


def newton_rhs(row_ptr, head, K, mass_e, f, w, v0, h, alpha=0.0, beta=0.0, g=(0.0, -9.81, 0.0)):
    """b = h (f + M g - D w) + M (v_n - w): the Newton right-hand side."""
    nv = row_ptr.shape[0] - 1
    b = np.empty((nv, 3))
    lib().orc_newton_rhs(nv, _p(_i64(row_ptr)), _p(_i64(head)), _p(_f64(K)), _p(_f64(mass_e)), _p(_f64(f)),
                         _p(_f64(w)), _p(_f64(v0)), h, alpha, beta, _p(_f64(np.asarray(g))), _p(b))
    return b


def newton_step(mesh, model, u, v, mu, lam, free, h, iters=50, newton=2, alpha=0.0, beta=0.0,
                g=(0.0, -9.81, 0.0), mass="lumped"):
    """Backward Euler with `newton` Newton iterations: the first is the
    one-linearisation step (implicit_step), each later one maps f, K at
    x_k = u_n + h w_k, solves (M + hD + h^2 K) dw = b (newton_rhs) with
    `iters` PCG iterations, then w += dw, u += h dw."""
    out = implicit_step(mesh, model, u, v, mu, lam, free, h, iters, alpha, beta, g, mass)
    me = consistent_mass(mesh.e, mesh.W, mesh.rho, mesh.ne) if mass == "consistent" else lumped_as_edges(mesh)
    x, w = out["u"], out["v"]
    v0 = _f64(v)
    for _ in range(newton - 1):
        f, K, en, inv = element_map(model, mesh.X, x, mesh.tets, mesh.Dminv, mesh.W, mu, lam,
                                    e=mesh.e, ne=mesh.ne)
        if mass == "consistent":
            A, _b = implicit_assemble_consistent(mesh.row_ptr, mesh.head, K, me, f, w, h, alpha, beta, g)
        else:
            A, _b = implicit_assemble(mesh.row_ptr, mesh.head, K, mesh.mass, f, w, h, alpha, beta, g)
        b = newton_rhs(mesh.row_ptr, mesh.head, K, me, f, w, v0, h, alpha, beta, g)
        dw, hist, ns = pcg(mesh.row_ptr, mesh.head, A, b, free, iters)
        w = w + dw
        x = x + h * dw
        out = dict(out, u=x, v=w, f=f, K=K, A=A, b=b, dv=dw, rho=hist, not_spd=ns or out["not_spd"])
    return out


def implicit_step(mesh, model, u, v, mu, lam, free, h, iters=50, alpha=0.0, beta=0.0,
                  g=(0.0, -9.81, 0.0), mass="lumped"):
    """O9+O10: map (f, K), assemble, PCG(iters), v += dv, u += h v.
    mass="consistent": the edge-relation Galerkin mass (density mesh.rho)."""
    f, K, en, inv = element_map(model, mesh.X, u, mesh.tets, mesh.Dminv, mesh.W, mu, lam,
                                e=mesh.e, ne=mesh.ne)
    if mass == "consistent":
        me = consistent_mass(mesh.e, mesh.W, mesh.rho, mesh.ne)
        A, b = implicit_assemble_consistent(mesh.row_ptr, mesh.head, K, me, f, v, h, alpha, beta, g)
    else:
        A, b = implicit_assemble(mesh.row_ptr, mesh.head, K, mesh.mass, f, v, h, alpha, beta, g)
    dv, hist, not_spd = pcg(mesh.row_ptr, mesh.head, A, b, free, iters)
    u2, v2 = implicit_update(dv, h, u, v)
    return dict(u=u2, v=v2, f=f, K=K, A=A, b=b, dv=dv, rho=hist, energy=en,
                inverted=inv, not_spd=not_spd)


# ---------------------------------------------------------------- Fig. 2 spring-mass
def spring_init_len(tail, head, pos):
    """initLen: rest_len[e] = |pos[head] - pos[tail]|."""
    L = np.empty(tail.shape[0])
    lib().orc_spring_init_len(tail.shape[0], _p(_i64(tail)), _p(_i64(head)), _p(_f64(pos)), _p(L))
    return L


def spring_forces(row_ptr, head, q, rest_len, K, force=None):
    """computeInternalForces: force += K sum (rest_len dir - dq)."""
    nv = row_ptr.shape[0] - 1
    f = np.zeros((nv, 3)) if force is None else _f64(force).copy()
    lib().orc_spring_forces(nv, _p(_i64(row_ptr)), _p(_i64(head)), _p(_f64(q)), _p(_f64(rest_len)), K, _p(f))
    return f


def spring_apply(mass, dt, q, qd, force):
    """applyForces: returns (q, qd, force = 0)."""
    q, qd, f = _f64(q).copy(), _f64(qd).copy(), _f64(force).copy()
    lib().orc_spring_apply(q.shape[0], _p(_f64(mass)), dt, _p(q), _p(qd), _p(f))
    return q, qd, f


def kinetic_energy(mass, qd):
    """measureTotalEnergy: sum 0.5 m qd.qd."""
    return lib().orc_kinetic_energy(_f64(mass).shape[0], _p(_f64(mass)), _p(_f64(qd)))


def spring_steps(row_ptr, head, rest_len, mass, K, dt, q, qd, steps):
    """The Fig. 2 loop body `steps` times (force starts at 0)."""
    f = np.zeros_like(_f64(q))
    for _ in range(steps):
        f = spring_forces(row_ptr, head, q, rest_len, K, f)
        q, qd, f = spring_apply(mass, dt, q, qd, f)
    return q, qd


# ---------------------------------------------------------------- regular 2-D grid (Fig. 3)
def grid2_stencil(nx, ny, field, offsets, weights):
    """out[c] = sum_k w_k field[cell(i+dx_k, j+dy_k)] (periodic); field (nx*ny, comps)."""
    f = _f64(field).reshape(nx * ny, -1)
    out = np.empty_like(f)
    off = _i64(np.asarray(offsets)).reshape(-1, 2)
    lib().orc_grid2_stencil(nx, ny, f.shape[1], _p(f), _p(out), off.shape[0], _p(off), _p(_f64(weights)))
    return out


def grid2_point_locate(nx, ny, pos):
    pos = _f64(pos).reshape(-1, 3)
    d = np.empty(pos.shape[0], dtype=np.int64)
    lib().orc_grid2_point_locate(nx, ny, pos.shape[0], _p(pos), _p(d))
    return d


def grid2_particle_vel(nx, ny, cell_vel, pos, dual):
    cv = _f64(cell_vel).reshape(nx * ny, -1)
    pos = _f64(pos).reshape(-1, 3)
    vel = np.empty((pos.shape[0], cv.shape[1]))
    lib().orc_grid2_particle_vel(nx, ny, cv.shape[1], _p(cv), pos.shape[0], _p(pos), _p(_i64(dual)), _p(vel))
    return vel

