"""Seeded synthetic tetrahedral meshes shaped like the paper's FEM workloads.

This module is shared by the oracle (``oracle/``) and the CUDA path
(``paper_1506_07577_b200``).  It holds NO arithmetic of the method: it only
builds lattice connectivity, relabels vertices with seeded permutations and
places vertices.  Element orientation is fixed combinatorially (integer
determinant of lattice offsets), never from floating-point geometry.

Workloads:
  * ``kuhn6(n)``   -- unit cube, n^3 cells, each split into 6 Kuhn/Freudenthal
                      tets (C1: n=4 -> 384 tets; C2: n=55 -> 998,250 tets).
  * ``alt5(n)``    -- 5-tet alternating split (SPEC S:527 lattice; 5-tet cube).
  * ``blob(T)``    -- 4-centre metaball made of Kuhn cubes (C3 "blob").
  * ``single_tet``/``two_tets`` -- SPEC S:369-370 examples.
The paper's own meshes (dragon, hose, turtle, sphere, bunny)
are not available; these stand in with the same element type and degree
structure (<=24 tets and <=15 edge rows per vertex for Kuhn meshes).
"""
from __future__ import annotations

import itertools

import numpy as np


def rng(seed: int) -> np.random.Generator:
    """Counter-based generator (Philox) so any consumer can reproduce inputs."""
    return np.random.Generator(np.random.Philox(seed))


def _orient_lattice(ijk: np.ndarray, tets: np.ndarray) -> np.ndarray:
    """Swap v2,v3 where the integer lattice determinant is negative.

    ``ijk`` are integer lattice coordinates; the determinant of integer
    offsets is exact, so this is a combinatorial orientation, not geometry.
    """
    a = ijk[tets[:, 1]] - ijk[tets[:, 0]]
    b = ijk[tets[:, 2]] - ijk[tets[:, 0]]
    c = ijk[tets[:, 3]] - ijk[tets[:, 0]]
    det = (a[:, 0] * (b[:, 1] * c[:, 2] - b[:, 2] * c[:, 1])
           - a[:, 1] * (b[:, 0] * c[:, 2] - b[:, 2] * c[:, 0])
           + a[:, 2] * (b[:, 0] * c[:, 1] - b[:, 1] * c[:, 0]))
    assert np.all(det != 0), "degenerate lattice tet"
    out = tets.copy()
    neg = det < 0
    out[neg, 2], out[neg, 3] = tets[neg, 3], tets[neg, 2]
    return out


def _lattice(n: int):
    idx = np.arange(n + 1)
    k, j, i = np.meshgrid(idx, idx, idx, indexing="ij")
    ijk = np.stack([i.ravel(), j.ravel(), k.ravel()], axis=1).astype(np.int64)
    return ijk


def _vid(n, i, j, k):
    return i + (n + 1) * (j + (n + 1) * k)


def kuhn6_cells(n: int, cells: np.ndarray) -> np.ndarray:
    """Kuhn split of the given cube corners (C,3) on an (n+1)^3 lattice."""
    ci, cj, ck = cells[:, 0], cells[:, 1], cells[:, 2]
    out = []
    for perm in itertools.permutations(range(3)):
        cur = np.stack([ci, cj, ck], axis=1).copy()
        path = [_vid(n, cur[:, 0], cur[:, 1], cur[:, 2])]
        for ax in perm:
            cur[:, ax] += 1
            path.append(_vid(n, cur[:, 0], cur[:, 1], cur[:, 2]))
        out.append(np.stack(path, axis=1))
    # tets of one cube are consecutive: (C, 6, 4) -> (6C, 4)
    return np.stack(out, axis=1).reshape(-1, 4)


def kuhn6(n: int, L: float = 1.0):
    """(X (V,3) f64, tets (T,4) i64) for n^3 cubes split into 6 tets each."""
    ijk = _lattice(n)
    c = np.arange(n)
    k, j, i = np.meshgrid(c, c, c, indexing="ij")
    cells = np.stack([i.ravel(), j.ravel(), k.ravel()], axis=1)
    tets = _orient_lattice(ijk, kuhn6_cells(n, cells))
    X = ijk.astype(np.float64) * (L / n)
    return X, tets


# 5-tet split of a unit cube; local corner id b = dx + 2 dy + 4 dz.
_ALT5_EVEN = [(0, 1, 2, 4), (3, 1, 2, 7), (5, 1, 4, 7), (6, 2, 4, 7), (1, 2, 4, 7)]
_ALT5_ODD = [(1, 0, 3, 5), (2, 0, 3, 6), (4, 0, 5, 6), (7, 3, 5, 6), (0, 3, 5, 6)]


def alt5(n: int, L: float = 1.0):
    """Alternating 5-tet split (conforming: the split flips with cube parity)."""
    ijk = _lattice(n)
    tl = []
    for ck in range(n):
        for cj in range(n):
            for ci in range(n):
                corner = [_vid(n, ci + (b & 1), cj + ((b >> 1) & 1), ck + ((b >> 2) & 1)) for b in range(8)]
                pat = _ALT5_EVEN if (ci + cj + ck) % 2 == 0 else _ALT5_ODD
                for t in pat:
                    tl.append([corner[b] for b in t])
    tets = _orient_lattice(ijk, np.asarray(tl, dtype=np.int64))
    return ijk.astype(np.float64) * (L / n), tets


def single_tet():
    """One unit right tet (16 edge rows)."""
    X = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1]], dtype=np.float64)
    return X, np.array([[0, 1, 2, 3]], dtype=np.int64)


def two_tets():
    """Tets (0,1,2,3),(1,2,3,4) sharing a face (23 edge rows)."""
    X = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1], [1, 1, 1]], dtype=np.float64)
    ijk = X.astype(np.int64)
    tets = _orient_lattice(ijk, np.array([[0, 1, 2, 3], [1, 2, 3, 4]], dtype=np.int64))
    return X, tets


def permute_vertices(X: np.ndarray, tets: np.ndarray, seed: int):
    """Relabel vertices with a seeded random permutation (input order scrambled)."""
    V = X.shape[0]
    perm = rng(seed).permutation(V)          # new label of old vertex v is inv[v]
    inv = np.empty(V, dtype=np.int64)
    inv[perm] = np.arange(V)
    return X[perm].copy(), inv[tets]


def permute_tets(tets: np.ndarray, seed: int):
    return tets[rng(seed).permutation(tets.shape[0])].copy()


BLOB_CENTRES = np.array([[.35, .40, .45], [.65, .55, .50], [.50, .35, .65], [.45, .65, .35]])
BLOB_RADII = np.array([.25, .22, .22, .20])


def _blob_cells(n: int) -> np.ndarray:
    c = (np.arange(n) + 0.5) / n
    k, j, i = np.meshgrid(np.arange(n), np.arange(n), np.arange(n), indexing="ij")
    p = np.stack([c[i.ravel()], c[j.ravel()], c[k.ravel()]], axis=1)
    phi = np.zeros(p.shape[0])
    for ctr, r in zip(BLOB_CENTRES, BLOB_RADII):
        d2 = np.sum((p - ctr) ** 2, axis=1)
        phi += r * r / np.maximum(d2, 1e-30)
    keep = phi >= 1.0
    return np.stack([i.ravel()[keep], j.ravel()[keep], k.ravel()[keep]], axis=1)


def blob_n_for(target_T: int) -> int:
    """Smallest n with 6 * (#kept cubes) >= target_T.  The kept volume fraction
    is estimated on a 48^3 grid, then n is refined by a local search."""
    frac = _blob_cells(48).shape[0] / 48 ** 3
    n = max(4, int(round((target_T / (6.0 * frac)) ** (1.0 / 3.0))))
    while n > 4 and 6 * _blob_cells(n - 1).shape[0] >= target_T:
        n -= 1
    while 6 * _blob_cells(n).shape[0] < target_T:
        n += 1
    return n


def blob(target_T: int = 10_000_000, n: int | None = None, jitter_seed: int = 3, order_seed: int = 4):
    """C3 blob: Kuhn cubes of a 4-centre metaball, jittered +-0.1/n, random order.

    A jitter of 0.1 cell cannot invert a Kuhn tet (its smallest altitude is
    h/sqrt(2) and each vertex moves at most 0.1*sqrt(3) h), so W>0 holds by
    construction; the oracle asserts it (O1).
    """
    if n is None:
        n = blob_n_for(target_T)
    cells = _blob_cells(n)
    tets = kuhn6_cells(n, cells)
    used = np.unique(tets)
    remap = -np.ones((n + 1) ** 3, dtype=np.int64)
    remap[used] = np.arange(used.size)
    ii = used % (n + 1)
    jj = (used // (n + 1)) % (n + 1)
    kk = used // ((n + 1) * (n + 1))
    ijk = np.stack([ii, jj, kk], axis=1)
    tets = _orient_lattice(ijk, remap[tets])
    X = ijk.astype(np.float64) / n
    X += rng(jitter_seed).uniform(-0.1 / n, 0.1 / n, size=X.shape)
    X, tets = permute_vertices(X, tets, order_seed)
    return X, tets, n


def kuhn_counts(n: int):
    """Closed-form sizes of the Kuhn-6 cube (SURVEY §8 header)."""
    T = 6 * n ** 3
    V = (n + 1) ** 3
    U = 3 * n * (n + 1) ** 2 + 3 * n * n * (n + 1) + n ** 3
    return T, V, U, 2 * U + V
