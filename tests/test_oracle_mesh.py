"""Pins for oracle O1-O5 (connectivity, renumbering, partition, rest data).

Every expected value here comes from SPEC/PAPER examples (tests/golden), closed
forms, or brute force on tiny inputs -- never from the oracle itself.
"""
import itertools
import json
import os

import numpy as np
import pytest

import oracle
from synth import mesh as M
from synth import state as S

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def brute_edges(nv, tets):
    """Brute force: set of ordered pairs within a tet plus all self-loops."""
    s = {(v, v) for v in range(nv)}
    for t in tets:
        for a in t:
            for b in t:
                s.add((int(a), int(b)))
    return sorted(s)


def test_spec_edge_counts():
    g = _gold("spec_examples.json")
    for key in ("tetmesh_one_tet", "tetmesh_two_tets"):
        tets = np.array(g[key]["tets"])
        nv = tets.max() + 1
        tail, head, row_ptr, e = oracle.edges(nv, tets)
        assert tail.size == g[key]["n_edges"]


@pytest.mark.parametrize("row", _gold("kuhn_counts.json")["kuhn6"][:4])
def test_kuhn_counts(row):
    X, tets = M.kuhn6(row["n"])
    m = oracle.Mesh(X, tets)
    assert (m.nv, m.nt, m.ne) == (row["V"], row["T"], row["E"])
    T, V, U, E = M.kuhn_counts(row["n"])
    assert (T, V, E) == (row["T"], row["V"], row["E"])
    # closed form E = 2U + V
    assert m.ne == 2 * row["U"] + row["V"]


@pytest.mark.parametrize("row", _gold("kuhn_counts.json")["alt5"])
def test_alt5_counts(row):
    X, tets = M.alt5(row["n"])
    m = oracle.Mesh(X, tets)
    assert (m.nv, m.nt, m.ne) == (row["V"], row["T"], row["E"])


def test_kuhn_euler_and_degrees():
    X, tets = M.kuhn6(4)
    m = oracle.Mesh(X, tets)
    faces = set()
    for t in m.tets:
        for f in itertools.combinations(sorted(t), 3):
            faces.add(f)
    U = (m.ne - m.nv) // 2
    assert len(faces) == 864
    assert m.nv - U + len(faces) - m.nt == 1
    assert np.max(np.diff(m.row_ptr)) == 15
    assert np.max(np.bincount(m.tets.ravel())) == 24


@pytest.mark.parametrize("gen", [M.single_tet, M.two_tets, lambda: M.kuhn6(2), lambda: M.alt5(2)])
def test_edges_brute_force_and_e_matrix(gen):
    X, tets = gen()
    m = oracle.Mesh(X, tets)
    assert list(zip(m.tail.tolist(), m.head.tolist())) == brute_edges(m.nv, m.tets)
    # CSR: row_ptr ranges partition [0,E) and group by tail
    for v in range(m.nv):
        assert np.all(m.tail[m.row_ptr[v]:m.row_ptr[v + 1]] == v)
    assert m.row_ptr[0] == 0 and m.row_ptr[-1] == m.ne
    # e[i][j]: tail = v[i], head = v[j]
    for t in range(m.nt):
        for i in range(4):
            for j in range(4):
                r = m.e[t, i, j]
                assert m.tail[r] == m.tets[t, i] and m.head[r] == m.tets[t, j]


def test_orientation_swap_and_degenerate():
    X, tets = M.single_tet()
    flipped = tets[:, [0, 1, 3, 2]]
    t2, swaps = oracle.orient(X, flipped)
    assert swaps == 1 and np.array_equal(t2, tets)
    Xd = X.copy()
    Xd[3] = [0.5, 0.5, 0.0]            # coplanar -> degenerate
    with pytest.raises(ValueError):
        oracle.orient(Xd, tets)


def test_morton_octant_blocks_on_lattice():
    """Z-order on a 4x4x4 lattice visits each 2x2x2 octant contiguously and the
    first 8 codes are the unit cube in x-fastest order (bit x at 0, y at 1, z at 2)."""
    X, tets = M.kuhn6(3)            # 4x4x4 lattice, coords i/3
    new_of_old, tet_src, tets_new = oracle.renumber(X, tets)
    order = np.argsort(new_of_old)  # old id at each new position
    ijk = np.rint(X[order] * 3).astype(int)
    first8 = [tuple(r) for r in ijk[:8]]
    assert first8 == [(0, 0, 0), (1, 0, 0), (0, 1, 0), (1, 1, 0), (0, 0, 1), (1, 0, 1), (0, 1, 1), (1, 1, 1)]
    for b in range(8):
        blk = ijk[8 * b:8 * b + 8] // 2
        assert np.all(blk == blk[0])
    codes = oracle.morton(X)[order]
    assert np.all(np.diff(codes.astype(np.float64)) >= 0)


def test_renumber_permutation_and_tet_order():
    X, tets = M.kuhn6(3)
    X, tets = M.permute_vertices(X, tets, seed=2)
    new_of_old, tet_src, tets_new = oracle.renumber(X, tets)
    assert np.array_equal(np.sort(new_of_old), np.arange(X.shape[0]))
    assert np.array_equal(np.sort(tet_src), np.arange(tets.shape[0]))
    assert np.array_equal(tets_new, new_of_old[tets[tet_src]])
    keys = np.sort(tets_new, axis=1)
    for a, b in zip(keys[:-1], keys[1:]):
        assert tuple(a) < tuple(b)
    # orientation kept: renumbered mesh needs no swaps
    Xn = np.empty_like(X)
    Xn[new_of_old] = X
    _, swaps = oracle.orient(Xn, tets_new)
    assert swaps == 0


def test_renumber_stable_on_duplicates():
    X = np.zeros((5, 3))                  # all positions equal: identity order
    tets = np.array([[0, 1, 2, 3]])
    new_of_old, _, _ = oracle.renumber(X, tets)
    assert np.array_equal(new_of_old, np.arange(5))


@pytest.mark.parametrize("P", [1, 2, 3, 8])
def test_partition_invariants(P):
    X, tets = M.kuhn6(4)
    m = oracle.Mesh(X, tets)
    part = oracle.partition(m.nv, m.tets, P, tail=m.tail)
    ot, ov = part["owner_t"], part["owner_v"]
    counts = np.bincount(ot, minlength=P)
    assert counts.max() - counts.min() <= 1                 # balanced tets
    assert np.bincount(ov, minlength=P).sum() == m.nv       # every vertex once
    for p in range(P):
        owned = set(np.nonzero(ov == p)[0].tolist())
        gh = set(part["ghosts"][p].tolist())
        assert not (owned & gh)
        assert list(part["ghosts"][p]) == sorted(gh)
        # every vertex of p's tets is owned or ghost on p
        used = set(m.tets[ot == p].ravel().tolist())
        assert used <= owned | gh
        for q in range(P):
            s = part["send"][p][q]
            if p != q:
                assert set(s.tolist()) == set(part["ghosts"][q].tolist()) & owned
                assert list(s) == sorted(s)
            else:
                assert len(s) == 0
    # a vertex is owned by the part of its lowest incident tet
    for v in range(m.nv):
        t0 = np.nonzero(np.any(m.tets == v, axis=1))[0].min()
        assert ov[v] == ot[t0]


def test_rest_volume_and_mass():
    for gen in (lambda: M.kuhn6(4), lambda: M.alt5(3)):
        X, tets = gen()
        m = oracle.Mesh(X, tets, rho=7.0)
        assert abs(m.W.sum() - 1.0) < 1e-13            # unit cube volume
        assert abs(m.mass.sum() - 7.0) < 1e-12         # rho * volume
        assert np.all(m.W > 0)
        # Dminv is the inverse of Dm
        for t in range(0, m.nt, 37):
            Dm = (X[m.tets[t, 1:]] - X[m.tets[t, 0]]).T
            assert np.allclose(m.Dminv[t] @ Dm, np.eye(3), atol=1e-12)


def test_morton_quantisation_closed_form():
    """O3 quantisation q = min(2^21-1, floor((x-lo)/(hi-lo) 2^21)), x bit at 3b:
    x = 0.5 -> q_x = 2^20 -> code 2^60; x = 1 -> q_x = 2^21-1 -> sum_b 2^(3b)."""
    X = np.array([[0.0, 0.0, 0.0], [0.5, 0.0, 0.0], [1.0, 0.0, 0.0], [0.0, 1.0, 1.0]])
    c = oracle.morton(X)
    assert int(c[0]) == 0
    assert int(c[1]) == 1 << 60
    assert int(c[2]) == sum(1 << (3 * b) for b in range(21))
    assert int(c[3]) == sum((1 << (3 * b + 1)) | (1 << (3 * b + 2)) for b in range(21))


def test_blob_generator_is_valid():
    """C3 blob recipe: positive volumes after jitter (no swaps needed), target
    size reached with the smallest n, every vertex used."""
    X, tets, n = M.blob(20_000)
    assert 6 * (tets.shape[0] // 6) == tets.shape[0] and tets.shape[0] >= 20_000
    assert n == M.blob_n_for(20_000)
    m = oracle.Mesh(X, tets)
    assert m.swaps == 0 and np.all(m.W > 0)
    assert np.all(np.bincount(m.tets.ravel(), minlength=m.nv) > 0)


@pytest.mark.parametrize("P", [1, 2, 3, 5])
def test_partition_overlap_invariants(P):
    """O4, overlapping decomposition: p's local tets are exactly the tets with
    an owned vertex, so every tet incident to an owned vertex -- every block
    of every owned edge row -- is local (no reverse add needed).  Ghosts are
    characterised independently through the edge relation (O2): the
    neighbours of owned vertices that p does not own."""
    X, tets = M.kuhn6(4)
    X, tets = M.permute_vertices(X, tets, 3)
    m = oracle.Mesh(X, tets)
    part = oracle.partition(m.nv, m.tets, P, mode="overlap")
    own = oracle.partition(m.nv, m.tets, P)
    ov = part["owner_v"]
    assert np.array_equal(ov, own["owner_v"]) and np.array_equal(part["owner_t"], own["owner_t"])
    for p in range(P):
        owned = np.nonzero(ov == p)[0]
        lt = part["ltets"][p]
        incident = np.nonzero(np.isin(m.tets, owned).any(axis=1))[0]
        assert np.array_equal(lt, incident)
        nb = set()
        for v in owned:                                  # edge-relation neighbours of owned vertices
            nb |= set(m.head[m.row_ptr[v]:m.row_ptr[v + 1]].tolist())
        assert part["ghosts"][p].tolist() == sorted(nb - set(owned.tolist()))
        assert np.array_equal(part["local"][p][:owned.size], owned)
        for q in range(P):
            s = part["send"][p][q]
            assert list(s) == sorted(s)
            if p != q:
                assert set(s.tolist()) == set(part["ghosts"][q].tolist()) & set(owned.tolist())
    # a tet is local exactly on the parts owning one of its vertices (so an
    # owned tet whose vertices all belong to lower parts is not local on its
    # owner: owner_v is the owner of the vertex's lowest tet)
    for t in range(m.nt):
        on = {p for p in range(P) if t in set(part["ltets"][p].tolist())}
        assert on == set(ov[m.tets[t]].tolist())
    if P == 1:
        assert part["ghosts"][0].size == 0 and part["ltets"][0].size == m.nt


@pytest.mark.parametrize("P", [2, 3])
def test_partition_reverse_lists_carry_every_foreign_partial_row(P):
    """oracle.partition_reverse pinned by the reverse-add semantics, with the
    oracle's element map (its own edge relation) instead of the pair
    enumeration: map each rank's computing tets alone; every force row and
    every stiffness row with a nonzero partial sum whose vertex / tail
    another rank q owns must be in the rank's list for q, and every listed
    row must be one its tets touch; every tet has exactly one computing rank,
    the owner of its lowest vertex, and the ranks' partial sums add up to the
    single-domain map."""
    X, tets = M.kuhn6(4)
    X, tets = M.permute_vertices(X, tets, 2)
    m = oracle.Mesh(X, tets)
    u = S.stretch_noise_u(X, 4, 1)
    mu, lam = S.materials(m.nt, 2e5, 0.3)
    key = np.random.default_rng(3).permutation(m.nv)         # any shared global numbering
    rv = oracle.partition_reverse(m.nv, m.tets, P, key=key)
    ov, comp = rv["owner_v"], rv["comp"]
    lo = m.tets[np.arange(m.nt), np.argmin(key[m.tets], axis=1)]
    assert np.array_equal(comp, ov[lo])
    f_all, K_all, _, _ = oracle.element_map("nh", m.X, u, m.tets, m.Dminv, m.W, mu, lam, e=m.e, ne=m.ne)
    f_sum, K_sum = np.zeros_like(f_all), np.zeros_like(K_all)
    for r in range(P):
        sel = comp == r
        f_r, K_r, _, _ = oracle.element_map("nh", m.X, u, m.tets[sel], m.Dminv[sel], m.W[sel], mu[sel], lam[sel],
                                            e=m.e[sel], ne=m.ne)
        f_sum += f_r
        K_sum += K_r
        touched_v = np.unique(m.tets[sel].ravel())
        for q in range(P):
            if q == r:
                continue
            fv = rv["fsend"][r][q]
            nz_v = np.nonzero(np.abs(f_r).sum(axis=1) > 0)[0]
            want_v = np.intersect1d(touched_v, np.nonzero(ov == q)[0])
            assert np.array_equal(np.sort(fv), want_v)            # the touched vertices q owns
            assert np.array_equal(key[fv], np.sort(key[fv]))      # in key order
            assert set(nz_v[ov[nz_v] == q]) <= set(fv.tolist())   # every nonzero partial force row
            rows = {(int(m.tail[e]), int(m.head[e])) for e in range(m.ne)
                    if ov[m.tail[e]] == q and np.abs(K_r[e]).sum() > 0}
            listed = {tuple(x) for x in rv["ksend"][r][q].tolist()}
            assert rows <= listed                                 # every nonzero partial stiffness row
            assert all(ov[a] == q for a, _ in listed)
            kl = [(key[a], key[b]) for a, b in rv["ksend"][r][q].tolist()]
            assert kl == sorted(kl) and len(set(kl)) == len(kl)
    assert np.allclose(f_sum, f_all, rtol=0, atol=1e-9 * np.abs(f_all).max())
    assert np.allclose(K_sum, K_all, rtol=0, atol=1e-9 * np.abs(K_all).max())
