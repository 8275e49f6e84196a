"""Full-size parity at BASELINE configs[2] (C3): StVK / NH force+stiffness map
on the ~1e7-tet blob, fp32, in the launch configuration the sweep times.
The oracle cannot run the whole map in seconds, so it computes exact rows for
a seeded sample of vertices: the sub-mesh of every tet touching a sampled
vertex reproduces that vertex's force and all of its stiffness rows."""
import numpy as np
import pytest

import oracle
from helpers import rel_l2
from synth import mesh as M
from synth import state as S

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1506_07577_b200 import ebb
    c = ebb.Context(0)
    yield c
    c.close()


@pytest.fixture(scope="module")
def c3():
    X, tets, n = M.blob(10_000_000)
    free = S.fixed_mask(X, n)
    u = S.twist_u(X, n, 6, free=free).astype(np.float32).astype(np.float64)
    mu, lam = S.materials(tets.shape[0], 1e6, 0.3, spread=0.1)
    mu = mu.astype(np.float32).astype(np.float64)
    lam = lam.astype(np.float32).astype(np.float64)
    new_of_old, tet_src, tets_new = oracle.renumber(X, tets)
    return dict(X=X, tets=tets, n=n, free=free, u=u, mu=mu, lam=lam, new_of_old=new_of_old, tet_src=tet_src,
                tets_new=tets_new)


@pytest.mark.parametrize("model", ["stvk", "nh"])
def test_c3_blob_map_sampled_rows(ctx, c3, model):
    from paper_1506_07577_b200.tetfem import TetFEM
    d = c3
    fem = TetFEM(ctx, d["X"], d["tets"], dtype="f32", mu=d["mu"], lam=d["lam"], free=d["free"], u=d["u"],
                 name=f"c3{model}")
    order = np.argsort(d["new_of_old"])
    assert np.array_equal(fem.vert_order(), order)            # a2 bit-exact at 1e7 tets
    assert np.array_equal(fem.tet_order(), d["tet_src"])
    fem.map_forces(model)
    f_gpu = fem.f.read()
    index = fem.index.read().astype(np.int64)
    head = fem.head.read().astype(np.int64)
    K_gpu = fem.K.read().reshape(-1, 3, 3)
    # seeded vertex sample, all their incident tets (stored numbering)
    Xs = d["X"][order]
    tets_s = d["tets_new"]
    rng = M.rng(11)
    sample = np.unique(rng.integers(0, Xs.shape[0], size=400))
    touch = np.isin(tets_s, sample).any(axis=1)
    sub_t = np.nonzero(touch)[0]
    sub_v = np.unique(tets_s[sub_t])
    local = np.searchsorted(sub_v, tets_s[sub_t])
    m = oracle.Mesh(Xs[sub_v], local)
    mu_s, lam_s = d["mu"][d["tet_src"]][sub_t], d["lam"][d["tet_src"]][sub_t]
    f, K, en, inv = oracle.element_map(model, m.X, d["u"][order][sub_v], m.tets, m.Dminv, m.W, mu_s, lam_s,
                                       e=m.e, ne=m.ne)
    li = np.searchsorted(sub_v, sample)
    assert rel_l2(f_gpu[sample], f[li]) <= 1e-5
    got, ref = [], []
    for v, lv in zip(sample, li):
        heads_gpu = head[index[v]:index[v + 1]]
        heads_ora = sub_v[m.head[m.row_ptr[lv]:m.row_ptr[lv + 1]]]
        assert np.array_equal(heads_gpu, heads_ora)           # same edge rows, same order
        got.append(K_gpu[index[v]:index[v + 1]])
        ref.append(K[m.row_ptr[lv]:m.row_ptr[lv + 1]])
    assert rel_l2(np.concatenate(got), np.concatenate(ref)) <= 1e-5
