"""GPU parity of the setup steps a1-a3 and O4 (bit-exact integer maps) through
the C ABI, plus ABI error behaviour."""
import json
import os

import numpy as np
import pytest

import oracle
from helpers import Case, gpu_fem, oracle_renumbered, rel_l2
from synth import mesh as M

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def ctx():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1506_07577_b200 import ebb
    c = ebb.Context(0)
    yield c
    c.close()


def test_key_field_bounds_error(ctx):
    from paper_1506_07577_b200 import ebb
    V = ctx.relation("kb.verts", 3)
    E = ctx.relation("kb.edges", 4)
    with pytest.raises(ebb.EbbError) as ei:
        E.key_field("head", V, (1, 1), [0, 1, 2, 3])       # S:90 example: 3 is out of bounds
    assert ei.value.name == "EBB_E_BOUNDS"
    with pytest.raises(ebb.EbbError) as ei:
        ctx.relation("kb.verts", 5)
    assert ei.value.name == "EBB_E_DUP"
    with pytest.raises(ebb.EbbError) as ei:
        ctx.relation("kb.empty", 0)
    assert ei.value.name == "EBB_E_SIZE"


@pytest.mark.parametrize("key", ["groupby", "groupby_sorted"])
def test_group_by_spec_example(ctx, key):
    from paper_1506_07577_b200 import ebb
    g = json.load(open(os.path.join(GOLD, "spec_examples.json")))[key]
    V = ctx.relation(f"{key}.v", g["n_source"])
    E = ctx.relation(f"{key}.e", len(g["tail"]))
    ids = E.field("orig", "u32", init=np.arange(len(g["tail"]), dtype=np.uint32))
    tail = E.key_field("tail", V, (1, 1), g["tail"])
    idx = E.group_by(tail)
    assert ids.read().tolist() == g["order_old_ids"]
    r = idx.read().tolist()
    assert [[r[i], r[i + 1]] for i in range(g["n_source"])] == g["ranges"]
    with pytest.raises(ebb.EbbError) as ei:
        E.group_by(tail)
    assert ei.value.name == "EBB_E_STATE"


def test_orientation_on_device(ctx):
    X, tets = M.kuhn6(3)
    flip = tets.copy()
    flip[::2, 2], flip[::2, 3] = tets[::2, 3], tets[::2, 2]
    from paper_1506_07577_b200.tetfem import TetFEM
    fem = TetFEM(ctx, X, flip, renumber=False, name="orient")
    assert fem.swaps == (tets.shape[0] + 1) // 2
    assert np.array_equal(fem.v.read(), tets)


@pytest.mark.parametrize("n,mesh", [(4, "kuhn6"), (9, "kuhn6"), (3, "alt5")])
def test_renumber_edges_bit_exact(ctx, n, mesh):
    case = Case(n=n, mesh=mesh)
    fem = gpu_fem(ctx, case, name=f"rn{n}{mesh}")
    m, new_of_old, tet_src, order = oracle_renumbered(case)
    assert np.array_equal(fem.vert_order(), order)                    # a2 vertex permutation
    assert np.array_equal(fem.tet_order(), tet_src)                   # a2 tet order
    assert np.array_equal(fem.v.read().astype(np.int64), m.tets)      # remapped keys
    assert fem.ne == m.ne
    assert np.array_equal(fem.tail.read(), m.tail)                    # a1 edge relation
    assert np.array_equal(fem.head.read(), m.head)
    assert np.array_equal(fem.index.read(), m.row_ptr)                # GroupBy index
    assert np.array_equal(fem.e.read().reshape(-1, 4, 4), m.e)        # tets.e[4][4]
    sl = fem.self_e.read()
    assert np.all(m.tail[sl] == np.arange(m.nv)) and np.all(m.head[sl] == np.arange(m.nv))


def test_rest_data_parity(ctx):
    case = Case(n=6)
    fem = gpu_fem(ctx, case, name="rest")
    m, *_ = oracle_renumbered(case)
    assert rel_l2(fem.W.read(), m.W) < 1e-14
    assert rel_l2(fem.Dminv.read(), m.Dminv) < 1e-14
    assert rel_l2(fem.mass.read(), m.mass) < 1e-14


@pytest.mark.parametrize("P", [2, 3, 8])
def test_partition_owner_maps_bit_exact(ctx, P):
    import ctypes as C
    case = Case(n=5)
    fem = gpu_fem(ctx, case, name=f"part{P}")
    m, *_ = oracle_renumbered(case)
    ot = fem.tets.field(f"owner_t{P}", "i32")
    ov = fem.verts.field(f"owner_v{P}", "i32")
    ctx.check(ctx.L.ebb_partition(ctx.h, fem.v.h, P, ot.h, ov.h))
    ref = oracle.partition(m.nv, m.tets, P)
    assert np.array_equal(ot.read(), ref["owner_t"])
    assert np.array_equal(ov.read(), ref["owner_v"])


def test_field_layout_roundtrip_and_view(ctx):
    R = ctx.relation("lay", 37)
    data = np.random.default_rng(0).standard_normal((37, 9))
    f = R.field("K", "f64", (3, 3), "soa", init=data)
    assert np.array_equal(f.read().reshape(37, 9), data)
    v = f.view()
    assert v["count"] == 37 and v["comp_stride"] == 37 * 8 and v["elem_stride"] == 8
    t = f.tensor()
    assert tuple(t.shape) == (9, 37)
    assert np.array_equal(t.cpu().numpy(), data.T)


def test_phase_error_on_alias(ctx):
    import ctypes as C
    from paper_1506_07577_b200 import _abi as A
    from paper_1506_07577_b200 import ebb
    case = Case(n=2)
    fem = gpu_fem(ctx, case, name="phase")
    d = A.TetMapDesc()
    d.model, d.zero_outputs = A.NH, 1
    d.v, d.e, d.u = fem.v.h, fem.e.h, fem.u.h
    d.Dminv, d.W, d.mu, d.lam = fem.Dminv.h, fem.W.h, fem.mu.h, fem.lam.h
    d.f, d.K, d.energy = fem.u.h, A.NONE, A.NONE      # f aliases u: read and reduce phases
    with pytest.raises(ebb.EbbError) as ei:
        ctx.check(ctx.L.ebb_map_tet_forces(ctx.h, C.byref(d), None))
    assert ei.value.name == "EBB_E_PHASE"
