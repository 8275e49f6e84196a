"""GPU parity of the matrix-free element-by-element matvec:
q = sum_t K_t p_t from the compact per-tet state equals the oracle's
assembled edge-relation product K p (K from the oracle's generic
4th-order-tensor element map) and the GPU's own assembled matvec.

Bars: fp64 <= 1e-12 relative, fp32 <= 1e-5 (oracle fed the fp32-rounded
inputs)."""
import numpy as np
import pytest

import oracle
from helpers import Case, gpu_fem, oracle_renumbered, rel_l2

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


@pytest.mark.parametrize("model", ["nh", "stvk"])
@pytest.mark.parametrize("dtype,tol", [("f64", 1e-12), ("f32", 1e-5)])
def test_ebe_matvec_equals_assembled_product(ctx, model, dtype, tol):
    case = Case(n=6, model=model, spread=0.1)
    if dtype == "f32":
        case.u = case.u.astype(np.float32).astype(np.float64)
        case.mu = case.mu.astype(np.float32).astype(np.float64)
        case.lam = case.lam.astype(np.float32).astype(np.float64)
    fem = gpu_fem(ctx, case, dtype=dtype, name=f"ebe{model}{dtype}")
    m, new_of_old, tet_src, order = oracle_renumbered(case)
    rng = np.random.default_rng(6)
    p = rng.uniform(-1, 1, size=(m.nv, 3))
    if dtype == "f32":
        p = p.astype(np.float32).astype(np.float64)
    f, K, en, inv = oracle.element_map(model, m.X, case.u[order], m.tets, m.Dminv, m.W, case.mu[tet_src],
                                       case.lam[tet_src], e=m.e, ne=m.ne)
    ref = oracle.edge_matvec(m.row_ptr, m.head, K, p)
    st = fem.ebe_state(model)
    P = fem.verts.field("p_ebe", dtype, (3, 1), init=p)
    Q = fem.verts.field("q_ebe", dtype, (3, 1))
    fem.ebe_matvec(st, P, Q, model=model)
    q = Q.read()
    assert rel_l2(q, ref) <= tol
    # the GPU's assembled product of the same state
    fem.map_forces(model)
    Q2 = fem.verts.field("q_asm", dtype, (3, 1))
    fem.matvec(fem.K, P, Q2)
    assert rel_l2(q, Q2.read()) <= tol
    assert ctx.error_counts(reset=True)["inverted"] == 0


def test_ebe_state_shape_is_checked(ctx):
    from paper_1506_07577_b200.ebb import EbbError
    case = Case(n=3)
    fem = gpu_fem(ctx, case, name="ebebad")
    st = fem.ebe_state("nh")                      # 15 words
    P = fem.verts.field("p", "f64", (3, 1))
    with pytest.raises(EbbError, match="EBB_E_TYPE"):
        fem.ebe_matvec(st, P, fem.verts.field("q", "f64", (3, 1)), model="stvk")   # StVK needs 26
    with pytest.raises(EbbError, match="EBB_E_PHASE"):
        fem.ebe_matvec(st, P, P, model="nh")
