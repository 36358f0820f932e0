"""K2-K5 parity on the GPU: Gram / combine / column norms against the
reference's block_vectors.cpp (golden + live), and the tile preconditioner
against ci::apply_preconditioner -- bitwise, because K5 keeps the
reference's operation order (precond.cu)."""
import numpy as np
import pytest

from conftest import gen_from
from oracle import ci_oracle as O
from paper_1609_01689_b200 import ci

pytestmark = pytest.mark.gpu
TOL = 1e-13


def rel(a, b):
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


def test_block_kernels_match_reference(golden):
    g = golden("blockvec")
    x = ci.random_block(1003, 24, 1)
    y = ci.random_block(1003, 20, 2)
    gg = 2.0 * ci.random_block(24, 16, 3)
    assert rel(ci.block_inner(x, y), g["block_inner"]) < TOL
    assert rel(ci.linear_combination(x, gg), g["linear_combination"]) < TOL
    yy = ci.random_block(1003, 16, 4)
    ci.add_linear_combination(yy, x, gg)
    assert rel(yy, g["add_linear_combination"]) < TOL
    np.testing.assert_allclose(ci.column_norms(x), np.sqrt(np.diag(O.block_inner(x, x))), rtol=1e-14)


@pytest.mark.parametrize("n", [1, 3, 4, 7, 8, 257, 4099, 100_003])
@pytest.mark.parametrize("kx,ky", [(1, 1), (3, 5), (8, 8), (17, 9), (48, 48), (48, 1)])
def test_gram_shapes(n, kx, ky):
    x = ci.random_block(n, kx, n + kx)
    y = ci.random_block(n, ky, n + ky + 1)
    assert rel(ci.block_inner(x, y), O.block_inner(x, y)) < 1e-12


@pytest.mark.parametrize("n", [1, 9, 1000, 65_537])
@pytest.mark.parametrize("kin,kout", [(1, 1), (5, 3), (16, 16), (48, 32), (24, 48)])
def test_combine_shapes(n, kin, kout):
    y = ci.random_block(n, kin, 3)
    g = ci.random_block(kin, kout, 4)
    assert rel(ci.linear_combination(y, g), O.linear_combination(y, g)) < 1e-12


def test_gram_deterministic():
    x = ci.random_block(300_001, 16, 1)
    a = ci.block_inner(x, x)
    assert np.array_equal(a, ci.block_inner(x, x))
    assert np.array_equal(a, a.T)  # same fixed-order sums for (a,b) and (b,a)


@pytest.fixture
def exact_order():
    dev = ci.Device.default()
    dev.set_exact_order(True)
    yield
    dev.set_exact_order(False)


@pytest.mark.parametrize("name", ["lu", "fom"])
def test_preconditioner_bitwise_vs_reference(golden, name, exact_order):
    g = golden("precond")
    h = gen_from(g[f"{name}_params"])
    td = ci.extract_tile_diagonal(h)
    r = ci.random_block(h.dim, 8, 31)
    w = ci.apply_preconditioner(td, r, ci.ShiftPlan(g[f"{name}_mu"], g[f"{name}_engage"]))
    assert np.array_equal(w, g[f"{name}_w"])


@pytest.mark.parametrize("name", ["lu", "fom"])
def test_preconditioner_fast_path_vs_reference(golden, name):
    """Default (tensor-core FOM) path: same result to rounding."""
    g = golden("precond")
    h = gen_from(g[f"{name}_params"])
    td = ci.extract_tile_diagonal(h)
    r = ci.random_block(h.dim, 8, 31)
    w = ci.apply_preconditioner(td, r, ci.ShiftPlan(g[f"{name}_mu"], g[f"{name}_engage"]))
    assert rel(w, g[f"{name}_w"]) < 1e-12


def test_preconditioner_live_reference(ref_lib, exact_order):
    h = gen_from((6144, 3, 256, 0.1, 0.4, 5, 0, 2000))
    rm = ref_lib.RefMatrix(h)
    rtd = ref_lib.RefTileDiagonal(rm, h.groups)
    td = ci.extract_tile_diagonal(h)
    r = ci.random_block(h.dim, 16, 2)
    mu = np.full(16, -3.5)
    mu[:4] = [-4.0, -3.9, -3.9, -3.8]
    en = np.ones(16, bool)
    en[[3, 9]] = False
    w = ci.apply_preconditioner(td, r, ci.ShiftPlan(mu, en))
    assert np.array_equal(w, ref_lib.apply_preconditioner(rtd, r, mu, en))


def test_preconditioner_identity_and_passthrough():
    """H~ = I, mu = 0 -> W = R; engage all false -> W = R."""
    bounds = np.array([0, 40, 64, 200], np.uint32)
    blocks = [np.eye(40), np.eye(24), np.eye(136)]
    td = ci.TileDiagonal.from_blocks(bounds, blocks)
    r = ci.random_block(200, 5, 9)
    w = ci.apply_preconditioner(td, r, ci.ShiftPlan(np.zeros(5), np.ones(5, bool)))
    np.testing.assert_allclose(w, r, rtol=1e-15, atol=0)
    w = ci.apply_preconditioner(td, r, ci.ShiftPlan(np.zeros(5), np.zeros(5, bool)))
    assert np.array_equal(w, r)


def test_preconditioner_exact_direct_solve():
    """one group = the whole H (n <= 64), shift below lambda_min
    -> W = (H - mu I)^{-1} R to 1e-10."""
    rng = np.random.default_rng(1)
    a = rng.standard_normal((50, 50))
    hb = a + a.T + 30 * np.eye(50)
    td = ci.TileDiagonal.from_blocks(np.array([0, 50], np.uint32), [hb])
    r = rng.standard_normal((50, 3))
    mu = np.linalg.eigvalsh(hb)[0] - 1.0
    w = ci.apply_preconditioner(td, r, ci.ShiftPlan(np.full(3, mu), np.ones(3, bool)))
    np.testing.assert_allclose(w, np.linalg.solve(hb - mu * np.eye(50), r), rtol=1e-10)


def test_preconditioner_singular_shift_passthrough(capfd):
    """precond.cpp:61-83: an exactly singular shifted block is perturbed once;
    a block singular for every shift passes the residual through (warning)."""
    z = np.zeros((8, 8))
    td = ci.TileDiagonal.from_blocks(np.array([0, 8], np.uint32), [z])
    r = ci.random_block(8, 2, 3)
    w = ci.apply_preconditioner(td, r, ci.ShiftPlan(np.zeros(2), np.ones(2, bool)))
    # (0 - mu) I with mu = 0 is singular; mu' = 1e-8 is not: W = -R / 1e-8
    np.testing.assert_allclose(w, r / -1e-8, rtol=1e-12)
    # diag(0, 1e-8, 1, ...) is singular at mu = 0 and at the perturbed 1e-8
    b = np.diag([0.0, 1e-8, 1.0, 2.0, 3.0, 4.0, 5.0, 6.0])
    td = ci.TileDiagonal.from_blocks(np.array([0, 8], np.uint32), [b])
    capfd.readouterr()
    w = ci.apply_preconditioner(td, r, ci.ShiftPlan(np.zeros(2), np.ones(2, bool)))
    assert np.array_equal(w, r)
    assert "singular shifted tile block" in capfd.readouterr().err


def test_fom_matches_direct_for_saturating_krylov():
    """10x10 SPD block, iters >= n is exact; here FOM(3) on a
    block with 3 distinct eigenvalues saturates the Krylov space."""
    rng = np.random.default_rng(2)
    q, _ = np.linalg.qr(rng.standard_normal((96, 96)))
    ev = np.repeat([5.0, 7.0, 11.0], 32)
    hb = (q * ev) @ q.T
    hb = 0.5 * (hb + hb.T)
    td = ci.TileDiagonal.from_blocks(np.array([0, 96], np.uint32), [hb])
    r = rng.standard_normal((96, 4))
    w = ci.apply_preconditioner(td, r, ci.ShiftPlan(np.zeros(4), np.ones(4, bool)))
    np.testing.assert_allclose(w, np.linalg.solve(hb, r), rtol=1e-9)
