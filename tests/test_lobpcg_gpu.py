"""LOBPCG on the GPU vs the reference's lobpcg_solve: identical iteration
count, identical per-iteration active (soft-locking) sets, identical
operation counters, eigenvalues to 1e-8 relative (fp64 H) / 1e-5 (fp32 H),
residuals under tol -- the BASELINE.json north-star parity contract -- plus
the SPEC.md:348-391 examples and invariants."""
import numpy as np
import pytest

from conftest import gen_from
from paper_1609_01689_b200 import ci, configs

pytestmark = pytest.mark.gpu


def diag100():
    n = 100
    return ci.CsbMatrix(dim=n, precision=1, block_boundaries=np.array([0, n], np.uint32),
                        entry_offsets=np.array([0, n], np.uint64), rows=np.arange(n, dtype=np.uint16),
                        cols=np.arange(n, dtype=np.uint16), values=np.arange(1, n + 1, dtype=np.float64),
                        groups=np.array([0, 50, n], np.uint32))


def active_sets(relres, kt, tol):
    rr = np.asarray(relres).reshape(-1, kt)
    return [tuple(np.nonzero(r > tol)[0]) for r in rr]


@pytest.mark.parametrize("name", ["diag100", "sector_f64", "sector_f64_prec", "sector_f32_prec"])
def test_lobpcg_matches_reference(golden, name):
    g = golden("lobpcg")
    k, kt, tol, pre, seed = g[f"{name}_meta"]
    k, kt, seed = int(k), int(kt), int(seed)
    h = diag100() if name == "diag100" else gen_from(g[f"{name}_params"])
    x0 = ci.random_block(h.dim, kt, seed)
    td = ci.extract_tile_diagonal(h) if pre else None
    rep = ci.lobpcg_solve(h, x0, ci.LobpcgOptions(k_want=k, tol=float(tol), preconditioner=td))
    assert rep.converged == bool(g[f"{name}_converged"])
    assert rep.iterations == int(g[f"{name}_iterations"])
    assert [rep.counters.spmm_calls, rep.counters.spmv_equivalents, rep.counters.precond_applications,
            rep.counters.orthogonalizations] == g[f"{name}_counters"].tolist()
    relres = np.array([r.relres for r in rep.history])
    assert active_sets(relres, kt, tol) == active_sets(g[f"{name}_relres"], kt, tol)
    is_f32 = name.endswith("f32_prec")
    np.testing.assert_allclose(rep.eigenvalues, g[f"{name}_eigenvalues"], rtol=1e-5 if is_f32 else 1e-8)
    if f"{name}_dense_eigs" in g:
        np.testing.assert_allclose(rep.eigenvalues, g[f"{name}_dense_eigs"], rtol=1e-6 if is_f32 else 1e-8)
    # the final residuals are under tol for the wanted pairs
    assert np.all(relres.reshape(-1, kt)[-1, :k] <= tol)


def test_spec_diag_example():
    """diag(1..100), k_want = 3, random X0 width 5 -> {1, 2, 3}."""
    rep = ci.lobpcg_solve(diag100(), ci.random_block(100, 5, 7), ci.LobpcgOptions(k_want=3, tol=1e-10))
    np.testing.assert_allclose(rep.eigenvalues, [1.0, 2.0, 3.0], atol=1e-8)


def test_lobpcg_config1_live_reference(ref_lib):
    """BASELINE config 1 end to end against the live reference."""
    cfg = configs.CFG1
    h = cfg.generate()
    x0 = ci.random_block(h.dim, cfg.kt, 42)
    rm = ref_lib.RefMatrix(h)
    for pre in (False, True):
        rtd = ref_lib.RefTileDiagonal(rm, h.groups) if pre else None
        rr = ref_lib.lobpcg_solve(rm, x0, cfg.k_want, cfg.tol, 500, rtd)
        td = ci.extract_tile_diagonal(h) if pre else None
        rep = ci.lobpcg_solve(h, x0, ci.LobpcgOptions(k_want=cfg.k_want, tol=cfg.tol, preconditioner=td))
        assert rep.iterations == rr.iterations and rep.converged == rr.converged
        assert rep.counters.precond_applications == rr.counters[2]
        assert active_sets([r.relres for r in rep.history], cfg.kt, cfg.tol) == \
            active_sets(rr.history.relres, cfg.kt, cfg.tol)
        np.testing.assert_allclose(rep.eigenvalues, rr.eigenvalues, rtol=1e-8)


def test_lobpcg_invariants_via_observer():
    """X^T X = I to 1e-10 each iteration; the trace of the
    k_want smallest Ritz values never increases; Ritz values bound the
    eigenvalues from above."""
    h = gen_from((2000, 4, 64, 0.1, 0.5, 11, 1, 500))
    exact = np.linalg.eigvalsh(h.to_dense())
    views = []
    ci.lobpcg_solve(h, ci.random_block(h.dim, 8, 42),
                    ci.LobpcgOptions(k_want=4, tol=1e-8, observer=lambda v: views.append(v)))
    assert len(views) > 5
    prev = np.inf
    for v in views:
        assert np.abs(v.X.T @ v.X - np.eye(8)).max() < 1e-10
        tr = v.theta[:4].sum()
        assert tr <= prev + 1e-10 * abs(tr)
        prev = tr
        assert np.all(v.theta >= exact[:8] - 1e-10)


def test_lobpcg_errors_and_nonconvergence():
    h = gen_from((2000, 4, 64, 0.1, 0.5, 11, 1, 500))
    with pytest.raises(ci.ConfigError):
        ci.lobpcg_solve(h, ci.random_block(h.dim, 3, 1), ci.LobpcgOptions(k_want=4))
    with pytest.raises(ci.DimensionMismatch):
        ci.lobpcg_solve(h, ci.random_block(h.dim + 1, 8, 1), ci.LobpcgOptions(k_want=4))
    x0 = ci.random_block(h.dim, 6, 1)
    x0[:, 3:] = x0[:, :3]  # only 3 independent columns
    with pytest.raises(ci.SubspaceCollapse):
        ci.lobpcg_solve(h, x0, ci.LobpcgOptions(k_want=4))
    rep = ci.lobpcg_solve(h, ci.random_block(h.dim, 8, 1), ci.LobpcgOptions(k_want=4, tol=1e-12, max_iter=3))
    assert not rep.converged and rep.iterations == 3


def test_lobpcg_fp32_config_scaled():
    """A 256-tile fp32 matrix with the config-4 solver settings (k_want 8,
    block 16, tol 1e-6, FOM(3) tile preconditioner) against dense eigenvalues."""
    h = gen_from((4096, 4, 256, 0.1, 0.4, 3, 0, 2000))
    td = ci.extract_tile_diagonal(h)
    rep = ci.lobpcg_solve(h, ci.random_block(h.dim, 16, 5), ci.LobpcgOptions(k_want=8, tol=1e-6, preconditioner=td))
    assert rep.converged
    exact = np.linalg.eigvalsh(h.to_dense())[:8]
    np.testing.assert_allclose(rep.eigenvalues, exact, rtol=1e-5)


def test_smoke_entry():
    import __graft_entry__

    __graft_entry__.smoke()


def test_trial_width_limit_is_a_config_error():
    """trial widths above 16 (Rayleigh-Ritz bases above 48
    columns) are not supported by the GPU solver -- a ConfigError with the
    reason, before any work (documented in INTEGRATION.md); ci::lobpcg_solve
    itself has no such limit."""
    h = gen_from((2000, 4, 64, 0.1, 0.5, 11, 1, 500))
    with pytest.raises(ci.ConfigError, match="above 16"):
        ci.lobpcg_solve(h, ci.random_block(h.dim, 17, 1), ci.LobpcgOptions(k_want=3, tol=1e-8))
