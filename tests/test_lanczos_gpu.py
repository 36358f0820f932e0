"""The Lanczos baseline on the GPU (cieg_lanczos_solve) vs the reference's
ci::lanczos_solve (lanczos.cpp:24-136): same step count, convergence,
operation counters and per-checkpoint convergence pattern, Ritz values to
1e-10 relative, Ritz vectors to 1e-6 up to sign -- against the committed
fixtures (tests/golden/lanczos.npz) and, where oracle/_ref is built, live."""
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


def check_against(rep, ref, tol, rtol=1e-10):
    """ref: dict-like with iterations/converged/counters/relres/theta/hist_iter/eigenvalues/eigenvectors."""
    assert rep.converged == bool(ref["converged"])
    assert rep.iterations == int(ref["iterations"])
    c = rep.counters
    assert [c.spmm_calls, c.spmv_equivalents, c.precond_applications, c.orthogonalizations] == list(ref["counters"])
    assert [r.iteration for r in rep.history] == list(ref["hist_iter"])
    assert [r.relres > tol for r in rep.history] == [x > tol for x in ref["relres"]]
    np.testing.assert_allclose([r.theta for r in rep.history], ref["theta"], rtol=1e-9, atol=1e-12)
    np.testing.assert_allclose(rep.eigenvalues, ref["eigenvalues"], rtol=rtol)
    ov = np.abs(np.sum(rep.eigenvectors * ref["eigenvectors"], axis=0))
    np.testing.assert_allclose(ov, 1.0, atol=1e-6)


@pytest.mark.parametrize("name", ["diag100_restart", "sector_f64", "sector_f32"])
def test_lanczos_matches_reference_golden(golden, name):
    g = golden("lanczos")
    k, tol, max_iter, _ = g[f"{name}_meta"]
    h = diag100() if name.startswith("diag") else gen_from(g[f"{name}_params"])
    rep = ci.lanczos_solve(h, g[f"{name}_v0"], ci.LanczosOptions(k_want=int(k), tol=float(tol),
                                                                 max_iter=int(max_iter)))
    ref = {key: g[f"{name}_{key}"] for key in ("converged", "iterations", "counters", "relres", "theta",
                                               "hist_iter", "eigenvalues", "eigenvectors")}
    check_against(rep, ref, float(tol))
    np.testing.assert_allclose(rep.eigenvalues, g[f"{name}_dense_eigs"], rtol=1e-7)
    assert rep.norm_estimate == pytest.approx(float(g[f"{name}_norm_estimate"]), rel=1e-10)


def test_lanczos_config1_live_reference(ref_lib):
    """BASELINE config 1 (n = 2e4, fp64 H) from the lowest-sector start,
    against the live compiled reference."""
    cfg = configs.CFG1
    h = cfg.generate()
    v0 = ci.lanczos_default_start(h.dim, h.dim // cfg.sectors)
    rep = ci.lanczos_solve(h, v0, ci.LanczosOptions(k_want=4, tol=1e-8, max_iter=500))
    r = ref_lib.lanczos_solve(ref_lib.RefMatrix(h), v0, 4, 1e-8, 500)
    ref = {"converged": r.converged, "iterations": r.iterations, "counters": r.counters.tolist(),
           "relres": r.history.relres, "theta": r.history.theta, "hist_iter": r.history.iteration,
           "eigenvalues": r.eigenvalues, "eigenvectors": r.trial_vectors}
    check_against(rep, ref, 1e-8)
    assert rep.converged


def test_lanczos_basis_invariants_via_observer():
    """Full reorthogonalisation keeps the basis orthonormal, and V^T H V
    reproduces the tridiagonal (alpha on the diagonal, beta beside it)."""
    h = gen_from((2000, 4, 64, 0.1, 0.5, 11, 1, 500))
    hd = h.to_dense()
    seen = []

    def obs(m, basis, alpha, beta):
        seen.append(m)
        g = basis.T @ basis
        assert np.abs(g - np.eye(m)).max() < 1e-12
        if m == 30:
            t = basis.T @ hd @ basis
            np.testing.assert_allclose(np.diag(t), alpha, atol=1e-12)
            np.testing.assert_allclose(np.diag(t, -1), beta[: m - 1], atol=1e-12)

    v0 = ci.random_block(2000, 1, 3)[:, 0]
    ci.lanczos_solve(h, v0, ci.LanczosOptions(k_want=4, tol=1e-8, max_iter=60, observer=obs))
    assert seen == [10, 20, 30, 40, 50, 60]


def test_lanczos_errors_and_nonconvergence():
    h = diag100()
    with pytest.raises(ci.DimensionMismatch):
        ci.lanczos_solve(h, np.ones(99))
    with pytest.raises(ci.ConfigError):
        ci.lanczos_solve(h, np.zeros(100))
    with pytest.raises(ci.ConfigError):
        ci.lanczos_solve(h, np.ones(100), ci.LanczosOptions(k_want=0))
    rep = ci.lanczos_solve(h, ci.random_block(100, 1, 5)[:, 0], ci.LanczosOptions(k_want=3, tol=1e-14, max_iter=7))
    assert rep.iterations == 7 and not rep.converged  # last step is always analysed (lanczos.cpp:102)
    assert len(rep.eigenvalues) == 3


def test_lanczos_vs_lobpcg_same_spectrum():
    """The paper's comparison: both solvers find the same lowest eigenvalues
    on the same fp32 sector matrix."""
    h = gen_from((3072, 3, 256, 0.2, 0.4, 13, 0, 2000))
    la = ci.lanczos_solve(h, ci.lanczos_default_start(h.dim, 1024), ci.LanczosOptions(k_want=4, tol=1e-7))
    lo = ci.lobpcg_solve(h, ci.random_block(h.dim, 8, 43),
                         ci.LobpcgOptions(k_want=4, tol=1e-7, preconditioner=ci.extract_tile_diagonal(h)))
    assert la.converged and lo.converged
    np.testing.assert_allclose(la.eigenvalues, lo.eigenvalues, rtol=1e-7)
