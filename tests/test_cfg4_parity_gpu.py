"""LOBPCG on the GPU against the live reference (oracle/_ref: the unmodified
proj/src/lobpcg.cpp:216-387) at the settings the config-4/5 solve numbers are
quoted on: trial width kt = 16, k_want = 8, tol 1e-6, fp32 H, 256-row tiles,
the tile-diagonal preconditioner (FOM(3) on 256-row groups, LU on the 64-row
sector tails). These exercise what the config-1 checks do not: the NT = 2 K1
inside the solve (active widths 9-16), the 48-wide Rayleigh-Ritz Grams and
FOM on 256-row groups.

Contract (BASELINE.json north_star): identical iteration count, convergence
flag, operation counters and per-iteration active (soft-locking) sets;
eigenvalues to 1e-5 relative for fp32 H (asserted at 1e-9 here), final
residuals under tol.
"""
import os

import numpy as np
import pytest

from paper_1609_01689_b200 import ci, configs

pytestmark = pytest.mark.gpu


def active_sets(relres, kt, tol):
    rr = np.asarray(relres).reshape(-1, kt)
    return [tuple(np.nonzero(r > tol)[0]) for r in rr]


def cfg4_shaped(n_per_sector, stored_per_row, seed):
    """The config-4 generator shape at test size: 25 sectors of
    k * 256 + 64 rows (256-row FOM groups and a 64-row LU tail per sector)."""
    n = 25 * n_per_sector
    return configs.Config("cfg4-shape", n, 25, 256, None, 0.4, 0, n * stored_per_row, k_want=8, kt=16, tol=1e-6,
                          seed=seed)


def compare(rep, rr, kt, k_want, tol):
    assert rep.iterations == rr.iterations
    assert rep.converged == rr.converged
    assert [rep.counters.spmm_calls, rep.counters.spmv_equivalents, rep.counters.precond_applications,
            rep.counters.orthogonalizations] == rr.counters.tolist()
    assert active_sets([r.relres for r in rep.history], kt, tol) == active_sets(rr.history.relres, kt, tol)
    np.testing.assert_allclose(rep.eigenvalues, rr.eigenvalues, rtol=1e-9)


def reference_counts(ref_lib, rm, x0, k_want, tol, rtd):
    """The reference's iteration count from X0 and from two perturbations of
    X0 by 1e-15 relative noise: an LOBPCG count is only a parity target
    where the reference itself is stable under rounding-level changes
    (clustered Ritz values near tol can move it by 10+ iterations)."""
    rng = np.random.default_rng(0)
    rr = ref_lib.lobpcg_solve(rm, x0, k_want, tol, 500, rtd)
    counts = {rr.iterations}
    for _ in range(2):
        xp = x0 * (1.0 + 1e-15 * rng.standard_normal(x0.shape))
        counts.add(ref_lib.lobpcg_solve(rm, xp, k_want, tol, 500, rtd).iterations)
    return rr, counts


@pytest.mark.parametrize("n_per_sector,per_row,seed,x_seed,pre", [
    (2368, 400, 3, 42, True),    # 9 x 256 + 64 rows per sector, ~380 stored per row
    (2112, 600, 7, 5, True),     # 8 x 256 + 64, denser
    (1088, 300, 13, 9, False),   # 4 x 256 + 64, unpreconditioned (255 it)
    (832, 400, 17, 3, False),    # 3 x 256 + 64, unpreconditioned (271 it)
    (1088, 300, 11, 9, False),   # rounding-sensitive: the reference gives 304 or 318 under 1e-15 noise
])
def test_lobpcg_cfg4_settings_live_reference(ref_lib, n_per_sector, per_row, seed, x_seed, pre):
    cfg = cfg4_shaped(n_per_sector, per_row, seed)
    h = cfg.generate()
    x0 = ci.random_block(h.dim, cfg.kt, x_seed)
    rm = ref_lib.RefMatrix(h)
    rtd = ref_lib.RefTileDiagonal(rm, h.groups) if pre else None
    rr, counts = reference_counts(ref_lib, rm, x0, cfg.k_want, cfg.tol, rtd)
    td = ci.extract_tile_diagonal(h) if pre else None
    rep = ci.lobpcg_solve(h, x0, ci.LobpcgOptions(k_want=cfg.k_want, tol=cfg.tol, preconditioner=td))
    assert rr.converged and rep.converged
    if len(counts) == 1:  # a stable count: the full contract
        compare(rep, rr, cfg.kt, cfg.k_want, cfg.tol)
    else:  # a count the reference itself does not hold under rounding noise
        assert rep.iterations in counts
        # two converged solves stopping at different iterations (relres 1e-6):
        # eigenvalues agree to ~relres^2 relative, within north_star's 1e-5
        np.testing.assert_allclose(rep.eigenvalues, rr.eigenvalues, rtol=1e-7)
    assert np.all(np.array([r.relres for r in rep.history]).reshape(-1, cfg.kt)[-1, :cfg.k_want] <= cfg.tol)
    if pre:
        assert rep.counters.precond_applications > 0  # the FOM/LU groups were exercised


def _host_ram_gb():
    try:
        import psutil

        return psutil.virtual_memory().available / 2**30
    except Exception:
        return 0.0


@pytest.mark.slow
@pytest.mark.skipif(os.environ.get("CIEG_SKIP_SLOW") == "1", reason="CIEG_SKIP_SLOW=1")
def test_lobpcg_cfg4_full_size_capped(ref_lib):
    """The full config-4 matrix (n = 5e6, S = 5e9, fp32 H, 256-row tiles,
    tile preconditioner), both sides capped at 6 iterations: per-iteration
    Ritz values and relative residuals, active sets and counters against
    ci::lobpcg_solve. Our matrix is generated on the GPU
    (cieg_generate_device), the reference's by the oracle's generator
    (oracle/ref_gen.cpp) -- two independent builds of the same seeded matrix."""
    if _host_ram_gb() < 160:
        pytest.skip("needs ~120 GB of host memory for the reference's copy of config 4")
    cfg = configs.CFG4
    it_cap = 6
    rm = ref_lib.generate(cfg.n, cfg.sectors, cfg.tile, cfg.p(), cfg.q, cfg.seed, cfg.precision, cfg.beta)
    starts = []
    for s in range(cfg.sectors):
        a, b = cfg.n * s // cfg.sectors, cfg.n * (s + 1) // cfg.sectors
        starts.extend(range(a, b, cfg.tile))
    bounds = np.array(starts + [cfg.n], np.uint32)
    rtd = ref_lib.RefTileDiagonal(rm, bounds)
    x0 = ci.random_block(cfg.n, cfg.kt, 42)
    rr = ref_lib.lobpcg_solve(rm, x0, cfg.k_want, cfg.tol, it_cap, rtd)
    del rtd, rm
    dm = cfg.generate_device()
    assert dm.nnz == int(ref_lib.count_nnz(cfg.n, cfg.sectors, cfg.tile, cfg.p(), cfg.q, cfg.seed))
    td = ci.tile_diagonal_from_matrix(dm)
    rep = ci.lobpcg_solve(dm, x0, ci.LobpcgOptions(k_want=cfg.k_want, tol=cfg.tol, max_iter=it_cap,
                                                   preconditioner=td))
    assert rep.iterations == rr.iterations == it_cap and not rep.converged and not rr.converged
    assert rep.counters.spmm_calls == rr.counters[0]
    assert rep.counters.precond_applications == rr.counters[2]
    th = np.array([r.theta for r in rep.history])
    rel = np.array([r.relres for r in rep.history])
    np.testing.assert_allclose(th, rr.history.theta, rtol=1e-11)
    np.testing.assert_allclose(rel, rr.history.relres, rtol=1e-7)
    assert active_sets(rel, cfg.kt, cfg.tol) == active_sets(rr.history.relres, cfg.kt, cfg.tol)
