"""Seeded randomized sweep of the generator parameters (sizes, sectors, tile
sizes, band, tile / entry densities, precision) and block widths: the CUDA
SpMM against the oracle's sequential restatement of spmm (csb.cpp:118-193),
and the GPU generator bit-identical to host generation + upload. Exercises
the tiler, panel planning and the bank-aware entry order on irregular
shapes the fixed configs do not reach."""
import numpy as np
import pytest

from conftest import single_pass_shards
from oracle import ci_oracle as O
from paper_1609_01689_b200 import ci

pytestmark = pytest.mark.gpu

rng = np.random.default_rng(20261020)
CASES = []
for _ in range(24):
    sectors = int(rng.integers(1, 7))
    tile = int(rng.choice([8, 16, 33, 64, 100, 128, 200, 256]))
    n = int(rng.integers(max(sectors, 40), 6000)) // sectors * sectors
    CASES.append(dict(n=n, sectors=sectors, tile=tile, p=float(rng.uniform(0.05, 1.0)),
                      q=float(rng.uniform(0.05, 1.0)), seed=int(rng.integers(1, 1 << 30)),
                      precision=int(rng.integers(0, 2)), beta=max(tile, 256), band=int(rng.integers(0, 4)),
                      m=int(rng.integers(1, 21))))


@pytest.mark.parametrize("c", CASES, ids=[f"n{c['n']}s{c['sectors']}t{c['tile']}b{c['band']}p{c['precision']}m{c['m']}"
                                          for c in CASES])
def test_random_generator_configs(c):
    h = ci.generate_sector_matrix(c["n"], c["sectors"], c["tile"], c["p"], c["q"], c["seed"], c["precision"],
                                  c["beta"], band=c["band"])
    x = ci.random_block(h.dim, c["m"], c["seed"] % 1000)
    dm = ci.DeviceMatrix(h)
    y = dm.spmm_host(x)
    yo = O.spmm(h, x)
    scale = max(np.abs(yo).max(), 1e-300)
    assert np.abs(y - yo).max() <= 1e-14 * scale
    for mode in ("owner", "single"):  # both K1 modes, whatever auto chose
        dm.device.set_spmm_mode(mode)
        try:
            assert np.abs(dm.spmm_host(x) - yo).max() <= 1e-14 * scale
        finally:
            dm.device.set_spmm_mode("auto")
    # single-pass row shards (world 2), partials reduced at their owners
    if len(h.groups) > 2:
        ys = single_pass_shards(h, 2, c["m"], x)
        assert np.abs(ys - yo).max() <= 1e-14 * scale
    dev = ci.DeviceMatrix.generate(c["n"], c["sectors"], c["tile"], c["p"], c["q"], c["seed"], c["precision"],
                                   c["beta"], band=c["band"])
    host = ci.DeviceMatrix(h)
    for a, b in zip(dev.export(), host.export()):
        assert np.array_equal(a, b)


rng2 = np.random.default_rng(7)
LOBPCG_CASES = []
for _ in range(16):
    sectors = int(rng2.integers(2, 6))
    tile = int(rng2.choice([32, 64, 128]))
    n = int(rng2.integers(800, 4000)) // sectors * sectors
    kt = int(rng2.choice([4, 6, 8]))
    LOBPCG_CASES.append(dict(n=n, sectors=sectors, tile=tile, p=float(rng2.uniform(0.1, 0.6)),
                             q=float(rng2.uniform(0.2, 0.6)), seed=int(rng2.integers(1, 1 << 30)),
                             precision=int(rng2.integers(0, 2)), band=int(rng2.integers(1, 3)), kt=kt,
                             k=int(rng2.integers(1, kt // 2 + 1)), prec=bool(rng2.integers(0, 2))))


@pytest.mark.parametrize("c", LOBPCG_CASES,
                         ids=[f"n{c['n']}t{c['tile']}k{c['k']}kt{c['kt']}p{c['precision']}{'P' if c['prec'] else ''}"
                              for c in LOBPCG_CASES])
def test_random_lobpcg_vs_live_reference(ref_lib, c):
    """The north-star contract on random small problems: same iteration count
    and counters as the reference's lobpcg_solve, eigenvalues to 1e-8 (fp64 H)
    / 1e-5 (fp32 H) relative."""
    h = ci.generate_sector_matrix(c["n"], c["sectors"], c["tile"], c["p"], c["q"], c["seed"], c["precision"], 2000,
                                  band=c["band"])
    tol = 1e-8 if c["precision"] == 1 else 1e-6
    x0 = ci.random_block(h.dim, c["kt"], c["seed"] % 997)
    td = ci.extract_tile_diagonal(h) if c["prec"] else None
    rep = ci.lobpcg_solve(h, x0, ci.LobpcgOptions(k_want=c["k"], tol=tol, preconditioner=td))
    rm = ref_lib.RefMatrix(h)
    rtd = ref_lib.RefTileDiagonal(rm, h.groups) if c["prec"] else None
    r = ref_lib.lobpcg_solve(rm, x0, c["k"], tol, 500, rtd)
    assert rep.converged == r.converged
    assert rep.iterations == r.iterations
    assert [rep.counters.spmm_calls, rep.counters.spmv_equivalents, rep.counters.precond_applications,
            rep.counters.orthogonalizations] == r.counters.tolist()
    np.testing.assert_allclose(rep.eigenvalues, r.eigenvalues, rtol=1e-8 if c["precision"] == 1 else 1e-5)


rng3 = np.random.default_rng(11)
LANCZOS_CASES = []
for _ in range(6):
    sectors = int(rng3.integers(2, 6))
    n = int(rng3.integers(600, 3000)) // sectors * sectors
    LANCZOS_CASES.append(dict(n=n, sectors=sectors, tile=int(rng3.choice([32, 64, 128])),
                              p=float(rng3.uniform(0.1, 0.6)), q=float(rng3.uniform(0.2, 0.6)),
                              seed=int(rng3.integers(1, 1 << 30)), precision=int(rng3.integers(0, 2)),
                              k=int(rng3.integers(1, 5))))


@pytest.mark.parametrize("c", LANCZOS_CASES, ids=[f"n{c['n']}k{c['k']}p{c['precision']}" for c in LANCZOS_CASES])
def test_random_lanczos_vs_live_reference(ref_lib, c):
    h = ci.generate_sector_matrix(c["n"], c["sectors"], c["tile"], c["p"], c["q"], c["seed"], c["precision"], 2000)
    v0 = ci.lanczos_default_start(h.dim, h.dim // c["sectors"])
    rep = ci.lanczos_solve(h, v0, ci.LanczosOptions(k_want=c["k"], tol=1e-8, max_iter=300))
    r = ref_lib.lanczos_solve(ref_lib.RefMatrix(h), v0, c["k"], 1e-8, 300)
    assert rep.converged == r.converged and rep.iterations == r.iterations
    np.testing.assert_allclose(rep.eigenvalues, r.eigenvalues, rtol=1e-10)
