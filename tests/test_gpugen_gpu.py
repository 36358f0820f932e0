"""The GPU generator (cieg_generate_device) writes the same device tile
stream as generating on the host and re-tiling at upload -- bit for bit --
and its device-built tile diagonal equals ci::extract_tile_diagonal's."""
import numpy as np
import pytest

from conftest import gen_from
from paper_1609_01689_b200 import ci, configs

pytestmark = pytest.mark.gpu

CASES = [(20000, 10, 64, 0.05, 0.5, 1, 1, 2000), (60000, 3, 256, 0.02, 0.4, 3, 0, 2000),
         (30000, 4, 200, 0.05, 0.4, 9, 0, 2000)]


@pytest.mark.parametrize("params", CASES)
def test_device_generator_bit_identical(params):
    n, s, t, p, q, seed, prec, beta = params
    host = ci.DeviceMatrix(gen_from(params))
    dev = ci.DeviceMatrix.generate(n, s, t, p, q, seed, prec, beta)
    assert (dev.nnz, dev.ntiles, dev.npanels, dev.tile_edge) == (host.nnz, host.ntiles, host.npanels, host.tile_edge)
    for a, b in zip(dev.export(), host.export()):
        assert np.array_equal(a, b)


# generator tiles smaller than half the device panel (16 / 24-row groups merged
# into 128 / 64-row panels): a diagonal tile spans several groups
SMALL_TILES = [(6000, 3, 16, 0.1, 0.5, 5, 0, 2000), (6000, 3, 24, 0.1, 0.5, 6, 1, 2000)]


@pytest.mark.parametrize("params", CASES[:2] + SMALL_TILES)
def test_device_generator_spmm_and_precond(params):
    n, s, t, p, q, seed, prec, beta = params
    h = gen_from(params)
    dev = ci.DeviceMatrix.generate(n, s, t, p, q, seed, prec, beta)
    x = ci.random_block(n, 16, 4)
    assert np.array_equal(dev.spmm_host(x), ci.DeviceMatrix(h).spmm_host(x))
    td_dev = ci.tile_diagonal_from_matrix(dev)
    td_host = ci.extract_tile_diagonal(h)
    r = ci.random_block(n, 8, 5)
    mu = np.linspace(-3, 1, 8)
    plan = ci.ShiftPlan(mu, np.ones(8, bool))
    assert np.array_equal(ci.apply_preconditioner(td_dev, r, plan), ci.apply_preconditioner(td_host, r, plan))


def test_device_generator_shard_matches_upload_shard():
    from paper_1609_01689_b200 import dist as D

    params = CASES[1]
    n, s, t, p, q, seed, prec, beta = params
    h = gen_from(params)
    rb, _, _ = D.row_partition(h, 3)
    for r in range(3):
        lo, hi = int(rb[r]), int(rb[r + 1])
        dev = ci.DeviceMatrix.generate(n, s, t, p, q, seed, prec, beta, rows=(lo, hi))
        x = ci.random_block(n, 8, 7)
        y = dev.spmm_host(x)
        assert y.shape == (hi - lo, 8)
        # shards are owner-computes: bitwise equal to the full matrix in that mode
        full = ci.DeviceMatrix(h)
        ci.Device.default().set_spmm_mode("owner")
        try:
            np.testing.assert_array_equal(y, full.spmm_host(x)[lo:hi])
        finally:
            ci.Device.default().set_spmm_mode("auto")


def test_lobpcg_on_generated_config1():
    cfg = configs.CFG1
    dm = cfg.generate_device()
    td = ci.tile_diagonal_from_matrix(dm)
    rep = ci.lobpcg_solve(dm, ci.random_block(cfg.n, cfg.kt, 42),
                          ci.LobpcgOptions(k_want=cfg.k_want, tol=cfg.tol, preconditioner=td))
    assert rep.converged and rep.iterations == 84


def test_generated_small_tile_shards():
    """Shards of a generator with 16-row tiles (merged into device panels),
    cut by dist.generated_row_bounds: every shard builds and its rows equal
    the full matrix's, bitwise in owner-computes."""
    import dataclasses

    from paper_1609_01689_b200 import dist as D

    cfg = dataclasses.replace(configs.CFG1, n=6000, sectors=3, tile=16, precision=0)
    full = cfg.generate_device()
    x = ci.random_block(cfg.n, 5, 3)
    dev = ci.Device.default()
    dev.set_spmm_mode("owner")
    try:
        yf = full.spmm_host(x)
        rb = D.generated_row_bounds(cfg, 3)
        for r in range(3):
            lo, hi = int(rb[r]), int(rb[r + 1])
            sh = cfg.generate_device(rows=(lo, hi))
            np.testing.assert_array_equal(sh.spmm_host(x), yf[lo:hi])
    finally:
        dev.set_spmm_mode("auto")

