"""Seeded randomized sweep of the generator parameters (sizes, sectors, tile
sizes, band, tile / entry densities, precision) and block widths: the CUDA
SpMM against the oracle's sequential restatement of spmm (csb.cpp:118-193),
and the GPU generator bit-identical to host generation + upload. Exercises
the tiler, panel planning and the bank-aware entry order on irregular
shapes the fixed configs do not reach."""
import numpy as np
import pytest

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
    y = ci.DeviceMatrix(h).spmm_host(x)
    yo = O.spmm(h, x)
    assert np.abs(y - yo).max() <= 1e-14 * max(np.abs(yo).max(), 1e-300)
    dev = ci.DeviceMatrix.generate(c["n"], c["sectors"], c["tile"], c["p"], c["q"], c["seed"], c["precision"],
                                   c["beta"], band=c["band"])
    host = ci.DeviceMatrix(h)
    for a, b in zip(dev.export(), host.export()):
        assert np.array_equal(a, b)
