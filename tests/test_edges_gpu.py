"""Edge cases of the SpMM path vs the oracle's sequential restatement of
spmm (csb.cpp:118-193, bitwise equal to spmm_serial): rows and panels with
no stored entries, tiny and ragged dimensions, an empty block, a matrix
assembled by the reference itself (physics basis, small groups), forced
tile edges, fp32 subnormal / extreme values."""
import numpy as np
import pytest

from conftest import gen_from
from oracle import ci_oracle as O
from paper_1609_01689_b200 import ci

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True, params=["auto", "owner", "single"])
def spmm_mode(request):
    """Every edge case in each K1 mode: owner-computes, single pass (DMMA;
    the scalar consumer at m <= 2) and the default per-width choice."""
    dev = ci.Device.default()
    dev.set_spmm_mode(request.param)
    yield request.param
    dev.set_spmm_mode("auto")


def csb_from_coo(n, r, c, v, block_rows, precision=1, groups=None):
    """Lower-triangle CSB (csb.hpp layout) from global (r >= c) triplets."""
    bb = np.asarray(block_rows, dtype=np.uint32)
    nb = len(bb) - 1
    bi = np.searchsorted(bb, r, side="right") - 1
    bj = np.searchsorted(bb, c, side="right") - 1
    lin = bi * (bi + 1) // 2 + bj
    order = np.lexsort((c, r, lin))
    r, c, v, lin, bi, bj = r[order], c[order], v[order], lin[order], bi[order], bj[order]
    counts = np.bincount(lin, minlength=nb * (nb + 1) // 2)
    eo = np.concatenate([[0], np.cumsum(counts)]).astype(np.uint64)
    return ci.CsbMatrix(dim=n, precision=precision, block_boundaries=bb, entry_offsets=eo,
                        rows=(r - bb[bi]).astype(np.uint16), cols=(c - bb[bj]).astype(np.uint16),
                        values=np.asarray(v, dtype=np.float32 if precision == 0 else np.float64), groups=groups)


def check(h, m=5, seed=1, **kw):
    x = ci.random_block(h.dim, m, seed)
    y = ci.DeviceMatrix(h, **kw).spmm_host(x)
    yo = O.spmm(h, x)
    # relative to the block's scale (cancellation makes single elements small)
    assert np.abs(y - yo).max() <= 1e-14 * max(np.abs(yo).max(), 1e-300)
    return y


def test_rows_and_panels_without_entries():
    """A 300-row band with no stored entries at all (not even the diagonal):
    its panels get no-op work items and their rows come out exactly 0."""
    rng = np.random.default_rng(0)
    n = 1000
    r = rng.integers(0, n, 6000)
    c = rng.integers(0, n, 6000)
    r, c = np.maximum(r, c), np.minimum(r, c)
    keep = ~(((r >= 300) & (r < 600)) | ((c >= 300) & (c < 600)))
    r, c = r[keep], c[keep]
    rc = np.unique(np.stack([r, c], 1), axis=0)
    r, c = rc[:, 0], rc[:, 1]
    h = csb_from_coo(n, r, c, rng.standard_normal(len(r)), [0, 256, 512, 768, n], groups=np.arange(0, n + 1, 100))
    for m in (1, 7):
        y = check(h, m)
        assert not y[300:600].any()


@pytest.mark.parametrize("n", [1, 2, 3, 5, 9, 67, 129])
def test_tiny_and_ragged_dimensions(n):
    rng = np.random.default_rng(n)
    r, c = np.tril_indices(n)
    keep = (rng.random(len(r)) < 0.5) | (r == c)
    h = csb_from_coo(n, r[keep], c[keep], rng.standard_normal(keep.sum()), [0, n], precision=0)
    for m in (1, 2, 3, 17):
        check(h, m)


def test_zero_width_block():
    h = gen_from((2000, 4, 64, 0.1, 0.5, 11, 1, 500))
    assert ci.DeviceMatrix(h).spmm_host(np.zeros((h.dim, 0))).shape == (h.dim, 0)


def test_matrix_assembled_by_the_reference(golden):
    """The 4He Nmax-4 Hamiltonian assembled by the reference
    (build_synthetic_problem): its own CSB block plan and small groups."""
    g = golden("multilevel")
    h = ci.CsbMatrix(dim=int(g["sub_block_boundaries"][-1]), precision=int(g["sub_precision"]),
                     block_boundaries=g["sub_block_boundaries"].astype(np.uint32),
                     entry_offsets=g["sub_entry_offsets"].astype(np.uint64), rows=g["sub_rows"], cols=g["sub_cols"],
                     values=g["sub_values"], groups=g["sub_groups"].astype(np.uint32))
    for m in (1, 8, 16, 24):
        check(h, m, seed=m)


@pytest.mark.parametrize("te", [64, 128])
def test_forced_tile_edges_fp32(te):
    h = gen_from((3072, 3, 256, 0.2, 0.4, 13, 0, 2000))
    dm = ci.DeviceMatrix(h, tile_edge=te)
    assert dm.tile_edge == te
    check(h, 16, tile_edge=te)


def test_fp32_subnormal_and_extreme_values():
    """fp32 values are promoted exactly (subnormals included) and products
    are formed in fp64: tiny and huge entries survive as in the reference."""
    n = 512
    r = np.arange(n)
    c = np.arange(n)
    v = np.full(n, 1.0, dtype=np.float32)
    v[:100] = np.float32(1e-40)      # fp32 subnormal
    v[100:200] = np.float32(3e38)    # near fp32 max
    v[200:300] = np.float32(-1.17549435e-38)  # smallest normal
    h = csb_from_coo(n, r, c, v, [0, n], precision=0)
    x = np.ones((n, 2))
    y = ci.DeviceMatrix(h).spmm_host(x)
    np.testing.assert_array_equal(y[:, 0], v.astype(np.float64))
    # off-diagonal coupling of a subnormal: exact in fp64
    h2 = csb_from_coo(4, np.array([0, 1, 2, 3, 3]), np.array([0, 0, 2, 3, 1]),
                      np.array([1.0, 1e-40, 2.0, 3.0, -2.5], dtype=np.float32), [0, 4], precision=0)
    check(h2, 3)
