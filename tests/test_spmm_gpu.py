"""K1 parity on the GPU: the CUDA SpMM (through the C ABI) against the
reference's spmm_serial (golden fixtures; live oracle/_ref when present), the
SPEC.md:229-242 properties, determinism, and size-independent properties at
the BASELINE config-2 scale."""
import numpy as np
import pytest

from conftest import gen_from
from oracle import ci_oracle as O
from paper_1609_01689_b200 import ci, configs

pytestmark = pytest.mark.gpu

# fp64 H: different summation order only -> ~1e-16 relative; fp32 H promoted
# exactly, fp64 accumulation -> same bound.
TOL = 1e-13


def rel(a, b):
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


@pytest.mark.parametrize("name", ["f64", "f32", "f32_t256"])
@pytest.mark.parametrize("m", [1, 5, 16])
def test_spmm_matches_reference_golden(golden, name, m):
    g = golden("spmm")
    h = gen_from(g[f"gen_{name}_params"])
    x = ci.random_block(h.dim, m, 100 + m)
    assert rel(ci.spmm(h, x), g[f"spmm_{name}_m{m}"]) < TOL


@pytest.mark.parametrize("m", [1, 2, 4, 7, 8, 13, 16, 17, 32, 48, 64])
def test_spmm_block_widths(m):
    """Config-1 matrix (fp64, 64-row tiles) at every LOBPCG width and the
    config-3 sweep widths."""
    h = configs.CFG1.generate()
    x = ci.random_block(h.dim, m, 7 + m)
    assert rel(ci.spmm(h, x), O.spmm(h, x)) < TOL


def test_spmm_live_reference(ref_lib):
    h = gen_from((30000, 3, 256, 0.02, 0.4, 77, 0, 2000))
    x = ci.random_block(h.dim, 16, 3)
    assert rel(ci.spmm(h, x), ref_lib.RefMatrix(h).spmm(x, serial=True)) < TOL


def test_spmm_diagonal_and_zero():
    n = 1000
    d = np.linspace(-2, 7, n)
    h = ci.CsbMatrix(dim=n, precision=1, block_boundaries=np.array([0, 500, n], np.uint32),
                     entry_offsets=np.array([0, 500, 500, n], np.uint64),
                     rows=np.concatenate([np.arange(500), np.arange(500)]).astype(np.uint16),
                     cols=np.concatenate([np.arange(500), np.arange(500)]).astype(np.uint16), values=d.copy())
    x = ci.random_block(n, 6, 1)
    assert np.array_equal(ci.spmm(h, x), d[:, None] * x)
    hs = configs.CFG1.generate()
    assert not ci.spmm(hs, np.zeros((hs.dim, 4))).any()


def test_spmm_linearity_symmetry_and_columns():
    """linearity, u^T(Hv) = v^T(Hu), width-k == k width-1
    products, deterministic run to run (bitwise)."""
    h = gen_from((20000, 4, 64, 0.05, 0.5, 5, 0, 2000))
    x = ci.random_block(h.dim, 8, 1)
    y = ci.random_block(h.dim, 8, 2)
    a, b = 0.75, -1.5
    lhs = ci.spmm(h, a * x + b * y)
    rhs = a * ci.spmm(h, x) + b * ci.spmm(h, y)
    assert rel(lhs, rhs) < 1e-12
    u, v = x[:, :1], y[:, :1]
    s1 = float(u[:, 0] @ ci.spmm(h, v)[:, 0])
    s2 = float(v[:, 0] @ ci.spmm(h, u)[:, 0])
    assert abs(s1 - s2) <= 1e-12 * abs(s1)
    full = ci.spmm(h, x)
    assert np.array_equal(ci.spmm(h, x), full)
    # auto mode picks the kernel per width (scalar single pass at m <= 2,
    # DMMA single pass at 3..8): columns agree to rounding across widths
    for j in range(8):
        assert rel(ci.spmm(h, x[:, j:j + 1])[:, 0], full[:, j]) < 1e-14
    # exact column independence at a fixed accumulation order --
    # owner-computes has one order for every width
    dev = ci.Device.default()
    dev.set_spmm_mode("owner")
    try:
        full_o = ci.spmm(h, x)
        for j in range(8):
            assert np.array_equal(ci.spmm(h, x[:, j:j + 1])[:, 0], full_o[:, j])
        wide = np.hstack([x, y])
        assert np.array_equal(ci.spmm(h, wide)[:, :8], full_o)
    finally:
        dev.set_spmm_mode("auto")


def test_spmm_dimension_mismatch():
    h = configs.CFG1.generate()
    with pytest.raises(ci.DimensionMismatch):
        ci.spmm(h, np.zeros((h.dim + 1, 2)))


def test_spmm_small_groups_merge_into_panels():
    """Physics-style small groups (the 6Li-like partition) are merged into
    <= 64/128-row panels; result unchanged."""
    h = gen_from((2000, 2, 64, 0.2, 0.5, 8, 1, 500))
    rng = np.random.default_rng(0)
    cuts = np.unique(np.concatenate([[0, 2000], rng.integers(1, 2000, 300)])).astype(np.uint32)
    h.groups = cuts
    x = ci.random_block(h.dim, 8, 2)
    assert rel(ci.DeviceMatrix(h).spmm_host(x), O.spmm(h, x)) < TOL


@pytest.mark.slow
def test_spmm_config2_scale_properties():
    """BASELINE config 2 (n = 2e6, ~0.8e9 stored nnz, m = 16): oracle-free,
    size-independent checks -- symmetry of the bilinear form, linearity, the
    exact diagonal contribution, bitwise determinism -- plus exact parity on
    a row sample against a CPU product restricted to those rows."""
    h = configs.CFG2.generate()
    dm = ci.DeviceMatrix(h)
    x = ci.random_block(h.dim, 16, 1)
    y = ci.random_block(h.dim, 16, 2)
    hx = dm.spmm_host(x)
    assert np.array_equal(hx, dm.spmm_host(x))
    hy = dm.spmm_host(y)
    s1 = np.einsum("ij,ij->j", y, hx)
    s2 = np.einsum("ij,ij->j", x, hy)
    assert np.abs(s1 - s2).max() <= 1e-11 * np.abs(s1).max()
    assert rel(dm.spmm_host(x + 2.0 * y), hx + 2.0 * hy) < 1e-12
    # row sample: U[rows] from the stored entries touching those rows
    rows = [0, 1, 99_999, 100_000, 1_234_567, h.dim - 1]
    want = np.array([_row_product(h, row, x) for row in rows])
    assert rel(hx[rows], want) < 1e-12


def _row_product(h, row, x):
    """(H X)[row] from the CSB blocks: row part from block row B(row), the
    transposed part from block column B(row) (the reference's two phases)."""
    bb = h.block_boundaries.astype(np.int64)
    offs = h.entry_offsets.astype(np.int64)
    b = int(np.searchsorted(bb, row, side="right") - 1)
    loc = row - bb[b]
    out = np.zeros(x.shape[1])
    for j in range(b + 1):  # phase one: blocks (b, j)
        k = b * (b + 1) // 2 + j
        e0, e1 = offs[k], offs[k + 1]
        sel = np.nonzero(h.rows[e0:e1] == loc)[0] + e0
        out += (h.values[sel].astype(np.float64)[:, None] * x[bb[j] + h.cols[sel].astype(np.int64)]).sum(0)
    for i in range(b, len(bb) - 1):  # phase two: blocks (i, b), strict on the diagonal
        k = i * (i + 1) // 2 + b
        e0, e1 = offs[k], offs[k + 1]
        m = h.cols[e0:e1] == loc
        if i == b:
            m &= h.rows[e0:e1] != loc
        sel = np.nonzero(m)[0] + e0
        out += (h.values[sel].astype(np.float64)[:, None] * x[bb[i] + h.rows[sel].astype(np.int64)]).sum(0)
    return out


def test_spmm_host_batch_matches_single_calls():
    """cieg_spmm_host_batch (pipelined copies) = cieg_spmm_host per product, bitwise."""
    h = gen_from((3072, 3, 256, 0.2, 0.4, 13, 0, 2000))
    dm = ci.DeviceMatrix(h)
    xs = [ci.random_block(h.dim, 16, s) for s in range(5)]
    ys = dm.spmm_host_batch(xs)
    for x, y in zip(xs, ys):
        assert np.array_equal(y, dm.spmm_host(x))
    assert dm.spmm_host_batch([]) == []


@pytest.mark.parametrize("prec", [0, 1])
@pytest.mark.parametrize("m", [1, 4, 16, 20])
def test_spmm_nonfinite_inputs_match_reference(prec, m):
    """Inf / NaN in X: the dense tile's explicit zeros must not turn into
    NaN (0 * Inf); only stored entries multiply, as in spmm (csb.cpp:118-193).
    Same non-finite pattern (NaN / +Inf / -Inf per element) as the oracle's
    sequential restatement, finite elements to rounding."""
    from oracle import ci_oracle as O

    h = gen_from((3072, 3, 256, 0.2, 0.4, 13, prec, 2000)) if prec == 0 else gen_from((2000, 4, 64, 0.1, 0.5, 11, 1, 500))
    x = ci.random_block(h.dim, m, 3)
    x[100, 0] = np.inf
    x[777, m - 1] = -np.inf
    x[1500, m // 2] = np.nan
    y = ci.spmm(h, x)
    yo = O.spmm(h, x)
    for mask in (np.isnan, np.isposinf, np.isneginf):
        assert np.array_equal(mask(y), mask(yo))
    fin = np.isfinite(yo)
    np.testing.assert_allclose(y[fin], yo[fin], rtol=1e-12, atol=1e-12)
    # finite inputs afterwards: the flag is per launch
    x2 = ci.random_block(h.dim, m, 4)
    np.testing.assert_allclose(ci.spmm(h, x2), O.spmm(h, x2), rtol=1e-12, atol=1e-12)


def test_spmm_nonfinite_on_a_shard():
    from oracle import ci_oracle as O

    h = gen_from((3072, 3, 256, 0.2, 0.4, 13, 0, 2000))
    x = ci.random_block(h.dim, 8, 5)
    x[1030, 2] = np.inf  # a halo row of the second shard's neighbour
    x[2100, 5] = np.nan
    yo = O.spmm(h, x)
    from paper_1609_01689_b200 import dist as D

    rb, hl, hh = D.row_partition(h, 2)
    for r in range(2):
        dm = ci.DeviceMatrix.__new__(ci.DeviceMatrix)
        import ctypes as C

        from paper_1609_01689_b200 import _lib

        lib = _lib.load()
        v = h.view()
        g = np.ascontiguousarray(h.groups, dtype=np.uint32)
        handle = C.c_void_p()
        ci._check(lib.cieg_matrix_upload_shard(ci.Device.default().handle, C.byref(v), ci._ptr(g, C.c_uint32),
                                               len(g) - 1, 0, int(rb[r]), int(rb[r + 1]), C.byref(handle)))
        dm = ci.DeviceMatrix(None, ci.Device.default(), _handle=handle)
        y = dm.spmm_host(x)
        ref = yo[rb[r]:rb[r + 1]]
        for mask in (np.isnan, np.isposinf, np.isneginf):
            assert np.array_equal(mask(y), mask(ref))
        fin = np.isfinite(ref)
        np.testing.assert_allclose(y[fin], ref[fin], rtol=1e-12, atol=1e-12)


# ---------------------------------------------------------------- K1 modes
# Single pass (one item per stored tile, H·X and Hᵀ·X from the same shared
# tile, transposed half through per-tile partials) and owner-computes must
# both match the oracle at every width and tile shape, and stay bitwise
# deterministic run to run.
_MODE_MATS = {
    "f64_t64": (20_000, 10, 64, 0.05, 0.5, 1, 1, 2000),
    "f32_t128": (30_000, 3, 256, 0.02, 0.4, 77, 0, 2000),
    "f32_t64": (20_000, 4, 64, 0.05, 0.5, 5, 0, 2000),
}


@pytest.fixture
def spmm_mode():
    dev = ci.Device.default()
    yield dev.set_spmm_mode
    dev.set_spmm_mode("auto")


@pytest.mark.parametrize("mode", ["single", "owner"])
@pytest.mark.parametrize("mat", list(_MODE_MATS))
@pytest.mark.parametrize("m", [1, 2, 3, 8, 9, 16, 24])
def test_spmm_modes_match_reference(spmm_mode, mode, mat, m):
    spmm_mode(mode)
    h = gen_from(_MODE_MATS[mat])
    dm = ci.DeviceMatrix(h)
    x = ci.random_block(h.dim, m, 40 + m)
    y = dm.spmm_host(x)
    assert rel(y, O.spmm(h, x)) < TOL
    assert np.array_equal(y, dm.spmm_host(x))


def test_spmm_single_pass_equals_owner_to_rounding(spmm_mode):
    """The two modes sum in different orders: equal to ~1e-16, and each
    column independent of the block width."""
    h = gen_from(_MODE_MATS["f32_t128"])
    dm = ci.DeviceMatrix(h)
    x = ci.random_block(h.dim, 8, 9)
    spmm_mode("single")
    ys = dm.spmm_host(x)
    for b in range(2):  # DMMA single pass (m >= 3): one accumulation order, bitwise
        assert np.array_equal(dm.spmm_host(x[:, 4 * b:4 * b + 4]), ys[:, 4 * b:4 * b + 4])
    for j in range(8):  # the scalar single pass (m = 1): to rounding
        assert rel(dm.spmm_host(x[:, j:j + 1])[:, 0], ys[:, j]) < 1e-14
    spmm_mode("owner")
    yo = dm.spmm_host(x)
    assert rel(ys, yo) < TOL


@pytest.mark.parametrize("mode", ["single", "owner"])
def test_spmm_modes_generated_and_leading_view(spmm_mode, mode):
    """Device-generated matrix (cieg_generate_device) and a leading-block
    view (own schedules over the parent's tile stream) in both modes."""
    spmm_mode(mode)
    p = _MODE_MATS["f32_t128"]
    dm = ci.DeviceMatrix.generate(p[0], p[1], p[2], p[3], p[4], p[5], p[6], p[7])
    h = gen_from(p)
    x = ci.random_block(h.dim, 5, 2)
    assert rel(dm.spmm_host(x), O.spmm(h, x)) < TOL
    hc = gen_from(p)
    dmc = ci.DeviceMatrix(hc, cuts=[12_288])
    lead = dmc.leading(12_288)
    xl = ci.random_block(12_288, 4, 3)
    full = np.zeros((h.dim, 4))
    full[:12_288] = xl
    assert rel(lead.spmm_host(xl), O.spmm(h, full)[:12_288]) < TOL


@pytest.mark.parametrize("m", [2, 16])
def test_spmm_single_pass_nonfinite(spmm_mode, m):
    """Inf / NaN in X under single pass: the owner slab (transposed half) is
    sanitised like the partner slab and the exact terms added afterwards."""
    spmm_mode("single")
    h = gen_from((3072, 3, 256, 0.2, 0.4, 13, 0, 2000))
    x = ci.random_block(h.dim, m, 3)
    x[100, 0] = np.inf
    x[777, m - 1] = -np.inf
    x[1500, m // 2] = np.nan
    y = ci.spmm(h, x)
    yo = O.spmm(h, x)
    for mask in (np.isnan, np.isposinf, np.isneginf):
        assert np.array_equal(mask(y), mask(yo))
    fin = np.isfinite(yo)
    np.testing.assert_allclose(y[fin], yo[fin], rtol=1e-12, atol=1e-12)


def test_spmm_mode_rejects_unknown():
    with pytest.raises(ValueError):
        ci.Device.default().set_spmm_mode("fast")
