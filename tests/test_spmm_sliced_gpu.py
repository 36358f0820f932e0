"""The integer-slice K1 (CIEG_SPMM_SLICED, csrc/spmm_i8.cu: Ozaki slices on
the tcgen05 int8 tensor cores) against the reference's spmm / the oracle:
1e-13 relative at every width, under wide dynamic ranges of X (per-panel
exponents) and of H (per-row exponents), zero columns, Inf/NaN inputs, the
diagonal tiles and ragged sector tails, deterministic run to run; plus the
fall-back when H holds non-finite values, and LOBPCG parity in this mode."""
import numpy as np
import pytest

from conftest import gen_from
from oracle import ci_oracle as O
from paper_1609_01689_b200 import ci, configs

pytestmark = pytest.mark.gpu

TOL = 1e-13


def rel_cols(a, b):
    """max over columns of max|a - b| / max|b| (column-wise scale)."""
    s = np.maximum(np.abs(b).max(axis=0), 1e-300)
    return float((np.abs(a - b).max(axis=0) / s).max())


@pytest.fixture(scope="module")
def sliced():
    dev = ci.Device.default()
    dev.set_spmm_mode("sliced")
    yield dev
    dev.set_spmm_mode("auto")


# fp32 H, 256-row generator tiles -> 128-row panels (two per tile, sector tails)
MATS = [(30000, 3, 256, 0.02, 0.4, 77, 0, 2000), (12000, 4, 200, 0.08, 0.4, 5, 0, 2000),
        (9000, 3, 128, 0.1, 0.5, 9, 0, 2000)]


@pytest.mark.parametrize("params", MATS)
@pytest.mark.parametrize("m", [1, 3, 8, 9, 16, 24, 32])
def test_sliced_matches_reference(sliced, ref_lib, params, m):
    h = gen_from(params)
    x = ci.random_block(h.dim, m, 100 + m)
    y_ref = ref_lib.RefMatrix(h).spmm(x, serial=True)
    y = ci.spmm(h, x)
    assert rel_cols(y, y_ref) < TOL
    assert np.array_equal(ci.spmm(h, x), y)  # deterministic


def _with_values(h, vals):
    return ci.CsbMatrix(dim=h.dim, precision=0, block_boundaries=h.block_boundaries, entry_offsets=h.entry_offsets,
                        rows=h.rows, cols=h.cols, values=vals, groups=h.groups, beta=h.beta)


def _global_rc(h):
    nb = h.block_count()
    bi = np.concatenate([np.full(i + 1, i) for i in range(nb)])
    bj = np.concatenate([np.arange(i + 1) for i in range(nb)])
    counts = np.diff(h.entry_offsets.astype(np.int64))
    r = h.block_boundaries[np.repeat(bi, counts)].astype(np.int64) + h.rows
    c = h.block_boundaries[np.repeat(bj, counts)].astype(np.int64) + h.cols
    return r, c


def test_sliced_dynamic_range_of_x(sliced, ref_lib):
    """X digits are scaled per 128-row panel and column: panels of X spanning
    1e-150 .. 1e150 (and zero columns) keep every output accurate entrywise
    against |H| |x|."""
    h = gen_from(MATS[0])
    rng = np.random.default_rng(3)
    x = ci.random_block(h.dim, 16, 9)
    g = h.groups.astype(np.int64)
    for a0, a1 in zip(g[:-1], g[1:]):  # generator tiles are unions of device panels
        x[a0:a1] *= 10.0 ** rng.integers(-150, 150)
    x[:, 5] = 0.0
    y = ci.spmm(h, x)
    y_ref = ref_lib.RefMatrix(h).spmm(x, serial=True)
    mag = ref_lib.RefMatrix(_with_values(h, np.abs(h.values))).spmm(np.abs(x), serial=True)
    assert np.all(y[:, 5] == 0.0)
    assert np.all(np.abs(y - y_ref) <= 1e-13 * mag)


def test_sliced_dynamic_range_of_h(sliced, ref_lib):
    """H slices are scaled per row (the largest off-diagonal |h| touching
    the row): a symmetric scaling D H D, d in 1e-2 .. 1e2, stays within
    1e-12 of the row scale -- |err_r| <= 1e-12 max_c |h_rc| sum_c |x_c|
    (the bound of a 40-bit row-scaled representation; entries above 2^-16
    of their row maximum are exact)."""
    h = gen_from(MATS[0])
    rng = np.random.default_rng(4)
    d = 10.0 ** rng.uniform(-2, 2, size=h.dim)
    r, c = _global_rc(h)
    vals = (h.values.astype(np.float64) * d[r] * d[c]).astype(np.float32)
    hs = _with_values(h, vals)
    x = ci.random_block(h.dim, 16, 4)
    y = ci.spmm(hs, x)
    y_ref = ref_lib.RefMatrix(hs).spmm(x, serial=True)
    off = r != c
    rowmax = np.zeros(h.dim)
    np.maximum.at(rowmax, r[off], np.abs(vals[off]).astype(np.float64))
    np.maximum.at(rowmax, c[off], np.abs(vals[off]).astype(np.float64))
    ones = np.where(off, 1.0, 0.0).astype(np.float32)
    pat = ref_lib.RefMatrix(_with_values(h, ones)).spmm(np.abs(x), serial=True)
    diag_terms = np.zeros(h.dim)
    diag_terms[r[~off]] = np.abs(vals[~off])
    err = np.abs(y - y_ref)
    assert np.all(err <= 1e-12 * rowmax[:, None] * pat + 1e-15 * diag_terms[:, None] * np.abs(x))


def test_sliced_nonfinite_x_matches_reference(sliced, ref_lib):
    h = gen_from(MATS[1])
    x = ci.random_block(h.dim, 12, 8)
    x[17, 3] = np.inf
    x[4000, 0] = -np.inf
    x[9000, 7] = np.nan
    y_ref = ref_lib.RefMatrix(h).spmm(x, serial=True)
    y = ci.spmm(h, x)
    assert np.array_equal(np.isnan(y), np.isnan(y_ref))
    assert np.array_equal(np.isposinf(y), np.isposinf(y_ref))
    assert np.array_equal(np.isneginf(y), np.isneginf(y_ref))
    fin = np.isfinite(y_ref)
    assert np.abs(y[fin] - y_ref[fin]).max() <= 1e-13 * np.abs(y_ref[fin]).max()


def test_sliced_nonfinite_h_falls_back_to_dmma(sliced, ref_lib):
    """Inf/NaN stored values cannot be sliced: the matrix runs the fp64 DMMA
    single pass instead (still on the GPU) and matches the reference."""
    h = gen_from(MATS[2])
    vals = h.values.copy()
    vals[1234] = np.inf
    hb = ci.CsbMatrix(dim=h.dim, precision=0, block_boundaries=h.block_boundaries, entry_offsets=h.entry_offsets,
                      rows=h.rows, cols=h.cols, values=vals, groups=h.groups, beta=h.beta)
    x = ci.random_block(h.dim, 16, 2)
    y_ref = ref_lib.RefMatrix(hb).spmm(x, serial=True)
    y = ci.spmm(hb, x)
    assert np.array_equal(np.isnan(y), np.isnan(y_ref))
    fin = np.isfinite(y_ref)
    assert np.abs(y[fin] - y_ref[fin]).max() <= 1e-13 * np.abs(y_ref[fin]).max()


def test_sliced_config2_properties(sliced):
    """BASELINE config 2 (n = 2e6, S = 8e8) at m = 16: linearity and
    u^T (H v) = v^T (H u) at full size, and agreement with the fp64 DMMA
    owner-computes kernel to 1e-13."""
    dm = configs.CFG2.generate_device()
    x = ci.random_block(dm.dim, 16, 1)
    z = ci.random_block(dm.dim, 16, 2)
    y = dm.spmm_host(x)
    yz = dm.spmm_host(z)
    assert rel_cols(dm.spmm_host(0.5 * x - 2.0 * z), 0.5 * y - 2.0 * yz) < 1e-13
    assert abs(float(z[:, 0] @ y[:, 0]) - float(x[:, 0] @ yz[:, 0])) < 1e-11 * abs(float(z[:, 0] @ y[:, 0]))
    dev = ci.Device.default()
    dev.set_spmm_mode("owner")
    try:
        y_dmma = dm.spmm_host(x)
    finally:
        dev.set_spmm_mode("sliced")
    assert rel_cols(y, y_dmma) < TOL


def test_sliced_lobpcg_matches_reference(sliced, ref_lib):
    """The config-4 settings (kt 16, k 8, fp32 H, 256-row tiles, FOM/LU tile
    preconditioner) with every SpMM on the int8 tensor cores: identical
    iteration count, counters and active sets to ci::lobpcg_solve."""
    cfg = configs.Config("cfg4-shape", 25 * 2368, 25, 256, None, 0.4, 0, 25 * 2368 * 400, k_want=8, kt=16,
                         tol=1e-6, seed=3)
    h = cfg.generate()
    x0 = ci.random_block(h.dim, 16, 42)
    rm = ref_lib.RefMatrix(h)
    rr = ref_lib.lobpcg_solve(rm, x0, 8, 1e-6, 500, ref_lib.RefTileDiagonal(rm, h.groups))
    rep = ci.lobpcg_solve(h, x0, ci.LobpcgOptions(k_want=8, tol=1e-6, preconditioner=ci.extract_tile_diagonal(h)))
    assert rep.iterations == rr.iterations and rep.converged == rr.converged
    assert [rep.counters.spmm_calls, rep.counters.spmv_equivalents, rep.counters.precond_applications,
            rep.counters.orthogonalizations] == rr.counters.tolist()
    np.testing.assert_allclose(rep.eigenvalues, rr.eigenvalues, rtol=1e-9)


# ---- the chunk-pipelined host call (cieg_spmm_host on the sliced kernel)

def _device_spmm(dm, x):
    """One-launch sliced SpMM on device-resident X (cieg_spmm)."""
    import torch

    xd = torch.from_numpy(x).cuda()
    yd = torch.empty_like(xd)
    torch.cuda.synchronize()
    dm.spmm_ptr(xd.data_ptr(), yd.data_ptr(), x.shape[1])
    dm.device.synchronize()
    return yd.cpu().numpy()


@pytest.mark.parametrize("chunks", [1, 2, 5, 12, 40])
@pytest.mark.parametrize("m", [1, 7, 16])
def test_host_pipeline_bitwise(sliced, ref_lib, monkeypatch, chunks, m):
    """Upload, kernels and download pipelined over row chunks: bitwise the
    one-launch result at every chunk count (the fixed-point accumulation does
    not depend on the order of the additions), pageable and pinned buffers."""
    import torch

    h = gen_from((40000, 10, 256, 0.02, 0.4, 21, 0, 2000))
    dm = ci.device_matrix(h)
    x = ci.random_block(h.dim, m, 300 + m)
    y_one = _device_spmm(dm, x)
    assert rel_cols(y_one, ref_lib.RefMatrix(h).spmm(x, serial=True)) < TOL
    monkeypatch.setenv("CIEG_HOST_CHUNKS", str(chunks))
    assert np.array_equal(dm.spmm_host(x), y_one)
    xp = torch.from_numpy(x).pin_memory()
    yp = torch.empty_like(xp).pin_memory()
    ci._check(ci._lib.load().cieg_spmm_host(dm.device.handle, dm.handle, ci._ptr(xp.numpy()), ci._ptr(yp.numpy()), m))
    assert np.array_equal(yp.numpy(), y_one)


def test_host_pipeline_nonfinite_and_tiny(sliced, ref_lib, monkeypatch):
    """Inf/NaN rows of X (fixed up after the pipeline, U downloaded again) and
    the tiny-entry terms added per converted row range."""
    h = gen_from((40000, 10, 256, 0.02, 0.4, 22, 0, 2000))
    vals = h.values.copy()
    vals[::1000] *= 2.0 ** -30  # entries too small for their row's slices: the fp64 tiny list
    h2 = _with_values(h, vals)
    dm = ci.DeviceMatrix(h2)
    x = ci.random_block(h.dim, 16, 17)
    monkeypatch.setenv("CIEG_HOST_CHUNKS", "9")
    y = dm.spmm_host(x)
    y_ref = ref_lib.RefMatrix(h2).spmm(x, serial=True)
    assert rel_cols(y, y_ref) < TOL
    assert np.array_equal(y, _device_spmm(dm, x))
    x[123, 3] = np.inf
    x[30000, 0] = np.nan
    y = dm.spmm_host(x)
    y_ref = ref_lib.RefMatrix(h2).spmm(x, serial=True)
    assert np.array_equal(np.isnan(y), np.isnan(y_ref)) and np.array_equal(np.isinf(y), np.isinf(y_ref))
    fin = np.isfinite(y_ref)
    assert np.abs(y[fin] - y_ref[fin]).max() <= TOL * np.abs(y_ref[fin]).max()


def test_host_pipeline_unbanded(sliced, ref_lib, monkeypatch):
    """A matrix whose last panel couples to the first (two sectors, band
    covering both): no panel is final before the last owner ran; the pipeline
    degenerates to upload, compute, download."""
    h = gen_from((6000, 2, 128, 0.1, 0.5, 4, 0, 2000))
    dm = ci.device_matrix(h)
    x = ci.random_block(h.dim, 16, 5)
    monkeypatch.setenv("CIEG_HOST_CHUNKS", "6")
    y = dm.spmm_host(x)
    assert np.array_equal(y, _device_spmm(dm, x))
    assert rel_cols(y, ref_lib.RefMatrix(h).spmm(x, serial=True)) < TOL


def test_sliced_full_lowest_slice(sliced, ref_lib):
    """The lowest H slice is streamed as a per-item sparse list (at most 512
    entries per tile). Values spread over 14 binades within every row fill
    that slice for about half the entries -- far more than the list holds --
    so this matrix keeps five dense planes; same result either way."""
    h = gen_from((12000, 4, 200, 0.08, 0.4, 5, 0, 2000))
    rng = np.random.default_rng(11)
    mag = np.exp2(-rng.integers(0, 15, h.values.size)).astype(np.float32)
    vals = (np.sign(h.values) * mag * np.float32(0.01)).astype(np.float32)
    vals[h.values == 0] = 0
    h2 = _with_values(h, vals)
    x = ci.random_block(h.dim, 16, 23)
    y = ci.spmm(h2, x)
    y_ref = ref_lib.RefMatrix(h2).spmm(x, serial=True)
    assert rel_cols(y, y_ref) < TOL
    assert np.array_equal(ci.spmm(h2, x), y)


def test_sliced_sparse_and_dense_lowest_slice_agree(tmp_path):
    """CIEG_SLICED_DENSE5=1 (five dense planes) and the default (sparse lowest
    slice) run the same arithmetic: bitwise equal results."""
    import subprocess, sys, os

    script = tmp_path / "run.py"
    script.write_text(
        "import sys, numpy as np\n"
        "sys.path.insert(0, %r)\n"
        "from paper_1609_01689_b200 import ci\n"
        "h = ci.generate_sector_matrix(20000, 5, 256, 0.03, 0.4, 31, 0, 2000)\n"
        "ci.Device.default().set_spmm_mode('sliced')\n"
        "x = ci.random_block(h.dim, 16, 3)\n"
        "np.save(sys.argv[1], ci.spmm(h, x))\n" % os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    outs = []
    for dense5 in ("0", "1"):
        out = tmp_path / f"y{dense5}.npy"
        env = dict(os.environ, CIEG_SLICED_DENSE5=dense5)
        subprocess.run([sys.executable, str(script), str(out)], check=True, env=env, timeout=300)
        outs.append(np.load(out))
    assert np.array_equal(outs[0], outs[1])
