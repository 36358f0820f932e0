"""CPU suite: pins the numpy oracle (oracle/ci_oracle.py) and the host-side
library logic against the golden fixtures produced by the UNMODIFIED
reference (tests/golden/make_golden.py) and against the SPEC.md known answers.
No GPU needed."""
import numpy as np
import pytest

from conftest import gen_from
from oracle import ci_oracle as O
from paper_1609_01689_b200 import ci


# ------------------------------------------------------------------ generator

@pytest.mark.parametrize("precision", [0, 1])
def test_generator_port_is_bitwise(precision):
    """C++ generator == numpy restatement (small case; the port is slow)."""
    a = ci.generate_sector_matrix(384, 2, 64, 0.3, 0.5, seed=9, precision=precision, beta=256)
    b = O.generate(384, 2, 64, 0.3, 0.5, 9, precision, beta=256)
    for f in ("block_boundaries", "entry_offsets", "rows", "cols", "values", "groups"):
        assert np.array_equal(getattr(a, f), getattr(b, f)), f


def test_generator_digests_are_pinned(golden):
    """Deterministic across builds/platforms: the SHA-256 of the generated
    arrays matches the fixture (generated next to the reference)."""
    import hashlib

    g = golden("spmm")
    for name in ("f64", "f32", "f32_t256"):
        h = gen_from(g[f"gen_{name}_params"])
        m = hashlib.sha256()
        for a in (h.block_boundaries, h.entry_offsets, h.rows, h.cols, h.values, h.groups):
            m.update(np.ascontiguousarray(a).tobytes())
        assert m.hexdigest() == str(g[f"gen_{name}_digest"])
        assert h.nnz_lower == int(g[f"gen_{name}_nnz"])


def test_generator_structure_invariants():
    """CSB invariants the reference's spmm relies on (csb.hpp:22-60): lower
    triangle, u16 offsets below the block extents, entries sorted by (r, c)
    per block, blocks cut at sector boundaries, one diagonal entry per row."""
    n, sectors = 6000, 3
    h = ci.generate_sector_matrix(n, sectors, 64, 0.08, 0.5, seed=4, precision=0, beta=1500)
    bb = h.block_boundaries.astype(np.int64)
    for s in range(1, sectors):
        assert (n * s) // sectors in set(bb.tolist())
    assert np.all(np.diff(bb) <= 1500) and bb[0] == 0 and bb[-1] == n
    r, c, v, ei, ej = O._global_entries(h)
    assert np.all(c <= r)
    assert np.all(h.rows.astype(np.int64) < (bb[ei + 1] - bb[ei]))
    assert np.all(h.cols.astype(np.int64) < (bb[ej + 1] - bb[ej]))
    offs = h.entry_offsets.astype(np.int64)
    key = h.rows.astype(np.int64) * 65536 + h.cols.astype(np.int64)
    for b in range(len(offs) - 1):
        assert np.all(np.diff(key[offs[b]:offs[b + 1]]) > 0)
    diag = r == c
    assert diag.sum() == n and np.array_equal(np.sort(r[diag]), np.arange(n))
    # diagonal d_i = 10 s_i + U(-2, 2)
    s_of = (r[diag] * sectors) // n
    assert np.all(np.abs(v[diag] - 10.0 * s_of) <= 2.0)
    # off-diagonal entries only between sectors |ds| <= 2
    sr, sc = (r * sectors) // n, (c * sectors) // n
    assert np.all(np.abs(sr - sc) <= 2)


def test_generator_expected_nnz():
    vals = [ci.generate_sector_matrix(20000, 10, 64, 0.05, 0.5, seed=s, precision=1).nnz_lower for s in range(1, 5)]
    e = ci.expected_nnz(20000, 10, 64, 0.05, 0.5)
    assert abs(np.mean(vals) - e) < 0.05 * e


def test_generator_rejects_bad_config():
    with pytest.raises(ci.ConfigError):
        ci.generate_sector_matrix(0, 1, 64, 0.1, 0.5)
    with pytest.raises(ci.BetaTooLarge):
        ci.generate_sector_matrix(1000, 1, 64, 0.1, 0.5, beta=70000)


def test_random_block_matches_reference_rule():
    a = ci.random_block(777, 9, 12345)
    assert np.array_equal(a, O.random_block(777, 9, 12345))
    assert a.min() >= -1.0 and a.max() < 1.0


# -------------------------------------------------- oracle vs reference golden

@pytest.mark.parametrize("name", ["f64", "f32", "f32_t256"])
@pytest.mark.parametrize("m", [1, 5, 16])
def test_oracle_spmm_bitwise(golden, name, m):
    g = golden("spmm")
    h = gen_from(g[f"gen_{name}_params"])
    x = ci.random_block(h.dim, m, 100 + m)
    assert np.array_equal(O.spmm(h, x), g[f"spmm_{name}_m{m}"])


def test_oracle_block_kernels_bitwise(golden):
    g = golden("blockvec")
    x = ci.random_block(1003, 24, 1)
    y = ci.random_block(1003, 20, 2)
    gg = 2.0 * ci.random_block(24, 16, 3)
    assert np.array_equal(O.block_inner(x, y), g["block_inner"])
    assert np.array_equal(O.linear_combination(x, gg), g["linear_combination"])
    assert np.array_equal(O.add_linear_combination(ci.random_block(1003, 16, 4), x, gg), g["add_linear_combination"])


def test_oracle_orthonormalize(golden):
    g = golden("blockvec")
    q = O.orthonormalize(ci.random_block(1003, 12, 5), 1e-8, ci.random_block(1003, 6, 6))
    assert q.shape == g["orthonormalize"].shape
    np.testing.assert_allclose(q, g["orthonormalize"], rtol=0, atol=1e-12)
    dup = ci.random_block(1003, 6, 7)
    dup = np.hstack([dup, dup[:, :2]])
    assert O.orthonormalize(dup).shape[1] == int(g["orthonormalize_dup_width"]) == 6


def _shift_cases(g):
    for c, (k, it, tol) in enumerate(g["cases"]):
        yield c, int(k), int(it), float(tol)


def test_oracle_choose_shifts_exact(golden):
    g = golden("shifts")
    for c, k, it, tol in _shift_cases(g):
        mu, en = O.choose_shifts(g[f"{c}_theta"], g[f"{c}_res_norm"], np.ones(k), g[f"{c}_relres"], it, tol)
        assert np.array_equal(mu, g[f"{c}_mu"]) and np.array_equal(en, g[f"{c}_engage"]), c


def test_library_choose_shifts_exact(golden):
    """The product's host choose_shifts (C ABI, CPU-callable) == reference."""
    g = golden("shifts")
    for c, k, it, tol in _shift_cases(g):
        plan = ci.choose_shifts(g[f"{c}_theta"], g[f"{c}_res_norm"], np.ones(k), g[f"{c}_relres"], it, tol)
        assert np.array_equal(plan.mu, g[f"{c}_mu"]) and np.array_equal(plan.engage, g[f"{c}_engage"]), c


@pytest.mark.parametrize("name", ["lu", "fom"])
def test_oracle_preconditioner(golden, name):
    g = golden("precond")
    h = gen_from(g[f"{name}_params"])
    tiles = O.extract_tile_diagonal(h, h.groups)
    r = ci.random_block(h.dim, 8, 31)
    w = O.apply_preconditioner(tiles, h.groups, r, g[f"{name}_mu"], g[f"{name}_engage"])
    np.testing.assert_allclose(w, g[f"{name}_w"], rtol=1e-9, atol=1e-12)
    assert np.array_equal(w[:, 5], r[:, 5])  # disengaged column passes through


@pytest.mark.parametrize("name", ["diag100", "sector_f64_prec"])
def test_oracle_lobpcg(golden, name):
    g = golden("lobpcg")
    k, kt, tol, pre, seed = g[f"{name}_meta"]
    if name == "diag100":
        n = 100
        h = ci.CsbMatrix(dim=n, precision=1, block_boundaries=np.array([0, n], np.uint32),
                         entry_offsets=np.array([0, n], np.uint64), rows=np.arange(n, dtype=np.uint16),
                         cols=np.arange(n, dtype=np.uint16), values=np.arange(1, n + 1, dtype=np.float64),
                         groups=np.array([0, 50, n], np.uint32))
    else:
        h = gen_from(g[f"{name}_params"])
    x0 = ci.random_block(h.dim, int(kt), int(seed))
    tiles = O.extract_tile_diagonal(h, h.groups) if pre else None
    r = O.lobpcg_solve(h, x0, int(k), float(tol), 500, tiles, h.groups)
    assert r.converged == bool(g[f"{name}_converged"])
    assert r.iterations == int(g[f"{name}_iterations"])
    assert r.counters == g[f"{name}_counters"].tolist()
    np.testing.assert_allclose(r.eigenvalues, g[f"{name}_eigenvalues"], rtol=1e-12)
    np.testing.assert_allclose(r.eigenvalues, g[f"{name}_dense_eigs"], rtol=1e-8)


def _diag100():
    n = 100
    return ci.CsbMatrix(dim=n, precision=1, block_boundaries=np.array([0, n], np.uint32),
                        entry_offsets=np.array([0, n], np.uint64), rows=np.arange(n, dtype=np.uint16),
                        cols=np.arange(n, dtype=np.uint16), values=np.arange(1, n + 1, dtype=np.float64),
                        groups=np.array([0, 50, n], np.uint32))


@pytest.mark.parametrize("name", ["diag100_restart", "sector_f64", "sector_f32"])
def test_oracle_lanczos(golden, name):
    """lanczos.cpp:24-136 restated in numpy vs the compiled reference: same
    step count, convergence, counters and per-checkpoint convergence pattern;
    Ritz values to 1e-10 relative (LAPACK vs Eigen tridiagonal QL), Ritz
    vectors to 1e-6 up to sign. diag100_restart exercises the breakdown restart."""
    g = golden("lanczos")
    k, tol, max_iter, _ = g[f"{name}_meta"]
    h = _diag100() if name.startswith("diag") else gen_from(g[f"{name}_params"])
    r = O.lanczos_solve(lambda x: O.spmm(h, x), g[f"{name}_v0"], int(k), float(tol), int(max_iter))
    assert r.converged == bool(g[f"{name}_converged"])
    assert r.iterations == int(g[f"{name}_iterations"])
    assert r.counters == g[f"{name}_counters"].tolist()
    hist = np.array([[it, rr > tol] for it, _, rr, _ in r.history])
    assert hist[:, 0].tolist() == g[f"{name}_hist_iter"].tolist()
    assert hist[:, 1].tolist() == (g[f"{name}_relres"] > tol).tolist()
    np.testing.assert_allclose([t for *_, t in r.history], g[f"{name}_theta"], rtol=1e-9, atol=1e-12)
    np.testing.assert_allclose(r.eigenvalues, g[f"{name}_eigenvalues"], rtol=1e-10)
    np.testing.assert_allclose(r.eigenvalues, g[f"{name}_dense_eigs"], rtol=1e-7)
    ov = np.abs(np.sum(r.trial_vectors * g[f"{name}_eigenvectors"], axis=0))
    np.testing.assert_allclose(ov, 1.0, atol=1e-6)


def test_oracle_multilevel_guess(golden):
    """guess.cpp:66-117 restated (leading blocks as the level problems) vs the
    reference's own multilevel_guess on 4He Nmax 6: same level dimensions,
    iteration counts and convergence; the guess spans the same columns."""
    from conftest import multilevel_operator

    g = golden("multilevel")
    h = multilevel_operator(g)
    guess, lv = O.multilevel_guess(h, g["level_dims"].tolist(), k_want=8, k_trial=12, tol=1e-6)
    assert [r[0] for r in lv] == g["level_dims"].tolist()
    assert [r[1] for r in lv] == g["level_iterations"].tolist()
    assert [r[2] for r in lv] == g["level_converged"].tolist()
    head = g["guess_head"]
    assert guess.shape == (h.dim, int(g["guess_width"]))
    assert np.all(guess[head.shape[0]:] == 0.0)
    ov = np.abs(np.sum(guess[: head.shape[0]] * head, axis=0))
    np.testing.assert_allclose(ov[:8], 1.0, atol=1e-8)
    np.testing.assert_allclose(ov, 1.0, atol=1e-4)


# ------------------------------------------------------- SPEC known answers

def test_spec_spmm_known_answers():
    """diagonal H -> U = d X; X = 0 -> U = 0; dense oracle."""
    n = 300
    d = np.linspace(-3, 5, n)
    h = ci.CsbMatrix(dim=n, precision=1, block_boundaries=np.array([0, n], np.uint32),
                     entry_offsets=np.array([0, n], np.uint64), rows=np.arange(n, dtype=np.uint16),
                     cols=np.arange(n, dtype=np.uint16), values=d.copy())
    x = ci.random_block(n, 4, 1)
    assert np.array_equal(O.spmm(h, x), d[:, None] * x)
    hs = ci.generate_sector_matrix(900, 3, 64, 0.2, 0.5, seed=1, precision=0, beta=300)
    assert not O.spmm(hs, np.zeros((900, 3))).any()
    x = ci.random_block(900, 12, 2)
    dense = O.to_dense(hs)
    u = O.spmm(hs, x)
    np.testing.assert_allclose(u, dense @ x, rtol=0, atol=1e-12 * np.abs(dense @ x).max())


def test_spec_fom_known_answers():
    """block = c I -> rhs/(c - mu) in one step; zero rhs -> 0."""
    n = 10
    rhs = np.random.default_rng(0).standard_normal((n, 3))
    rhs[:, 2] = 0.0
    x = O.fom_solve(4.0 * np.eye(n), [1.0, 2.0, 0.5], rhs, 1)
    np.testing.assert_allclose(x[:, 0], rhs[:, 0] / 3.0, rtol=1e-14)
    np.testing.assert_allclose(x[:, 1], rhs[:, 1] / 2.0, rtol=1e-14)
    assert not x[:, 2].any()


def test_spec_choose_shifts_examples():
    """SPEC.md:429-432."""
    mu, en = O.choose_shifts([-30.0, -29.0], [0.004, 0.01], [1.0, 1.0], [1e-4, 2e-3], 2, 1e-6)
    assert not en.any()
    mu, en = O.choose_shifts([-30.0, -29.0], [0.004, 0.01], [1.0, 1.0], [1e-4, 2e-3], 5, 1e-6)
    assert mu[0] == pytest.approx(-30.008) and en.all()
    mu, en = O.choose_shifts([-30.0], [5.0], [1.0], [0.5], 5, 1e-6)
    assert not en.any()


@pytest.mark.parametrize("prec,beta", [(0, 100), (1, 100), (0, 2000)])
def test_oracle_cpp_generator_matches_python_restatement(ref_lib, prec, beta):
    """oracle/ref_gen.cpp (the generator the reference arm and the CPU
    baselines build the reference's ci::CsbMatrix with) is bit for bit
    ci_oracle.generate, and its leading-block sample is the leading principal
    submatrix entry for entry."""
    o = O.generate(600, 3, 32, 0.3, 0.5, 7, prec, beta=beta)
    r = ref_lib.generate(600, 3, 32, 0.3, 0.5, 7, prec, beta=beta)
    assert r.nnz == int(o.entry_offsets[-1]) == ref_lib.count_nnz(600, 3, 32, 0.3, 0.5, 7)
    x = O.random_block(600, 3, 1)
    np.testing.assert_array_equal(r.spmm_dim(x), O.spmm(o, x))
    nb = r.nb_total
    lead = ref_lib.generate(600, 3, 32, 0.3, 0.5, 7, prec, beta=beta, nbk=nb // 2)
    d = lead.dim
    dense = O.to_dense(o)[:d, :d]
    xs = x[:d]
    np.testing.assert_allclose(lead.spmm_dim(xs), dense @ xs, rtol=1e-12, atol=1e-12)
    assert np.isclose(ref_lib.calibrated_p(600, 3, 32, 0.5, ref_lib.expected_nnz(600, 3, 32, 0.3, 0.5)), 0.3)
