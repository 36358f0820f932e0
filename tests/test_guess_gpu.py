"""Starting blocks and the public lobpcg.hpp helpers on the GPU:
multilevel_guess (guess.cpp:66-117) over leading-block views of the resident
H vs the reference's own multilevel_guess (golden fixture from 4He Nmax 6,
and live where oracle/_ref is built); orthonormalize / rayleigh_ritz /
residual_norms vs the reference; leading views; BVEC files."""
import os
import tempfile

import numpy as np
import pytest

from conftest import gen_from, multilevel_operator
from paper_1609_01689_b200 import ci

pytestmark = pytest.mark.gpu


def check_guess(guess, head, width, dim):
    assert guess.shape == (dim, width)
    assert np.all(guess[head.shape[0]:] == 0.0)
    ov = np.abs(np.sum(guess[: head.shape[0]] * head, axis=0))
    np.testing.assert_allclose(ov[:8], 1.0, atol=1e-8)
    np.testing.assert_allclose(ov, 1.0, atol=1e-4)


def test_multilevel_matches_reference_golden(golden):
    g = golden("multilevel")
    h = multilevel_operator(g)
    res = ci.multilevel_guess(h, g["level_dims"].tolist(), ci.MultilevelOptions(k_want=8, k_trial=12, tol=1e-6))
    assert [lv.dim for lv in res.levels] == g["level_dims"].tolist()
    assert [lv.iterations for lv in res.levels] == g["level_iterations"].tolist()
    assert [lv.converged for lv in res.levels] == g["level_converged"].tolist()
    check_guess(res.guess, g["guess_head"], int(g["guess_width"]), h.dim)
    # the guess is orthonormal and a good start: LOBPCG on the Nmax-4 block
    # from the padded level-2 block converges at once
    np.testing.assert_allclose(res.guess.T @ res.guess, np.eye(12), atol=1e-12)


def test_multilevel_live_reference(ref_lib):
    """The full 4He Nmax 6 problem assembled by the reference itself."""
    from oracle.ref import SyntheticProblem, multilevel_guess

    spec, params = (2, 2, 0, 1, 6, 1.0), (1, 0.1, 2, 2000, 0)
    p = SyntheticProblem(*spec, seed=1, offdiag=0.1, d=2, beta=2000, precision=0)
    with tempfile.TemporaryDirectory() as td:
        h = p.csb(os.path.join(td, "he.csb"))
    gref, lvref = multilevel_guess(spec, params, levels=3, k_want=8, k_trial=12, tol=1e-6)
    dims = [r[1] for r in lvref]  # the stratum ends of Nmax 2 and 4
    assert dims == p.strata[2:4].tolist()
    res = ci.multilevel_guess(h, dims, ci.MultilevelOptions(k_want=8, k_trial=12, tol=1e-6))
    assert [(lv.dim, lv.iterations, lv.converged) for lv in res.levels] == [(r[1], r[2], r[3]) for r in lvref]
    check_guess(res.guess, gref[: dims[-1]], gref.shape[1], h.dim)


def test_multilevel_single_level_and_collapse():
    h = gen_from((2000, 4, 64, 0.1, 0.5, 11, 1, 500))
    res = ci.multilevel_guess(h, [], ci.MultilevelOptions(k_want=4, k_trial=6))
    np.testing.assert_allclose(res.guess.T @ res.guess, np.eye(6), atol=1e-12)
    assert res.levels == []
    with pytest.raises(ci.SubspaceCollapse):  # a 3-row level cannot hold k_want = 4 columns
        ci.multilevel_guess(h, [3, 500], ci.MultilevelOptions(k_want=4, k_trial=6))
    with pytest.raises(ci.DimensionMismatch):
        ci.multilevel_guess(h, [500, 400], ci.MultilevelOptions(k_want=4, k_trial=6))


def test_leading_view_spmm():
    """A leading view multiplies like the leading principal block (sector
    boundaries of the generator are panel boundaries; arbitrary cuts too)."""
    h = gen_from((3072, 3, 256, 0.2, 0.4, 13, 0, 2000))
    dm = ci.DeviceMatrix(h, cuts=[1000])
    dense = h.to_dense()
    for d in (1024, 1000, 2048):
        v = dm.leading(d)
        assert v.dim == d and v.row_hi == d
        x = ci.random_block(d, 5, d)
        np.testing.assert_allclose(v.spmm_host(x), dense[:d, :d] @ x, rtol=0, atol=1e-12)
    with pytest.raises(ci.DimensionMismatch):
        dm.leading(1001)
    # a view is a full-fledged operand: LOBPCG on it = LOBPCG on the block
    ev = np.linalg.eigvalsh(dense[:1024, :1024])[:4]
    rep = ci.lobpcg_solve(dm.leading(1024), ci.random_block(1024, 8, 3), ci.LobpcgOptions(k_want=4, tol=1e-8))
    assert rep.converged
    np.testing.assert_allclose(rep.eigenvalues, ev, rtol=1e-8)


def test_orthonormalize_rayleigh_ritz_residual_norms_vs_reference(ref_lib):
    h = gen_from((2000, 4, 64, 0.1, 0.5, 11, 1, 500))
    y = ci.random_block(2000, 10, 5)
    # a zero column is dropped deterministically (its remaining diagonal is
    # exactly 0); nearly dependent columns sit at the drop threshold
    # (drop_tol^2 = 1e-16 relative), where Gram rounding decides
    y[:, 7] = 0.0
    q = ci.orthonormalize(y)
    qr = ref_lib.orthonormalize(y)
    assert q.shape == qr.shape == (2000, 9)
    np.testing.assert_allclose(q, qr, atol=1e-12)
    a = ci.random_block(2000, 3, 9)
    a = ci.orthonormalize(a)
    qa = ci.orthonormalize(ci.random_block(2000, 4, 11), against=a)
    np.testing.assert_allclose(qa, ref_lib.orthonormalize(ci.random_block(2000, 4, 11), against=a), atol=1e-12)
    assert np.abs(a.T @ qa).max() < 1e-13
    hq = ci.spmm(h, q)
    th, coeff = ci.rayleigh_ritz(q, hq, 4)
    thr, gr = ref_lib.rayleigh_ritz(q, hq, 4)
    np.testing.assert_allclose(th, thr, rtol=1e-12)
    np.testing.assert_allclose(np.abs(coeff.g), np.abs(gr), atol=1e-10)
    assert coeff.x_width == 9 and coeff.w_width == 0 and coeff.p_width == 0
    with pytest.raises(ci.IndefiniteGram):
        ci.rayleigh_ritz(y, ci.spmm(h, y), 4)
    x = q @ coeff.g
    rn = ci.residual_norms(h, x, th)
    np.testing.assert_allclose(rn, ref_lib.residual_norms(ref_lib.RefMatrix(h), x, th), rtol=1e-10)
    np.testing.assert_allclose(ci.residual_norms(h, x, th, norm_est=5.0),
                               ref_lib.residual_norms(ref_lib.RefMatrix(h), x, th, 5.0), rtol=1e-10)


def test_bvec_round_trip(tmp_path):
    x = ci.orthonormalize(ci.random_block(500, 6, 2))
    p = str(tmp_path / "g.bvec")
    ci.save_vectors(x, p)
    raw = open(p, "rb").read()
    assert raw[:4] == b"BVEC" and len(raw) == 4 + 8 + 4 + 500 * 6 * 8
    y = ci.load_guess_file(p, 500, 4)
    np.testing.assert_allclose(np.abs(np.sum(y * x[:, :4], axis=0)), 1.0, atol=1e-12)
    with pytest.raises(ci.DimensionMismatch):
        ci.load_guess_file(p, 499, 4)
    with pytest.raises(ci.DimensionMismatch):
        ci.load_guess_file(p, 500, 7)
    open(p, "wb").write(b"XXXX")
    with pytest.raises(ci.FormatError):
        ci.load_guess_file(p, 500, 4)
