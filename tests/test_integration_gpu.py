"""The reference-side drop-in (integration/ci_gpu_dropin.cpp): the reference's
own ci::lobpcg_solve signature, compiled against the reference headers, now
running on the GPU -- same iteration count and eigenvalues as the
reference's CPU solve (golden fixture)."""
import ctypes as C
import os

import numpy as np
import pytest

from conftest import ROOT, gen_from
from paper_1609_01689_b200 import ci

pytestmark = pytest.mark.gpu
LIB = os.path.join(ROOT, "integration", "_build", "libcieigen_gpu.so")


@pytest.mark.parametrize("name", ["sector_f64", "sector_f64_prec"])
def test_dropin_lobpcg_matches_reference(golden, name):
    if not os.path.exists(LIB):
        pytest.skip("integration/_build not built (needs the reference headers at build time)")
    lib = C.CDLL(LIB)
    g = golden("lobpcg")
    k, kt, tol, pre, seed = g[f"{name}_meta"]
    h = gen_from(g[f"{name}_params"])
    x0 = ci.random_block(h.dim, int(kt), int(seed))
    v = h.view()
    groups = np.ascontiguousarray(h.groups, dtype=np.uint32)
    eig = np.zeros(int(k))
    iters = C.c_int()
    rc = lib.dropin_lobpcg(C.byref(v), groups.ctypes.data_as(C.POINTER(C.c_uint32)), C.c_uint32(len(groups) - 1),
                           x0.ctypes.data_as(C.POINTER(C.c_double)), C.c_uint32(int(kt)), C.c_int(int(k)),
                           C.c_double(float(tol)), C.c_int(int(pre)), eig.ctypes.data_as(C.POINTER(C.c_double)),
                           C.byref(iters))
    assert rc == 0
    assert iters.value == int(g[f"{name}_iterations"])
    np.testing.assert_allclose(eig, g[f"{name}_eigenvalues"], rtol=1e-10)


@pytest.mark.parametrize("name", ["sector_f64", "sector_f32"])
def test_dropin_lanczos_matches_reference(golden, name):
    """ci::lanczos_solve through the reference-side drop-in on the GPU."""
    if not os.path.exists(LIB):
        pytest.skip("integration/_build not built (needs the reference headers at build time)")
    lib = C.CDLL(LIB)
    g = golden("lanczos")
    k, tol, max_iter, _ = g[f"{name}_meta"]
    h = gen_from(g[f"{name}_params"])
    v0 = np.ascontiguousarray(g[f"{name}_v0"])
    v = h.view()
    eig = np.zeros(int(k))
    iters = C.c_int()
    rc = lib.dropin_lanczos(C.byref(v), v0.ctypes.data_as(C.POINTER(C.c_double)), C.c_int(int(k)),
                            C.c_double(float(tol)), C.c_int(int(max_iter)), eig.ctypes.data_as(C.POINTER(C.c_double)),
                            C.byref(iters))
    assert rc == 0
    assert iters.value == int(g[f"{name}_iterations"])
    np.testing.assert_allclose(eig, g[f"{name}_eigenvalues"], rtol=1e-10)


def test_dropin_orthonormalize_and_residual_norms(ref_lib):
    """ci::orthonormalize / ci::residual_norms through the drop-in vs the reference."""
    if not os.path.exists(LIB):
        pytest.skip("integration/_build not built (needs the reference headers at build time)")
    lib = C.CDLL(LIB)
    y = ci.random_block(1500, 6, 4)
    out = np.zeros_like(y)
    kout = C.c_uint32()
    pd = lambda a: a.ctypes.data_as(C.POINTER(C.c_double))  # noqa: E731
    assert lib.dropin_orthonormalize(C.c_uint32(1500), C.c_uint32(6), pd(y), C.c_double(1e-8), pd(out),
                                     C.byref(kout)) == 0
    assert kout.value == 6
    np.testing.assert_allclose(out, ref_lib.orthonormalize(y), atol=1e-12)
    h = gen_from((2000, 4, 64, 0.1, 0.5, 11, 1, 500))
    x = ci.random_block(2000, 3, 8)
    th = np.array([0.5, -1.0, 2.0])
    r = np.zeros(3)
    v = h.view()
    assert lib.dropin_residual_norms(C.byref(v), pd(x), C.c_uint32(3), pd(th), pd(r)) == 0
    np.testing.assert_allclose(r, ref_lib.residual_norms(ref_lib.RefMatrix(h), x, th), rtol=1e-12)


SOLVE_GPU = os.path.join(ROOT, "integration", "_build", "ci_solve_gpu")
SOLVE_REF = os.path.join(ROOT, "integration", "_build", "ci_solve_ref")


def _run(exe, args):
    import json
    import subprocess

    out = subprocess.run([exe] + [str(a) for a in args], check=True, capture_output=True, text=True, timeout=600)
    return json.loads(out.stdout.strip().splitlines()[-1])


# (Z, N, M2, parity, Nmax, seed, offdiag, d, beta, precision, k_want, k_trial, tol, max_iter)
LINK_CASES = [(2, 2, 0, 1, 4, 1, 0.1, 2, 2000, 1, 4, 8, 1e-8, 500),
              (2, 2, 0, 1, 6, 3, 0.1, 2, 2000, 0, 4, 6, 1e-6, 500),
              (3, 3, 2, -1, 3, 5, 0.2, 2, 2000, 1, 3, 5, 1e-8, 500)]


@pytest.mark.parametrize("case", LINK_CASES)
def test_linked_dropin_build_matches_reference_build(case):
    """The same run_solver-equivalent driver (integration/ci_solve_main.cpp),
    linked once against all eleven reference TUs (CPU) and once with
    csb/block_vectors/lobpcg/precond/lanczos.cpp replaced by the drop-in
    (+ libcieg.so): identical iteration counts, counters and multilevel level
    iterations; every operator-level result to rounding."""
    if not (os.path.exists(SOLVE_GPU) and os.path.exists(SOLVE_REF)):
        pytest.skip("integration/_build not built (needs /root/reference at build time)")
    g, r = _run(SOLVE_GPU, case), _run(SOLVE_REF, case)
    for key in ("dim", "nnz", "iterations", "converged", "counters", "stats", "history_csv_lines",
                "multilevel_level_iterations", "multilevel_iterations"):
        assert g[key] == r[key], key
    tol_eig = 1e-5 if case[9] == 0 else 1e-9
    np.testing.assert_allclose(g["eigenvalues"], r["eigenvalues"], rtol=tol_eig)
    np.testing.assert_allclose(g["multilevel_eigenvalues"], r["multilevel_eigenvalues"], rtol=tol_eig)
    for key in ("spmm", "block_inner", "linear_combination", "add_linear_combination", "apply_preconditioner",
                "fom_solve", "csb_roundtrip_spmm"):
        np.testing.assert_allclose(g[key], r[key], rtol=1e-12, err_msg=key)
    np.testing.assert_allclose(g["column_norms"], r["column_norms"], rtol=1e-13)
    np.testing.assert_allclose(g["residual_norms"], r["residual_norms"], rtol=1e-3, atol=1e-12)


def test_dropin_cache_follows_content_not_address(ref_lib):
    """two matrices with the same structure and different values
    built at the same address (the CLI's `compare` loop) must not reuse the
    first upload: dropin_lobpcg builds its CsbMatrix / TileDiagonal on the
    stack, call after call."""
    if not os.path.exists(LIB):
        pytest.skip("integration/_build not built")
    lib = C.CDLL(LIB)
    for seed in (11, 12, 13):
        h = gen_from((3000, 3, 64, 0.1, 0.5, seed, 1, 2000))
        x0 = ci.random_block(h.dim, 6, 7)
        v = h.view()
        groups = np.ascontiguousarray(h.groups, dtype=np.uint32)
        eig = np.zeros(3)
        iters = C.c_int()
        assert lib.dropin_lobpcg(C.byref(v), groups.ctypes.data_as(C.POINTER(C.c_uint32)),
                                 C.c_uint32(len(groups) - 1), x0.ctypes.data_as(C.POINTER(C.c_double)), C.c_uint32(6),
                                 C.c_int(3), C.c_double(1e-8), C.c_int(1), eig.ctypes.data_as(C.POINTER(C.c_double)),
                                 C.byref(iters)) == 0
        rm = ref_lib.RefMatrix(h)
        rr = ref_lib.lobpcg_solve(rm, x0, 3, 1e-8, 500, ref_lib.RefTileDiagonal(rm, h.groups))
        assert iters.value == rr.iterations
        np.testing.assert_allclose(eig, rr.eigenvalues, rtol=1e-10)


CLI_GPU = os.path.join(ROOT, "integration", "_build", "ci_eigen_gpu")
CLI_REF = os.path.join(ROOT, "integration", "_build", "ci_eigen_ref")


def _cli(exe, *args):
    import subprocess

    p = subprocess.run([exe, *args], capture_output=True, text=True, timeout=600)
    return p.returncode, p.stdout


def _solve_summary(out):
    lines = out.splitlines()
    it = next(l for l in lines if l.startswith("solver "))
    ev = [float(l.split()[-1]) for l in lines if l.startswith("eigenvalue ")]
    ctr = next(l for l in lines if l.startswith("spmm_calls "))
    return it, ev, ctr


@pytest.mark.parametrize("args", [
    ["--nucleus", "4He", "--nmax", "4", "--k", "4", "--precond", "tile", "--tol", "1e-8", "--storage", "double"],
    ["--nucleus", "4He", "--nmax", "4", "--k", "4", "--tol", "1e-8", "--storage", "single"],
    ["--nucleus", "4He", "--nmax", "4", "--k", "3", "--solver", "lanczos", "--tol", "1e-8", "--storage", "double"],
    ["--nucleus", "4He", "--nmax", "4", "--k", "2", "--guess", "multilevel", "--levels", "2", "--precond", "tile",
     "--tol", "1e-8", "--storage", "double"],
])
def test_reference_cli_on_the_gpu(tmp_path, args):
    """The reference's own CLI (proj/tools/ci_eigen.cpp, unmodified; CLI11 API
    shim) linked against the drop-in: `solve` prints the same iteration
    count, operation counters and eigenvalues as the same CLI linked against
    the eleven reference TUs; --history writes the same CSV rows."""
    if not (os.path.exists(CLI_GPU) and os.path.exists(CLI_REF)):
        pytest.skip("integration/_build not built (needs the reference sources at build time)")
    hg, hr = str(tmp_path / "g.csv"), str(tmp_path / "r.csv")
    rg, og = _cli(CLI_GPU, "solve", *args, "--history", hg)
    rr, orf = _cli(CLI_REF, "solve", *args, "--history", hr)
    assert rg == rr, (og, orf)
    itg, evg, cg = _solve_summary(og)
    itr, evr, cr = _solve_summary(orf)
    assert itg == itr and cg == cr, (og, orf)
    np.testing.assert_allclose(evg, evr, rtol=1e-10, atol=1e-11)
    lg = open(hg).read().splitlines()
    lr = open(hr).read().splitlines()
    assert len(lg) == len(lr) and lg[0] == lr[0]


def test_reference_cli_assemble_and_compare(tmp_path):
    """`assemble` (host code in both builds) writes byte-identical CSB1;
    `compare` runs the four preconditioner / guess solves per seed on the GPU
    with the reference's iteration counts."""
    if not (os.path.exists(CLI_GPU) and os.path.exists(CLI_REF)):
        pytest.skip("integration/_build not built (needs the reference sources at build time)")
    a = ["--nucleus", "4He", "--nmax", "4", "--storage", "double"]
    pg, pr = str(tmp_path / "g.csb"), str(tmp_path / "r.csb")
    assert _cli(CLI_GPU, "assemble", *a, "--out", pg)[0] == 0
    assert _cli(CLI_REF, "assemble", *a, "--out", pr)[0] == 0
    assert open(pg, "rb").read() == open(pr, "rb").read()
    c = ["--nucleus", "4He", "--nmax", "4", "--k", "2", "--tol", "1e-8", "--seeds", "1,2"]
    rg, og = _cli(CLI_GPU, "compare", *c)
    rr, orf = _cli(CLI_REF, "compare", *c)
    assert rg == rr == 0
    assert og == orf, (og, orf)
