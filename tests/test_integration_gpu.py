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
