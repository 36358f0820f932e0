"""TEST INFRASTRUCTURE ONLY -- ctypes binding of oracle/_ref/libciref.so, the
UNMODIFIED reference sources (/root/reference/proj/src) compiled against the
Eigen-API shim (oracle/Makefile, oracle/ref_capi.cpp)."""
from __future__ import annotations

import ctypes as C
import os
import pathlib
import weakref

import numpy as np

LIB_PATH = pathlib.Path(__file__).resolve().parent / "_ref" / "libciref.so"
_LIB = None


def available() -> bool:
    return LIB_PATH.exists()


def load() -> C.CDLL:
    global _LIB
    if _LIB is None:
        if not LIB_PATH.exists():
            raise ImportError(f"{LIB_PATH} missing: run `make -C oracle` where /root/reference exists")
        _LIB = C.CDLL(str(LIB_PATH), mode=os.RTLD_NOW | os.RTLD_LOCAL)
        _LIB.ciref_last_error.restype = C.c_char_p
    return _LIB


class RefError(RuntimeError):
    pass


def _chk(rc):
    if rc:
        raise RefError(load().ciref_last_error().decode())


def _p(a, t=C.c_double):
    return a.ctypes.data_as(C.POINTER(t))


def set_threads(n: int) -> None:
    load().ciref_set_threads(int(n))


def max_threads() -> int:
    return int(load().ciref_max_threads())


class RefMatrix:
    """ci::CsbMatrix built from the flattened arrays of a ci.CsbMatrix."""

    def __init__(self, h):
        lib = load()
        self.h = h  # keep arrays alive
        out = C.c_void_p()
        _chk(lib.ciref_matrix_create(C.c_uint32(h.dim), C.c_uint32(h.block_count()), C.c_int(h.precision),
                                     _p(h.block_boundaries, C.c_uint32), _p(h.entry_offsets, C.c_uint64),
                                     _p(h.rows, C.c_uint16), _p(h.cols, C.c_uint16),
                                     h.values.ctypes.data_as(C.c_void_p), C.byref(out)))
        self.handle = out
        self._fin = weakref.finalize(self, lib.ciref_matrix_destroy, out)

    def spmm(self, x, serial=False):
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = np.empty_like(x)
        _chk(load().ciref_spmm(self.handle, _p(x), C.c_uint32(x.shape[1]), _p(y), C.c_int(1 if serial else 0)))
        return y

    @classmethod
    def load(cls, path):
        """ci::load_csb of a CSB1 file (handle only; h-less)."""
        lib = load()
        out = C.c_void_p()
        _chk(lib.ciref_matrix_load(str(path).encode(), C.byref(out)))
        obj = cls.__new__(cls)
        obj.h = None
        obj.handle = out
        obj._fin = weakref.finalize(obj, lib.ciref_matrix_destroy, out)
        return obj

    def save(self, path):
        _chk(load().ciref_matrix_save(self.handle, str(path).encode()))

    def summary(self):
        d, z, nb, p = C.c_uint32(), C.c_uint64(), C.c_uint32(), C.c_int()
        load().ciref_matrix_summary(self.handle, C.byref(d), C.byref(z), C.byref(nb), C.byref(p))
        return d.value, z.value, nb.value, p.value

    def spmm_dim(self, x, serial=True):
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = np.empty_like(x)
        _chk(load().ciref_spmm(self.handle, _p(x), C.c_uint32(x.shape[1]), _p(y), C.c_int(1 if serial else 0)))
        return y

    def to_dense(self):
        d = np.empty((self.h.dim, self.h.dim), order="F")
        _chk(load().ciref_to_dense(self.handle, d.ctypes.data_as(C.POINTER(C.c_double))))
        return np.ascontiguousarray(d)


def block_inner(x, y, serial=False):
    x, y = (np.ascontiguousarray(a, dtype=np.float64) for a in (x, y))
    out = np.empty(x.shape[1] * y.shape[1])
    _chk(load().ciref_block_inner(C.c_uint32(x.shape[0]), _p(x), C.c_uint32(x.shape[1]), _p(y),
                                  C.c_uint32(y.shape[1]), C.c_int(1 if serial else 0), _p(out)))
    return out.reshape(y.shape[1], x.shape[1]).T.copy()


def linear_combination(y, g):
    y = np.ascontiguousarray(y, dtype=np.float64)
    gf = np.asfortranarray(g, dtype=np.float64)
    out = np.empty((y.shape[0], g.shape[1]))
    _chk(load().ciref_linear_combination(C.c_uint32(y.shape[0]), _p(y), C.c_uint32(y.shape[1]),
                                         gf.ctypes.data_as(C.POINTER(C.c_double)), C.c_uint32(g.shape[1]), _p(out)))
    return out


def add_linear_combination(y, x, g):
    x = np.ascontiguousarray(x, dtype=np.float64)
    yy = np.ascontiguousarray(y, dtype=np.float64).copy()
    gf = np.asfortranarray(g, dtype=np.float64)
    _chk(load().ciref_add_linear_combination(C.c_uint32(yy.shape[0]), _p(yy), C.c_uint32(yy.shape[1]), _p(x),
                                             C.c_uint32(x.shape[1]), gf.ctypes.data_as(C.POINTER(C.c_double))))
    return yy


def orthonormalize(y, drop_tol=1e-8, against=None):
    y = np.ascontiguousarray(y, dtype=np.float64)
    out = np.empty_like(y)
    kout = C.c_uint32()
    if against is not None and against.shape[1] > 0:
        a = np.ascontiguousarray(against, dtype=np.float64)
        ap, ka = _p(a), a.shape[1]
    else:
        ap, ka = None, 0
    _chk(load().ciref_orthonormalize(C.c_uint32(y.shape[0]), _p(y), C.c_uint32(y.shape[1]), C.c_double(drop_tol),
                                     ap, C.c_uint32(ka), _p(out), C.byref(kout)))
    k = kout.value  # the result is packed n x k (row-major)
    return out.reshape(-1)[: y.shape[0] * k].reshape(y.shape[0], k).copy() if k else np.zeros((y.shape[0], 0))


class RefTileDiagonal:
    def __init__(self, refmat: RefMatrix, bounds):
        lib = load()
        self.bounds = np.ascontiguousarray(bounds, dtype=np.uint32)
        out = C.c_void_p()
        _chk(lib.ciref_tilediag_create(refmat.handle, _p(self.bounds, C.c_uint32), C.c_uint32(len(self.bounds) - 1),
                                       C.byref(out)))
        self.handle = out
        self._fin = weakref.finalize(self, lib.ciref_tilediag_destroy, out)

    def blocks(self):
        sizes = np.diff(self.bounds.astype(np.int64))
        flat = np.empty(int((sizes ** 2).sum()))
        _chk(load().ciref_tilediag_blocks(self.handle, _p(flat)))
        out, o = [], 0
        for s in sizes:
            out.append(flat[o:o + s * s].reshape(s, s, order="F").copy())
            o += s * s
        return out


def _cfg(cfg):
    return None if cfg is None else _p(np.ascontiguousarray(cfg.as_array()))


def choose_shifts(theta, res_norm, x_norm, relres, iteration, tol, cfg=None):
    th, rn, xn, rr = (np.ascontiguousarray(a, dtype=np.float64) for a in (theta, res_norm, x_norm, relres))
    k = len(th)
    mu = np.zeros(k)
    en = np.zeros(k, dtype=np.int32)
    ca = None if cfg is None else np.ascontiguousarray(cfg.as_array())
    _chk(load().ciref_choose_shifts(C.c_uint32(k), _p(th), _p(rn), _p(xn), _p(rr), C.c_int(iteration),
                                    C.c_double(tol), None if ca is None else _p(ca), _p(mu), _p(en, C.c_int)))
    return mu, en.astype(bool)


def apply_preconditioner(td: RefTileDiagonal, r, mu, engage, cfg=None):
    r = np.ascontiguousarray(r, dtype=np.float64)
    w = np.empty_like(r)
    mu = np.ascontiguousarray(mu, dtype=np.float64)
    en = np.ascontiguousarray(engage, dtype=np.int32)
    ca = None if cfg is None else np.ascontiguousarray(cfg.as_array())
    _chk(load().ciref_apply_preconditioner(td.handle, C.c_uint32(r.shape[0]), _p(r), C.c_uint32(r.shape[1]), _p(mu),
                                           _p(en, C.c_int), None if ca is None else _p(ca), _p(w)))
    return w


def fom_solve(block, mu, rhs, iters):
    block = np.asfortranarray(block, dtype=np.float64)
    rhs = np.asfortranarray(rhs, dtype=np.float64)
    mu = np.ascontiguousarray(mu, dtype=np.float64)
    out = np.empty(rhs.shape, order="F")
    _chk(load().ciref_fom_solve(C.c_uint32(block.shape[0]), block.ctypes.data_as(C.POINTER(C.c_double)),
                                C.c_uint32(rhs.shape[1]), _p(mu), rhs.ctypes.data_as(C.POINTER(C.c_double)),
                                C.c_int(iters), out.ctypes.data_as(C.POINTER(C.c_double))))
    return np.ascontiguousarray(out)


class RefReport:
    pass


def _report(handle, dim):
    lib = load()
    conv, iters, ne = C.c_int(), C.c_int(), C.c_double()
    kt, nh, nev = C.c_uint32(), C.c_uint64(), C.c_uint32()
    cnt = np.zeros(4, dtype=np.uint64)
    lib.ciref_report_summary(handle, C.byref(conv), C.byref(iters), C.byref(ne), C.byref(kt), C.byref(nh),
                             _p(cnt, C.c_uint64), C.byref(nev))
    ev = np.zeros(nev.value)
    trial = np.zeros((dim, kt.value))
    n = nh.value
    hi, hc, hr, ht = np.zeros(n, np.int32), np.zeros(n, np.int32), np.zeros(n), np.zeros(n)
    lib.ciref_report_arrays(handle, _p(ev), _p(trial), _p(hi, C.c_int), _p(hc, C.c_int), _p(hr), _p(ht))
    lib.ciref_report_destroy(handle)
    r = RefReport()
    r.converged, r.iterations, r.norm_estimate = bool(conv.value), iters.value, ne.value
    r.eigenvalues, r.trial_vectors = ev, trial
    r.history = np.rec.fromarrays([hi, hc, hr, ht], names="iteration,column,relres,theta")
    r.counters = cnt.astype(np.int64)
    return r


def lobpcg_solve(refmat: RefMatrix, x0, k_want, tol, max_iter=500, tilediag: RefTileDiagonal = None, cfg=None):
    x0 = np.ascontiguousarray(x0, dtype=np.float64)
    out = C.c_void_p()
    ca = None if cfg is None else np.ascontiguousarray(cfg.as_array())
    _chk(load().ciref_lobpcg_solve(refmat.handle, _p(x0), C.c_uint32(x0.shape[1]), C.c_int(k_want), C.c_double(tol),
                                   C.c_int(max_iter), None if tilediag is None else tilediag.handle,
                                   None if ca is None else _p(ca), C.byref(out)))
    return _report(out, refmat.h.dim if refmat.h is not None else refmat.dim)


def lanczos_solve(refmat: RefMatrix, v0, k_want, tol, max_iter=500):
    v0 = np.ascontiguousarray(v0, dtype=np.float64)
    out = C.c_void_p()
    _chk(load().ciref_lanczos_solve(refmat.handle, _p(v0), C.c_int(k_want), C.c_double(tol), C.c_int(max_iter),
                                    C.byref(out)))
    return _report(out, refmat.h.dim)


class SyntheticProblem:
    """ci::build_synthetic_problem (hamiltonian.cpp:205-224): the reference's
    physics-basis synthetic Hamiltonian (basis enumeration, grouping, tiles,
    assembly), for pinning the multilevel guess."""

    def __init__(self, Z, N, M2, parity, Nmax, hw=1.0, seed=1, offdiag=0.1, d=2, beta=2000, precision=1):
        lib = load()
        self.spec = (Z, N, M2, parity, Nmax, hw)
        self.params = (seed, offdiag, d, beta, precision)
        out = C.c_void_p()
        _chk(lib.ciref_synthetic_problem(C.c_int(Z), C.c_int(N), C.c_int(M2), C.c_int(parity), C.c_int(Nmax),
                                         C.c_double(hw), C.c_uint64(seed), C.c_double(offdiag), C.c_int(d),
                                         C.c_uint32(beta), C.c_int(precision), C.byref(out)))
        self.handle = out
        self._fin = weakref.finalize(self, lib.ciref_problem_destroy, out)
        lib.ciref_problem_matrix.restype = C.c_void_p
        lib.ciref_problem_groups.restype = C.c_uint32
        lib.ciref_problem_strata.restype = C.c_uint32
        self.matrix_handle = C.c_void_p(lib.ciref_problem_matrix(out))
        ng = lib.ciref_problem_groups(out, None)
        self.groups = np.zeros(ng, np.uint32)
        lib.ciref_problem_groups(out, _p(self.groups, C.c_uint32))
        ns = lib.ciref_problem_strata(out, None)
        self.strata = np.zeros(ns, np.uint32)
        lib.ciref_problem_strata(out, _p(self.strata, C.c_uint32))

    def csb(self, path):
        """The assembled matrix as a ci.CsbMatrix (through a CSB1 file), with
        the problem's group partition attached."""
        from paper_1609_01689_b200 import ci

        _chk(load().ciref_matrix_save(self.matrix_handle, str(path).encode()))
        h = ci.load_csb(str(path))
        h.groups = self.groups.copy()
        return h


def multilevel_guess(spec, params, levels, k_want, k_trial, tol, max_iter=500, mseed=1):
    """ci::multilevel_guess (guess.cpp:66-117) with build_synthetic_problem as
    the factory. Returns (guess n x k, [(nmax, dim, iterations, converged)])."""
    lib = load()
    Z, N, M2, parity, Nmax, hw = spec
    seed, offdiag, d, beta, precision = params
    full = SyntheticProblem(*spec, seed=seed, offdiag=offdiag, d=d, beta=beta, precision=precision)
    dim = int(full.strata[-1])
    guess = np.zeros((dim, k_trial))
    kout, dout, nlv = C.c_uint32(), C.c_uint32(), C.c_int()
    lv = [np.zeros(levels, np.int32), np.zeros(levels, np.uint32), np.zeros(levels, np.int32), np.zeros(levels, np.int32)]
    _chk(lib.ciref_multilevel_guess(C.c_int(Z), C.c_int(N), C.c_int(M2), C.c_int(parity), C.c_int(Nmax),
                                    C.c_double(hw), C.c_uint64(seed), C.c_double(offdiag), C.c_int(d),
                                    C.c_uint32(beta), C.c_int(precision), C.c_int(levels), C.c_int(k_want),
                                    C.c_int(k_trial), C.c_double(tol), C.c_int(max_iter), C.c_uint64(mseed),
                                    _p(guess), C.byref(kout), C.byref(dout), C.byref(nlv),
                                    _p(lv[0], C.c_int), _p(lv[1], C.c_uint32), _p(lv[2], C.c_int), _p(lv[3], C.c_int)))
    g = guess.reshape(-1)[: dout.value * kout.value].reshape(dout.value, kout.value)
    rows = [(int(lv[0][i]), int(lv[1][i]), int(lv[2][i]), bool(lv[3][i])) for i in range(nlv.value)]
    return g, rows


def rayleigh_ritz(y, hy, k_trial):
    """ci::rayleigh_ritz (lobpcg.cpp:121-145) -> (theta, g m x k_trial)."""
    y = np.ascontiguousarray(y, dtype=np.float64)
    hy = np.ascontiguousarray(hy, dtype=np.float64)
    n, m = y.shape
    theta = np.zeros(k_trial)
    g = np.zeros(m * k_trial)
    _chk(load().ciref_rayleigh_ritz(C.c_uint32(n), _p(y), _p(hy), C.c_uint32(m), C.c_int(k_trial), _p(theta), _p(g)))
    return theta, g.reshape(k_trial, m).T.copy()


def residual_norms(refmat, x, theta, norm_est=None):
    """ci::residual_norms (lobpcg.cpp:147-169)."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    th = np.ascontiguousarray(theta, dtype=np.float64)
    out = np.zeros(x.shape[1])
    _chk(load().ciref_residual_norms(refmat.handle, _p(x), C.c_uint32(x.shape[1]), _p(th),
                                     C.c_double(norm_est if norm_est is not None else 0.0), _p(out)))
    return out


# --------------------------------------------------------------- generator
# ref_gen.cpp: the BASELINE sector generator restated for the oracle, building
# the reference's own ci::CsbMatrix without the product library.

def generate(n, sectors, tile, p, q, seed, precision, beta=2000, band=2, nbk=0):
    """ci::CsbMatrix of the leading nbk CSB block rows (0: all) of the sector
    matrix -> a handle-only RefMatrix (its .nnz / .nb_total are set)."""
    lib = load()
    out, nnz, nbt = C.c_void_p(), C.c_uint64(), C.c_uint32()
    rc = lib.ciref_generate(C.c_uint64(n), C.c_uint32(sectors), C.c_uint32(tile), C.c_double(p), C.c_double(q),
                            C.c_uint64(seed), C.c_int(precision), C.c_uint32(beta), C.c_uint32(band),
                            C.c_uint32(nbk), C.c_int(0), C.byref(out), C.byref(nnz), C.byref(nbt))
    if rc:
        raise RefError("ciref_generate failed")
    obj = RefMatrix.__new__(RefMatrix)
    obj.h = None
    obj.handle = out
    obj._fin = weakref.finalize(obj, lib.ciref_matrix_destroy, out)
    obj.nnz = nnz.value
    obj.nb_total = nbt.value
    obj.dim = obj.summary()[0]
    return obj


def count_nnz(n, sectors, tile, p, q, seed, band=2):
    """Stored entries of the full sector matrix (no storage)."""
    lib = load()
    nnz, nbt = C.c_uint64(), C.c_uint32()
    rc = lib.ciref_generate(C.c_uint64(n), C.c_uint32(sectors), C.c_uint32(tile), C.c_double(p), C.c_double(q),
                            C.c_uint64(seed), C.c_int(0), C.c_uint32(2000), C.c_uint32(band), C.c_uint32(0),
                            C.c_int(1), None, C.byref(nnz), C.byref(nbt))
    if rc:
        raise RefError("ciref_generate (count) failed")
    return nnz.value


def expected_nnz(n, sectors, tile, p, q, band=2):
    lib = load()
    lib.ciref_generate_expected_nnz.restype = C.c_double
    return lib.ciref_generate_expected_nnz(C.c_uint64(n), C.c_uint32(sectors), C.c_uint32(tile), C.c_double(p),
                                           C.c_double(q), C.c_uint32(band))


def calibrated_p(n, sectors, tile, q, target_nnz, band=2):
    """p giving target_nnz expected stored entries (configs.Config.p restated)."""
    s0 = expected_nnz(n, sectors, tile, 0.0, q, band)
    s1 = expected_nnz(n, sectors, tile, 1.0, q, band)
    return (target_nnz - s0) / (s1 - s0)


def spmm_timed(rm, x, reps):
    """ci::spmm timed inside the reference library: per-call seconds and U."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.empty_like(x)
    secs = np.empty(reps)
    _chk(load().ciref_spmm_timed(rm.handle, _p(x), C.c_uint32(x.shape[1]), C.c_int(reps), _p(secs), _p(y)))
    return secs, y
