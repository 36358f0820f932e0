"""Generate tests/golden/*.npz from the UNMODIFIED reference (oracle/_ref,
compiled from /root/reference/proj/src). Run here, where /root/reference
exists:  python tests/golden/make_golden.py
The fixtures pin the numpy oracle (oracle/ci_oracle.py) on the CPU and the
CUDA path on the GPU box, where /root/reference is absent."""
import hashlib
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import ref  # noqa: E402
from paper_1609_01689_b200 import ci  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))

# (n, sectors, tile, p, q, seed, precision, beta)
SPMM_CASES = {
    "f64": (3000, 3, 64, 0.1, 0.5, 2, 1, 500),
    "f32": (3000, 3, 64, 0.1, 0.5, 2, 0, 500),
    "f32_t256": (4096, 2, 256, 0.2, 0.4, 5, 0, 2000),
}
LOBPCG_CASES = {
    # name: (gen params, k_want, kt, tol, precond, x0 seed)
    "sector_f64": ((2000, 4, 64, 0.1, 0.5, 11, 1, 500), 4, 8, 1e-8, False, 42),
    "sector_f64_prec": ((2000, 4, 64, 0.1, 0.5, 11, 1, 500), 4, 8, 1e-8, True, 42),
    "sector_f32_prec": ((3072, 3, 256, 0.2, 0.4, 13, 0, 2000), 4, 8, 1e-6, True, 43),
}


LANCZOS_CASES = {
    # name: (gen params or None = diag(1..100), v0 kind, k_want, tol, max_iter)
    "diag100_restart": (None, "e0+e1", 3, 1e-10, 100),
    "sector_f64": ((2000, 4, 64, 0.1, 0.5, 11, 1, 500), "stratum", 4, 1e-8, 300),
    "sector_f32": ((3072, 3, 256, 0.2, 0.4, 13, 0, 2000), "stratum", 4, 1e-6, 300),
}


def diag100():
    n = 100
    return ci.CsbMatrix(dim=n, precision=1, block_boundaries=np.array([0, n], np.uint32),
                        entry_offsets=np.array([0, n], np.uint64), rows=np.arange(n, dtype=np.uint16),
                        cols=np.arange(n, dtype=np.uint16), values=np.arange(1, n + 1, dtype=np.float64),
                        groups=np.array([0, 50, n], np.uint32))


def lanczos_start(kind, n, sectors):
    v = np.zeros(n)
    if kind == "e0+e1":
        v[0] = v[1] = 1.0
    else:  # lanczos_default_start on the first sector (the lowest stratum)
        v[: n // sectors] = 1.0
    return v


def make_lanczos():
    la = {}
    for name, (p, kind, k, tol, max_iter) in LANCZOS_CASES.items():
        h = diag100() if p is None else gen(p)
        v0 = lanczos_start(kind, h.dim, 1 if p is None else int(p[1]))
        rm = ref.RefMatrix(h)
        r = ref.lanczos_solve(rm, v0, k, tol, max_iter)
        if p is not None:
            la[f"{name}_params"] = np.array(p, dtype=np.float64)
        la[f"{name}_meta"] = np.array([k, tol, max_iter, 0.0 if kind == "e0+e1" else 1.0])
        la[f"{name}_v0"] = v0
        la[f"{name}_eigenvalues"] = r.eigenvalues
        la[f"{name}_eigenvectors"] = r.trial_vectors
        la[f"{name}_iterations"] = np.array(r.iterations)
        la[f"{name}_converged"] = np.array(r.converged)
        la[f"{name}_counters"] = r.counters
        la[f"{name}_relres"] = r.history.relres
        la[f"{name}_theta"] = r.history.theta
        la[f"{name}_hist_iter"] = r.history.iteration
        la[f"{name}_norm_estimate"] = np.array(r.norm_estimate)
        la[f"{name}_dense_eigs"] = np.linalg.eigvalsh(rm.to_dense())[:k]
        print("lanczos", name, "iterations", r.iterations, "converged", r.converged, r.eigenvalues)
    np.savez_compressed(os.path.join(OUT, "lanczos.npz"), **la)


MULTILEVEL_SPEC = (2, 2, 0, 1, 6, 1.0)    # 4He, Nmax 6: strata 0 | 1 | 59 | 952 | 7916
MULTILEVEL_PARAMS = (1, 0.1, 2, 2000, 0)  # seed, offdiag_scale, d, beta, fp32 H


def make_multilevel():
    """The reference's own multilevel_guess (guess.cpp:66-117, factory =
    build_synthetic_problem) on 4He Nmax 6, levels 3 (Nmax 2 / 4 / 6). The
    level solves only see the Nmax-4 space (dim 952) -- the leading block of
    the Nmax-6 Hamiltonian -- and the guess is zero below row 952, so the
    fixture stores the Nmax-4 matrix, the guess's leading 952 rows and the
    level reports."""
    import tempfile

    Z, N, M2, par, nmax, hw = MULTILEVEL_SPEC
    seed, off, d, beta, prec = MULTILEVEL_PARAMS
    full = ref.SyntheticProblem(*MULTILEVEL_SPEC, seed=seed, offdiag=off, d=d, beta=beta, precision=prec)
    sub = ref.SyntheticProblem(Z, N, M2, par, nmax - 2, hw, seed=seed, offdiag=off, d=d, beta=beta, precision=prec)
    with tempfile.TemporaryDirectory() as td:
        h = sub.csb(os.path.join(td, "sub.csb"))
    g, lv = ref.multilevel_guess(MULTILEVEL_SPEC, MULTILEVEL_PARAMS, levels=3, k_want=8, k_trial=12, tol=1e-6)
    dsub = int(sub.strata[-1])
    assert np.all(g[dsub:] == 0.0)
    ml = {"full_dim": np.array(int(full.strata[-1])), "strata": full.strata, "level_dims": np.array([r[1] for r in lv]),
          "level_nmax": np.array([r[0] for r in lv]), "level_iterations": np.array([r[2] for r in lv]),
          "level_converged": np.array([r[3] for r in lv]), "guess_head": g[:dsub], "guess_width": np.array(g.shape[1]),
          "sub_block_boundaries": h.block_boundaries, "sub_entry_offsets": h.entry_offsets, "sub_rows": h.rows,
          "sub_cols": h.cols, "sub_values": h.values, "sub_groups": sub.groups, "sub_precision": np.array(h.precision)}
    np.savez_compressed(os.path.join(OUT, "multilevel.npz"), **ml)
    print("multilevel levels", lv, "guess", g.shape)


def digest(h):
    m = hashlib.sha256()
    for a in (h.block_boundaries, h.entry_offsets, h.rows, h.cols, h.values, h.groups):
        m.update(np.ascontiguousarray(a).tobytes())
    return m.hexdigest()


def gen(p):
    n, s, t, pp, q, seed, prec, beta = p
    return ci.generate_sector_matrix(n, s, t, pp, q, seed, prec, beta)


def main():
    ref.set_threads(4)
    out = {}
    # generator digests (C++ generator; the slow numpy port is checked on a
    # small case in the tests) and SpMM outputs of the reference spmm_serial
    for name, p in SPMM_CASES.items():
        h = gen(p)
        out[f"gen_{name}_params"] = np.array(p[:5] + (p[5], p[6], p[7]), dtype=np.float64)
        out[f"gen_{name}_digest"] = np.array(digest(h))
        out[f"gen_{name}_nnz"] = np.array(h.nnz_lower)
        rm = ref.RefMatrix(h)
        for m in (1, 5, 16):
            x = ci.random_block(h.dim, m, 100 + m)
            out[f"spmm_{name}_m{m}"] = rm.spmm(x, serial=True)
    np.savez_compressed(os.path.join(OUT, "spmm.npz"), **out)

    # tall-skinny kernels
    bv = {}
    x = ci.random_block(1003, 24, 1)
    y = ci.random_block(1003, 20, 2)
    g = 2.0 * ci.random_block(24, 16, 3)
    bv["block_inner"] = ref.block_inner(x, y)
    bv["linear_combination"] = ref.linear_combination(x, g)
    bv["add_linear_combination"] = ref.add_linear_combination(ci.random_block(1003, 16, 4), x, g)
    bv["orthonormalize"] = ref.orthonormalize(ci.random_block(1003, 12, 5), 1e-8, ci.random_block(1003, 6, 6))
    dup = ci.random_block(1003, 6, 7)
    dup = np.hstack([dup, dup[:, :2]])
    bv["orthonormalize_dup_width"] = np.array(ref.orthonormalize(dup).shape[1])
    np.savez_compressed(os.path.join(OUT, "blockvec.npz"), **bv)

    # choose_shifts cases
    rng = np.random.default_rng(0)
    sh = {}
    cases = []
    for c in range(24):
        k = int(rng.integers(1, 12))
        theta = np.sort(rng.normal(-5, 3, k))
        relres = 10.0 ** rng.uniform(-9, 0, k)
        if c % 5 == 0:
            relres[0] = 0.5
        res_norm = relres * 10.0
        x_norm = np.ones(k)
        it = int(rng.integers(1, 8))
        tol = [1e-6, 1e-8][c % 2]
        mu, en = ref.choose_shifts(theta, res_norm, x_norm, relres, it, tol)
        cases.append((k, it, tol))
        for nm, v in (("theta", theta), ("res_norm", res_norm), ("relres", relres), ("mu", mu), ("engage", en)):
            sh[f"{c}_{nm}"] = v
    sh["cases"] = np.array(cases, dtype=np.float64)
    np.savez_compressed(os.path.join(OUT, "shifts.npz"), **sh)

    # preconditioner: 64-row groups (direct LU) and 256-row groups (FOM)
    pc = {}
    for name, p, k in (("lu", (2048, 2, 64, 0.1, 0.5, 21, 1, 500), 8), ("fom", (2048, 2, 256, 0.2, 0.4, 22, 0, 2000), 8)):
        h = gen(p)
        rm = ref.RefMatrix(h)
        td = ref.RefTileDiagonal(rm, h.groups)
        r = ci.random_block(h.dim, k, 31)
        mu = np.linspace(-4.0, 3.0, k)
        mu[2] = mu[1]  # shared shift
        en = np.ones(k, dtype=bool)
        en[5] = False
        pc[f"{name}_params"] = np.array(p, dtype=np.float64)
        pc[f"{name}_mu"] = mu
        pc[f"{name}_engage"] = en
        pc[f"{name}_w"] = ref.apply_preconditioner(td, r, mu, en)
    np.savez_compressed(os.path.join(OUT, "precond.npz"), **pc)

    # LOBPCG
    lo = {}
    # H = diag(1..100), k_want=3, random X0 width 5 -> {1,2,3}
    n = 100
    hd = ci.CsbMatrix(dim=n, precision=1, block_boundaries=np.array([0, n], np.uint32),
                      entry_offsets=np.array([0, n], np.uint64), rows=np.arange(n, dtype=np.uint16),
                      cols=np.arange(n, dtype=np.uint16), values=np.arange(1, n + 1, dtype=np.float64),
                      groups=np.array([0, 50, n], np.uint32))
    cases = {"diag100": (hd, 3, 5, 1e-10, False, 7)}
    for name, (p, k, kt, tol, pre, seed) in LOBPCG_CASES.items():
        cases[name] = (gen(p), k, kt, tol, pre, seed)
        lo[f"{name}_params"] = np.array(p, dtype=np.float64)
    for name, (h, k, kt, tol, pre, seed) in cases.items():
        rm = ref.RefMatrix(h)
        td = ref.RefTileDiagonal(rm, h.groups) if pre else None
        x0 = ci.random_block(h.dim, kt, seed)
        r = ref.lobpcg_solve(rm, x0, k, tol, 500, td)
        lo[f"{name}_eigenvalues"] = r.eigenvalues
        lo[f"{name}_iterations"] = np.array(r.iterations)
        lo[f"{name}_converged"] = np.array(r.converged)
        lo[f"{name}_counters"] = r.counters
        lo[f"{name}_relres"] = r.history.relres
        lo[f"{name}_theta"] = r.history.theta
        lo[f"{name}_norm_estimate"] = np.array(r.norm_estimate)
        lo[f"{name}_meta"] = np.array([k, kt, tol, 1.0 if pre else 0.0, seed])
        if h.dim <= 5000:
            lo[f"{name}_dense_eigs"] = np.linalg.eigvalsh(rm.to_dense())[:k]
        print(name, "iterations", r.iterations, "converged", r.converged, r.eigenvalues)
    np.savez_compressed(os.path.join(OUT, "lobpcg.npz"), **lo)
    for f in sorted(os.listdir(OUT)):
        if f.endswith(".npz"):
            print(f, os.path.getsize(os.path.join(OUT, f)))


if __name__ == "__main__":
    if sys.argv[1:] == ["lanczos"]:
        make_lanczos()
    elif sys.argv[1:] == ["multilevel"]:
        make_multilevel()
    else:
        main()
        make_lanczos()
        make_multilevel()
