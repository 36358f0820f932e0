"""Randomised LOBPCG stress against the live reference (test infrastructure,
not collected by pytest; needs oracle/_ref): iteration count, counters,
convergence and eigenvalues must match ci::lobpcg_solve exactly / to 1e-8
(fp64 H) / 1e-5 (fp32 H).
python tests/stress/lobpcg_stress.py <seed> <count>   (B200)"""
import sys, time; import os; sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))
import numpy as np
from oracle import ref as ref_lib
from paper_1609_01689_b200 import ci
rng2 = np.random.default_rng(int(sys.argv[1]))
bad = 0; t0 = time.time(); N = int(sys.argv[2])
for i in range(N):
    sectors = int(rng2.integers(2, 6)); tile = int(rng2.choice([16, 32, 64, 128, 256]))
    n = int(rng2.integers(600, 5000)) // sectors * sectors
    kt = int(rng2.choice([2, 3, 4, 6, 8, 12])); k = int(rng2.integers(1, max(2, kt // 2 + 1)))
    c = dict(n=n, sectors=sectors, tile=tile, p=float(rng2.uniform(0.1, 0.7)), q=float(rng2.uniform(0.2, 0.7)),
             seed=int(rng2.integers(1, 1 << 30)), precision=int(rng2.integers(0, 2)), band=int(rng2.integers(1, 3)),
             kt=kt, k=k, prec=bool(rng2.integers(0, 2)))
    h = ci.generate_sector_matrix(c["n"], c["sectors"], c["tile"], c["p"], c["q"], c["seed"], c["precision"], 2000, band=c["band"])
    tol = 1e-8 if c["precision"] == 1 else 1e-6
    x0 = ci.random_block(h.dim, c["kt"], c["seed"] % 997)
    td = ci.extract_tile_diagonal(h) if c["prec"] else None
    rep = ci.lobpcg_solve(h, x0, ci.LobpcgOptions(k_want=c["k"], tol=tol, preconditioner=td))
    rm = ref_lib.RefMatrix(h)
    rtd = ref_lib.RefTileDiagonal(rm, h.groups) if c["prec"] else None
    r = ref_lib.lobpcg_solve(rm, x0, c["k"], tol, 500, rtd)
    ok = rep.converged == r.converged and rep.iterations == r.iterations
    ok = ok and [rep.counters.spmm_calls, rep.counters.spmv_equivalents, rep.counters.precond_applications, rep.counters.orthogonalizations] == r.counters.tolist()
    ev = float(np.abs(rep.eigenvalues - r.eigenvalues).max() / np.abs(r.eigenvalues).max())
    ok = ok and ev <= (1e-8 if c["precision"] == 1 else 1e-5)
    if not ok:
        bad += 1
        print("MISMATCH", c, rep.iterations, r.iterations, rep.converged, r.converged, ev, flush=True)
print(f"lobpcg stress: {bad} mismatches of {N} in {time.time() - t0:.0f} s", flush=True)
