"""Randomised Lanczos stress against the live reference (test infrastructure,
not collected by pytest; needs oracle/_ref): step count and convergence must
match ci::lanczos_solve, Ritz values to 1e-10 relative.
python tests/stress/lanczos_stress.py <seed> <count>   (B200)"""
import os
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))
import numpy as np  # noqa: E402

from oracle import ref as ref_lib  # noqa: E402
from paper_1609_01689_b200 import ci  # noqa: E402

rng = np.random.default_rng(int(sys.argv[1]))
count = int(sys.argv[2])
bad = 0
t0 = time.time()
for _ in range(count):
    sectors = int(rng.integers(2, 6))
    n = int(rng.integers(600, 4000)) // sectors * sectors
    c = dict(n=n, sectors=sectors, tile=int(rng.choice([16, 32, 64, 128, 256])), p=float(rng.uniform(0.1, 0.7)),
             q=float(rng.uniform(0.2, 0.7)), seed=int(rng.integers(1, 1 << 30)), precision=int(rng.integers(0, 2)),
             k=int(rng.integers(1, 6)))
    h = ci.generate_sector_matrix(c["n"], c["sectors"], c["tile"], c["p"], c["q"], c["seed"], c["precision"], 2000)
    v0 = ci.lanczos_default_start(h.dim, h.dim // c["sectors"])
    rep = ci.lanczos_solve(h, v0, ci.LanczosOptions(k_want=c["k"], tol=1e-8, max_iter=300))
    r = ref_lib.lanczos_solve(ref_lib.RefMatrix(h), v0, c["k"], 1e-8, 300)
    ev = float(np.abs(rep.eigenvalues - r.eigenvalues).max() / np.abs(r.eigenvalues).max())
    if not (rep.converged == r.converged and rep.iterations == r.iterations and ev <= 1e-10):
        bad += 1
        print("MISMATCH", c, rep.iterations, r.iterations, rep.converged, r.converged, ev, flush=True)
print(f"lanczos stress: {bad} mismatches of {count} in {time.time() - t0:.0f} s", flush=True)
