"""Is the kt=16 unpreconditioned iteration count rounding-sensitive? Runs the
same problem through every K1 mode and the reference; reports iteration
counts and the first iteration whose active set differs from the reference."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
from paper_1609_01689_b200 import configs, ci
from oracle import ref

n_per, per_row, seed, xs = (int(a) for a in (sys.argv[1:5] if len(sys.argv) > 4 else (1088, 300, 11, 9)))
n = 25 * n_per
c = configs.Config("cfg4-shape", n, 25, 256, None, 0.4, 0, n * per_row, k_want=8, kt=16, tol=1e-6, seed=seed)
h = c.generate()
x0 = ci.random_block(n, 16, xs)
rm = ref.RefMatrix(h)
t = time.time()
rr = ref.lobpcg_solve(rm, x0, 8, 1e-6, 500, None)
print("ref", rr.iterations, rr.converged, round(time.time() - t, 1), flush=True)
ra = np.asarray(rr.history.relres).reshape(-1, 16)
dev = ci.Device.default()
for mode in ("auto", "owner", "single", "sliced"):
    dev.set_spmm_mode(mode)
    rep = ci.lobpcg_solve(h, x0, ci.LobpcgOptions(k_want=8, tol=1e-6))
    ga = np.array([r.relres for r in rep.history]).reshape(-1, 16)
    k = min(len(ga), len(ra))
    diff = [i for i in range(k) if not np.array_equal(ga[i] > 1e-6, ra[i] > 1e-6)]
    rel = np.abs(ga[:k] - ra[:k]) / np.maximum(ra[:k], 1e-300)
    first = diff[0] if diff else None
    print(mode, rep.iterations, rep.converged, "first active-set diff at", first,
          "max rel relres diff over first 50 it", float(rel[:50].max()), flush=True)
    if first is not None:
        print("  ref relres", ra[first], "\n  gpu relres", ga[first], flush=True)
dev.set_spmm_mode("auto")
