"""Scratch end-to-end check of the CUDA path against the reference oracle."""
import sys, time
import numpy as np
sys.path.insert(0, ".")
from paper_1609_01689_b200 import ci
from oracle import ref

def rel(a, b):
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))

h = ci.generate_sector_matrix(20000, 10, 64, 0.05, 0.5, seed=1, precision=1)
rm = ref.RefMatrix(h)
for m in (1, 4, 8, 13, 16, 32, 64):
    x = ci.random_block(h.dim, m, 7)
    yr = rm.spmm(x, serial=True)
    yg = ci.spmm(h, x)
    print("spmm fp64 m=%d rel %.3e" % (m, rel(yg, yr)), flush=True)
h32 = ci.generate_sector_matrix(60000, 3, 256, 0.02, 0.4, seed=3, precision=0)
rm32 = ref.RefMatrix(h32)
x = ci.random_block(h32.dim, 16, 9)
print("spmm fp32 m=16 rel %.3e" % rel(ci.spmm(h32, x), rm32.spmm(x, serial=True)), "tiles", ci.device_matrix(h32).ntiles, flush=True)
xa = ci.random_block(5000, 24, 1); ya = ci.random_block(5000, 20, 2)
print("block_inner rel %.3e" % rel(ci.block_inner(xa, ya), ref.block_inner(xa, ya)))
g = np.random.default_rng(0).standard_normal((24, 16))
print("lincomb rel %.3e" % rel(ci.linear_combination(xa, g), ref.linear_combination(xa, g)))
yy = ci.random_block(5000, 16, 5); y2 = yy.copy()
ci.add_linear_combination(y2, xa, g)
print("add_lincomb rel %.3e" % rel(y2, ref.add_linear_combination(yy, xa, g)))
# preconditioner
td_ref = ref.RefTileDiagonal(rm, h.groups)
td = ci.extract_tile_diagonal(h)
r = ci.random_block(h.dim, 8, 11)
mu = np.array([-3.0, -3.0, -2.5, -2.5, -2.5, 1.0, 1.0, 4.0]); en = np.array([1, 1, 1, 0, 1, 1, 0, 1], bool)
wg = ci.apply_preconditioner(td, r, ci.ShiftPlan(mu, en))
wr = ref.apply_preconditioner(td_ref, r, mu, en)
print("precond LU rel %.3e maxabs %.3e" % (rel(wg, wr), np.abs(wg - wr).max()))
td_ref32 = ref.RefTileDiagonal(rm32, h32.groups)
td32 = ci.extract_tile_diagonal(h32)
r32 = ci.random_block(h32.dim, 16, 12)
mu = np.linspace(-5, 5, 16); en = np.ones(16, bool); en[3] = False
wg = ci.apply_preconditioner(td32, r32, ci.ShiftPlan(mu, en))
wr = ref.apply_preconditioner(td_ref32, r32, mu, en)
print("precond FOM rel %.3e maxabs %.3e" % (rel(wg, wr), np.abs(wg - wr).max()))
# LOBPCG cfg1
x0 = ci.random_block(h.dim, 8, 42)
for use_prec in (False, True):
    t = time.time()
    rr = ref.lobpcg_solve(rm, x0, 4, 1e-8, 500, td_ref if use_prec else None)
    tr = time.time() - t
    t = time.time()
    rg = ci.lobpcg_solve(h, x0, ci.LobpcgOptions(k_want=4, tol=1e-8, preconditioner=td if use_prec else None))
    tg = time.time() - t
    print("lobpcg prec=%s ref it=%d conv=%s %.2fs | gpu it=%d conv=%s %.2fs" % (use_prec, rr.iterations, rr.converged, tr, rg.iterations, rg.converged, tg))
    print("  eig ref", rr.eigenvalues, "\n  eig gpu", rg.eigenvalues, " rel %.3e" % rel(rg.eigenvalues, rr.eigenvalues))
    print("  counters ref", rr.counters, "gpu", rg.counters, "timing", {k: round(v, 1) for k, v in rg.timing_ms.items()})
