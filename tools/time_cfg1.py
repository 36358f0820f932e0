"""Config-1 LOBPCG solve time, repeated (phase split vs total)."""
import sys, time
sys.path.insert(0, ".")
from paper_1609_01689_b200 import ci, configs

cfg = configs.CFG1
h = cfg.generate()
td = ci.extract_tile_diagonal(h)
x0 = ci.random_block(h.dim, cfg.kt, 42)
opt = ci.LobpcgOptions(k_want=cfg.k_want, tol=cfg.tol, preconditioner=td)
for r in range(5):
    t0 = time.perf_counter()
    rep = ci.lobpcg_solve(h, x0, opt)
    ms = (time.perf_counter() - t0) * 1e3
    parts = sum(v for k, v in rep.timing_ms.items() if k != "total")
    print(f"run {r}: wall {ms:.1f} ms  total {rep.timing_ms['total']:.1f}  phases {parts:.1f}  iters {rep.iterations}  "
          + " ".join(f"{k} {v:.1f}" for k, v in rep.timing_ms.items() if k != "total"))
