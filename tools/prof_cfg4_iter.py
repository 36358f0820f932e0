import sys; sys.path.insert(0, ".")
import numpy as np, torch
from paper_1609_01689_b200 import ci, configs
cfg = configs.CFG4
dm = cfg.generate_device()
td = ci.tile_diagonal_from_matrix(dm)
x0 = ci.random_block(cfg.n, cfg.kt, 42)
rep = ci.lobpcg_solve(dm, x0, ci.LobpcgOptions(k_want=cfg.k_want, tol=cfg.tol, max_iter=int(sys.argv[1]) if len(sys.argv) > 1 else 6, preconditioner=td))
print("ok", rep.iterations, rep.timing_ms)
