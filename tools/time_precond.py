import sys, time; sys.path.insert(0, ".")
import numpy as np, torch
from paper_1609_01689_b200 import ci, configs
for cfg in (configs.CFG2, configs.CFG4):
    dm = cfg.generate_device()
    td = ci.tile_diagonal_from_matrix(dm)
    r = ci.random_block(cfg.n, 16, 3)
    mu = np.full(16, -3.0)
    ci.apply_preconditioner(td, r, ci.ShiftPlan(mu, np.ones(16, bool)))
    t = time.time()
    for _ in range(3):
        w = ci.apply_preconditioner(td, r, ci.ShiftPlan(mu, np.ones(16, bool)))
    print(cfg.name, "precond incl. host copies ms", (time.time() - t) / 3 * 1e3)
    del td, dm
