import sys; sys.path.insert(0, ".")
import numpy as np, torch
from paper_1609_01689_b200 import ci, configs
cfg = configs.CFG2
dm = cfg.generate_device()
td = ci.tile_diagonal_from_matrix(dm)
r = ci.random_block(cfg.n, 16, 3)
mu = np.full(16, -3.0)
for _ in range(2):
    w = ci.apply_preconditioner(td, r, ci.ShiftPlan(mu, np.ones(16, bool)))
print("ok", w.shape)
