"""Config-4 LOBPCG time-to-solution on one B200 (generated on the GPU)."""
import json, sys, time
sys.path.insert(0, ".")
import numpy as np
import torch
from paper_1609_01689_b200 import ci, configs

cfg = configs.CFG4
max_iter = int(sys.argv[1]) if len(sys.argv) > 1 else 500
t0 = time.time()
dm = cfg.generate_device()
td = ci.tile_diagonal_from_matrix(dm)
torch.cuda.synchronize()
t_gen = time.time() - t0
x0 = ci.random_block(cfg.n, cfg.kt, 42)
t0 = time.time()
rep = ci.lobpcg_solve(dm, x0, ci.LobpcgOptions(k_want=cfg.k_want, tol=cfg.tol, max_iter=max_iter, preconditioner=td))
tts = time.time() - t0
relres = np.array([r.relres for r in rep.history]).reshape(-1, cfg.kt)
print(json.dumps({"workload": cfg.name, "n": cfg.n, "nnz": dm.nnz, "gen_s": round(t_gen, 2), "tts_s": round(tts, 3),
                  "iterations": rep.iterations, "converged": rep.converged,
                  "split_ms": {k: round(v, 1) for k, v in rep.timing_ms.items()},
                  "counters": vars(rep.counters), "eigenvalues": rep.eigenvalues.tolist(),
                  "final_relres": relres[-1, :cfg.k_want].tolist()}))
