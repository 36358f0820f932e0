"""Driver for ncu captures of the Lanczos kernels on config 4 (GPU-generated
matrix): a short run of `steps` steps (argv[1], default 120)."""
import sys; sys.path.insert(0, ".")
from paper_1609_01689_b200 import ci, configs
cfg = configs.CFG4
dm = cfg.generate_device()
steps = int(sys.argv[1]) if len(sys.argv) > 1 else 120
rep = ci.lanczos_solve(dm, ci.lanczos_default_start(cfg.n, cfg.n // cfg.sectors),
                       ci.LanczosOptions(k_want=cfg.k_want, tol=cfg.tol, max_iter=steps))
print("ok", rep.iterations, rep.timing_ms)
