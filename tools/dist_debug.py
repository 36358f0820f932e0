import os, sys, time
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import numpy as np
import torch, torch.distributed as dist
rank = int(os.environ.get("RANK", "0")); world = int(os.environ.get("WORLD_SIZE", "1"))
backend = sys.argv[1]
def log(*a):
    print(f"[{rank}] {time.time():.1f}", *a, flush=True)
torch.cuda.set_device(0)
if backend == "nccl":
    dist.init_process_group("nccl", device_id=torch.device("cuda", 0))
else:
    dist.init_process_group("gloo")
log("init ok")
from conftest import gen_from
from paper_1609_01689_b200 import ci, dist as D
g = dict(np.load("tests/golden/lobpcg.npz"))
name = "sector_f64"
h = gen_from(g[f"{name}_params"])
k, kt, tol, pre, seed = g[f"{name}_meta"]
dev = ci.Device(0)
sm = D.ShardedMatrix(h, rank, world, dev)
log("shard", sm.row_lo, sm.row_hi)
t = torch.ones(3, device="cuda") * (rank + 1)
D.allreduce_sum_(t); log("allreduce", t.tolist())
x = ci.random_block(h.dim, 7, 3)
y = sm.spmm(torch.from_numpy(x[sm.row_lo:sm.row_hi].copy()).cuda()).cpu().numpy()
log("spmm ok", np.abs(y - ci.spmm(h, x)[sm.row_lo:sm.row_hi]).max())
x0 = ci.random_block(h.dim, int(kt), int(seed))[sm.row_lo:sm.row_hi]
rep = D.lobpcg_solve_dist(sm, x0, ci.LobpcgOptions(k_want=int(k), tol=float(tol), max_iter=5))
log("solve ok", rep.iterations, rep.eigenvalues)
dist.destroy_process_group()
