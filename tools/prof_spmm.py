"""Driver for ncu captures of K1: generate a config, upload, run a few SpMMs."""
import argparse, sys, time
sys.path.insert(0, ".")
import numpy as np
import torch
from paper_1609_01689_b200 import ci, configs

ap = argparse.ArgumentParser()
ap.add_argument("--cfg", default="cfg2-spmm")
ap.add_argument("--m", type=int, default=16)
ap.add_argument("--reps", type=int, default=4)
ap.add_argument("--scale", type=float, default=1.0, help="fraction of n (keeps density)")
a = ap.parse_args()
cfg = configs.ALL[a.cfg]
if a.scale != 1.0:
    import dataclasses
    n = int(cfg.n * a.scale) // cfg.sectors * cfg.sectors
    cfg = dataclasses.replace(cfg, n=n, target_nnz=None if cfg.target_nnz is None else cfg.target_nnz * a.scale,
                              p_stated=cfg.p())
h = cfg.generate()
dev = ci.Device(0)
dm = ci.DeviceMatrix(h, dev)
x = torch.from_numpy(ci.random_block(h.dim, a.m, 5)).cuda()
y = torch.empty_like(x)
torch.cuda.synchronize()
for _ in range(a.reps):
    dm.spmm_ptr(x.data_ptr(), y.data_ptr(), a.m)
dev.synchronize()
print("ok", h.dim, h.nnz_lower, dm.ntiles, dm.npanels)
