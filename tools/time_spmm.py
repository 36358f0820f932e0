"""Time K1 alone on a config (GPU-generated matrix), CUDA events on the ctx stream."""
import argparse, sys
sys.path.insert(0, ".")
import torch
from paper_1609_01689_b200 import ci, configs

ap = argparse.ArgumentParser()
ap.add_argument("--cfg", default="cfg2-spmm")
ap.add_argument("--m", type=int, nargs="+", default=[16])
ap.add_argument("--reps", type=int, default=20)
ap.add_argument("--scale", type=float, default=1.0)
ap.add_argument("--te", type=int, default=0)
a = ap.parse_args()
cfg = configs.ALL[a.cfg]
if a.scale != 1.0:
    import dataclasses
    n = int(cfg.n * a.scale) // cfg.sectors * cfg.sectors
    cfg = dataclasses.replace(cfg, n=n, target_nnz=None, p_stated=cfg.p())
dev = ci.Device(0)
s = torch.cuda.Stream()
torch.cuda.set_stream(s)
dev.set_stream(s.cuda_stream)
import time; _t = time.time()
dm = ci.DeviceMatrix.generate(cfg.n, cfg.sectors, cfg.tile, cfg.p(), cfg.q, cfg.seed, cfg.precision, cfg.beta,
                             device=dev, tile_edge=a.te)
print(f"generate_device {time.time() - _t:.2f} s", flush=True)
S = dm.nnz
for m in a.m:
    x = torch.randn(cfg.n, m, dtype=torch.float64, device="cuda")
    y = torch.empty_like(x)
    for _ in range(3):
        dm.spmm_ptr(x.data_ptr(), y.data_ptr(), m)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(s)
    for _ in range(a.reps):
        dm.spmm_ptr(x.data_ptr(), y.data_ptr(), m)
    e1.record(s)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / a.reps
    gb = configs.spmm_bytes(S, cfg.n, m, cfg.precision) / ms / 1e6
    print(f"{cfg.name} m={m} {ms:.3f} ms {gb:.1f} GB/s", flush=True)
