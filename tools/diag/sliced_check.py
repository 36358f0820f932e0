"""Quick check of the int8 tensor-core K1 (sliced mode): accuracy against the
reference on a small matrix, then config-2 timing against owner-computes."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import torch
from paper_1609_01689_b200 import ci, configs
from oracle import ref

def relc(a, b):
    s = np.maximum(np.abs(b).max(axis=0), 1e-300)
    return float((np.abs(a - b).max(axis=0) / s).max())

dev = ci.Device.default()
h = ci.generate_sector_matrix(30000, 3, 256, 0.02, 0.4, 77, 0, 2000)
rm = ref.RefMatrix(h)
for m in (16, 9, 3, 1):
    x = ci.random_block(h.dim, m, 100 + m)
    yr = rm.spmm(x, serial=True)
    dev.set_spmm_mode("sliced")
    t = time.time(); y = ci.spmm(h, x); dt = time.time() - t
    dev.set_spmm_mode("owner")
    yo = ci.spmm(h, x)
    print(f"small m={m}: sliced rel {relc(y, yr):.3e} (owner {relc(yo, yr):.3e}) first call {dt:.2f}s", flush=True)
if len(sys.argv) > 1 and sys.argv[1] == "small":
    sys.exit(0)
dm = configs.CFG2.generate_device()
n, m = dm.dim, 16
x = torch.from_numpy(ci.random_block(n, m, 5)).cuda()
y = torch.empty_like(x)
nbytes = configs.spmm_bytes(dm.nnz, n, m, 0)
stream = torch.cuda.current_stream()
for mode in ("sliced", "owner", "single"):
    dev.set_spmm_mode(mode)
    dm.spmm_ptr(x.data_ptr(), y.data_ptr(), m)
    dev.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    own = torch.cuda.ExternalStream(dev.stream)
    e0.record(own)
    for _ in range(10):
        dm.spmm_ptr(x.data_ptr(), y.data_ptr(), m)
    e1.record(own)
    e1.synchronize()
    ms = e0.elapsed_time(e1) / 10
    out = y.cpu().numpy()
    if mode == "sliced":
        ys = out
        dm.spmm_ptr(x.data_ptr(), y.data_ptr(), m)
        dev.synchronize()
        print(f"cfg2 sliced run-to-run bitwise equal: {bool((y.cpu().numpy() == ys).all())}", flush=True)
    print(f"cfg2 m=16 {mode}: {ms:.3f} ms  {nbytes / ms / 1e6:.1f} GB/s  rel vs sliced {relc(ys, out):.3e}", flush=True)
dev.set_spmm_mode("auto")
