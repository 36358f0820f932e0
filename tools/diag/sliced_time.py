"""Config-2 SpMM device time per call in one K1 mode (default sliced), m = 16
(argv: m mode reps). Env knobs (CIEG_SLICED_ABLATE ...) are read by the library."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_1609_01689_b200 import ci, configs
m = int(sys.argv[1]) if len(sys.argv) > 1 else 16
mode = sys.argv[2] if len(sys.argv) > 2 else "sliced"
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 10
dev = ci.Device.default()
dev.set_spmm_mode(mode)
dm = configs.CFG2.generate_device()
x = torch.from_numpy(ci.random_block(dm.dim, m, 5)).cuda()
y = torch.empty_like(x)
own = torch.cuda.ExternalStream(dev.stream)
for _ in range(3):
    dm.spmm_ptr(x.data_ptr(), y.data_ptr(), m)
dev.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(own)
for _ in range(reps):
    dm.spmm_ptr(x.data_ptr(), y.data_ptr(), m)
e1.record(own)
e1.synchronize()
ms = e0.elapsed_time(e1) / reps
nbytes = configs.spmm_bytes(dm.nnz, dm.dim, m, 0)
print(f"cfg2 m={m} {mode} ablate={os.environ.get('CIEG_SLICED_ABLATE', '0')}: {ms:.3f} ms {nbytes / ms / 1e6:.1f} GB/s", flush=True)
