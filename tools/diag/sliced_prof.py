"""Config-2 K1 in sliced mode, a few launches (for ncu)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_1609_01689_b200 import ci, configs
m = int(sys.argv[1]) if len(sys.argv) > 1 else 16
mode = sys.argv[2] if len(sys.argv) > 2 else "sliced"
dev = ci.Device.default()
dev.set_spmm_mode(mode)
dm = configs.CFG2.generate_device()
x = torch.from_numpy(ci.random_block(dm.dim, m, 5)).cuda()
y = torch.empty_like(x)
for _ in range(3):
    dm.spmm_ptr(x.data_ptr(), y.data_ptr(), m)
dev.synchronize()
print("done", flush=True)
