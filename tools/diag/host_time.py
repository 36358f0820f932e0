"""Config-2 host SpMM call (cieg_spmm_host, ci::spmm's call in the drop-in):
wall time per call on pageable and on pinned X/U (argv: m reps). Env:
CIEG_HOST_PIPELINE=0 keeps the unpipelined call; CIEG_HOST_CHUNKS=n sets the
chunk count of the pipelined one."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import torch
from paper_1609_01689_b200 import ci, configs
m = int(sys.argv[1]) if len(sys.argv) > 1 else 16
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
dev = ci.Device.default()
dm = configs.CFG2.generate_device()
dm.prepare(m)
x = ci.random_block(dm.dim, m, 5)
y = np.empty_like(x)
xp = torch.from_numpy(x).pin_memory()
yp = torch.empty_like(xp).pin_memory()
lib = ci._lib.load()
nbytes = configs.spmm_bytes(dm.nnz, dm.dim, m, 0)
ref = None
for name, xa, ya in (("pageable", x, y), ("pinned", xp.numpy(), yp.numpy()), ("pageable X / pinned U", x, yp.numpy()),
                     ("pinned X / pageable U", xp.numpy(), y)):
    for _ in range(3):
        ci._check(lib.cieg_spmm_host(dev.handle, dm.handle, ci._ptr(xa), ci._ptr(ya), m))
    t0 = time.perf_counter()
    for _ in range(reps):
        ci._check(lib.cieg_spmm_host(dev.handle, dm.handle, ci._ptr(xa), ci._ptr(ya), m))
    ms = (time.perf_counter() - t0) / reps * 1e3
    if ref is None:
        ref = ya.copy()
    same = bool(np.array_equal(ref, ya))
    print(f"cfg2 m={m} host {name} pipeline={os.environ.get('CIEG_HOST_PIPELINE', '1')} "
          f"chunks={os.environ.get('CIEG_HOST_CHUNKS', 'auto')}: {ms:.3f} ms {nbytes / ms / 1e6:.1f} GB/s same={same}",
          flush=True)
