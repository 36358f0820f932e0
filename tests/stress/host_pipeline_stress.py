"""Randomised stress of the chunk-pipelined host SpMM (test infrastructure,
not collected by pytest): random fp32 sector matrices with 128-row panels
(banded and unbanded, ragged sector tails), widths 2..16, chunk counts 1..40,
pageable and pinned buffers, Inf/NaN injection -- every pipelined call bitwise
the one-launch device call, and that one within 1e-13 of the oracle.
python tests/stress/host_pipeline_stress.py <seed> [configs]   (B200; 60 configs, ~2 min)"""
import sys, time; import os; sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "..")); sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np
import torch
from oracle import ci_oracle as O
from paper_1609_01689_b200 import ci
rng = np.random.default_rng(int(sys.argv[1]) if len(sys.argv) > 1 else 1)
count = int(sys.argv[2]) if len(sys.argv) > 2 else 60
dev = ci.Device.default()
dev.set_spmm_mode("sliced")
lib = ci._lib.load()
bad = 0
t0 = time.time()
for it in range(count):
    sectors = int(rng.integers(1, 14)); tile = int(rng.choice([128, 256, 200, 384]))
    n = int(rng.integers(max(sectors * 130, 600), 60000)) // sectors * sectors
    prm = dict(n=n, sectors=sectors, tile=tile, p=float(rng.uniform(0.01, 0.2)), q=float(rng.uniform(0.1, 0.8)),
               seed=int(rng.integers(1, 1 << 30)), band=int(rng.integers(0, 4)))
    m = int(rng.integers(2, 17))
    h = ci.generate_sector_matrix(prm["n"], prm["sectors"], prm["tile"], prm["p"], prm["q"], prm["seed"], 0, 2000, band=prm["band"])
    dm = ci.DeviceMatrix(h)
    if dm.spmm_kernel(m) != "sliced":
        continue
    x = ci.random_block(h.dim, m, it)
    if rng.random() < 0.25:
        x[int(rng.integers(0, h.dim)), int(rng.integers(0, m))] = float(rng.choice([np.inf, -np.inf, np.nan]))
    xd = torch.from_numpy(x).cuda(); yd = torch.empty_like(xd)
    torch.cuda.synchronize()
    dm.spmm_ptr(xd.data_ptr(), yd.data_ptr(), m); dev.synchronize()
    y_one = yd.cpu().numpy()
    yo = O.spmm(h, x)
    fin = np.isfinite(yo)
    scale = np.maximum(np.abs(np.where(fin, yo, 0.0)).max(axis=0), 1e-300)
    ok = all(np.array_equal(f(y_one), f(yo)) for f in (np.isnan, np.isposinf, np.isneginf))
    ok = ok and bool((np.abs(np.where(fin, y_one - yo, 0.0)).max(axis=0) <= 1e-13 * scale).all())
    if not ok:
        bad += 1; print("MISMATCH vs oracle", it, prm, m, flush=True)
    xp = torch.from_numpy(x).pin_memory(); yp = torch.empty_like(xp).pin_memory()
    for chunks in sorted(set(int(c) for c in rng.integers(1, 41, 3))):
        os.environ["CIEG_HOST_CHUNKS"] = str(chunks)
        y = dm.spmm_host(x)
        ci._check(lib.cieg_spmm_host(dev.handle, dm.handle, ci._ptr(xp.numpy()), ci._ptr(yp.numpy()), m))
        for name, out in (("pageable", y), ("pinned", yp.numpy())):
            if not np.array_equal(out, y_one, equal_nan=True):
                bad += 1; print("MISMATCH pipelined", name, it, chunks, prm, m, flush=True)
print(f"done {count} configs, {bad} mismatches in {time.time() - t0:.0f} s", flush=True)
