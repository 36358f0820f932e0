"""Randomised K1 stress (test infrastructure, not collected by pytest):
random generator configs and widths, Inf/NaN injection, every SpMM mode and
world-2 single-pass shards against the oracle's restatement of spmm.
python tests/stress/spmm_stress.py <seed> [big]   (B200; 120 configs, ~1 min; "big": CSB
block bounds up to 65535 rows, n up to 2e5)"""
import sys, time; import os; sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "..")); sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np
from conftest import single_pass_shards
from oracle import ci_oracle as O
from paper_1609_01689_b200 import ci
rng = np.random.default_rng(int(sys.argv[1]) if len(sys.argv) > 1 else 1)
dev = ci.Device.default()
bad = 0
t0 = time.time()
for it in range(40 if len(sys.argv) > 2 and sys.argv[2] == 'big' else 120):
    sectors = int(rng.integers(1, 6)); tile = int(rng.choice([8, 16, 32, 50, 64, 96, 128, 256]))
    big = len(sys.argv) > 2 and sys.argv[2] == "big"  # maximum CSB block bounds, larger dimensions
    n = int(rng.integers(max(sectors, 30), 200_000 if big else 5000)) // sectors * sectors
    beta = int(rng.choice([4096, 30000, 65535])) if big else max(tile, 256)
    prm = dict(n=n, sectors=sectors, tile=tile, p=float(rng.uniform(0.05, 1.0)) * (0.02 if big else 1.0),
               q=float(rng.uniform(0.05, 1.0)), seed=int(rng.integers(1, 1 << 30)),
               precision=int(rng.integers(0, 2)), beta=max(beta, tile), band=int(rng.integers(0, 4)))
    m = int(rng.choice([1, 2, 3, 5, 8, 9, 13, 16, 17, 31]))
    h = ci.generate_sector_matrix(prm["n"], prm["sectors"], prm["tile"], prm["p"], prm["q"], prm["seed"], prm["precision"], prm["beta"], band=prm["band"])
    x = ci.random_block(h.dim, m, it)
    if rng.random() < 0.2:
        x[int(rng.integers(0, h.dim)), int(rng.integers(0, m))] = float(rng.choice([np.inf, -np.inf, np.nan]))
    yo = O.spmm(h, x)
    fin = np.isfinite(yo)
    scale = max(np.abs(yo[fin]).max() if fin.any() else 1.0, 1e-300)
    dm = ci.DeviceMatrix(h)
    outs = {}
    for mode in ("auto", "owner", "single"):
        dev.set_spmm_mode(mode)
        outs[mode] = dm.spmm_host(x)
    dev.set_spmm_mode("auto")
    if len(h.groups) > 2 and n > 200:
        outs["shards2"] = single_pass_shards(h, 2, m, x)
    for k, y in outs.items():
        ok = all(np.array_equal(f(y), f(yo)) for f in (np.isnan, np.isposinf, np.isneginf))
        ok = ok and np.abs(y[fin] - yo[fin]).max(initial=0.0) <= 1e-13 * scale
        if not ok:
            bad += 1
            print("MISMATCH", it, k, prm, m, flush=True)
print(f"done {bad} mismatches in {time.time() - t0:.0f} s", flush=True)
