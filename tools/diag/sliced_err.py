"""Where does the sliced K1's error come from? Diagonal tiles only / full,
fp32 sector matrices; error vs the reference per column, and its location."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
from paper_1609_01689_b200 import ci
from oracle import ref
dev = ci.Device.default()
dev.set_spmm_mode("sliced")
for name, prm in (("diag tiles only", (30000, 3, 256, 0.0, 0.4, 77, 0, 2000)),
                  ("full", (30000, 3, 256, 0.02, 0.4, 77, 0, 2000)),
                  ("full, 1 sector", (30000, 1, 256, 0.02, 0.4, 77, 0, 2000))):
    h = ci.generate_sector_matrix(*prm)
    x = ci.random_block(h.dim, 16, 3)
    y = ci.spmm(h, x)
    yr = ref.RefMatrix(h).spmm(x, serial=True)
    err = np.abs(y - yr)
    i, j = np.unravel_index(err.argmax(), err.shape)
    print(f"{name}: rel {err.max() / np.abs(yr).max():.3e}  worst row {i} col {j}: y {y[i, j]:.17g} ref {yr[i, j]:.17g}", flush=True)
    # error by row position within a 128-row panel
    e_r = err.max(axis=1)
    print("   err by row%128 (max over 8 buckets):", [f"{e_r[(np.arange(h.dim) % 128) // 16 == b].max():.1e}" for b in range(8)])
dev.set_spmm_mode("auto")
# exactness probe: dyadic H (multiples of 1/64), integer X -> every path is exact
h = ci.generate_sector_matrix(30000, 3, 256, 0.0, 0.4, 77, 0, 2000)
vals = (np.round(h.values.astype(np.float64) * 64) / 64).astype(np.float32)
hq = ci.CsbMatrix(dim=h.dim, precision=0, block_boundaries=h.block_boundaries, entry_offsets=h.entry_offsets,
                  rows=h.rows, cols=h.cols, values=vals, groups=h.groups, beta=h.beta)
x = np.rint(ci.random_block(h.dim, 16, 3) * 4)
dev.set_spmm_mode("sliced")
y = ci.spmm(hq, x)
dev.set_spmm_mode("auto")
yr = ref.RefMatrix(hq).spmm(x, serial=True)
d = y - yr
bad = np.argwhere(d != 0)
print("dyadic exactness: mismatches", len(bad), "of", d.size, "max |d|", np.abs(d).max())
for i, j in bad[:8]:
    print("   row", i, "col", j, "y", repr(y[i, j]), "ref", repr(yr[i, j]), "d", d[i, j], "log2|d|", np.log2(abs(d[i, j])))
for label, hv, xv in (("dyadic H, full X", vals, ci.random_block(h.dim, 16, 3)),
                      ("full H, integer X", h.values, np.rint(ci.random_block(h.dim, 16, 3) * 4)),
                      ("full H, X=1", h.values, np.ones((h.dim, 16)))):
    hh = ci.CsbMatrix(dim=h.dim, precision=0, block_boundaries=h.block_boundaries, entry_offsets=h.entry_offsets,
                      rows=h.rows, cols=h.cols, values=hv, groups=h.groups, beta=h.beta)
    dev.set_spmm_mode("sliced")
    y = ci.spmm(hh, xv)
    dev.set_spmm_mode("auto")
    yr = ref.RefMatrix(hh).spmm(xv, serial=True)
    d = np.abs(y - yr)
    print(label, "max |d|", d.max(), "log2", np.log2(d.max() + 1e-300), "rel", d.max() / np.abs(yr).max())
