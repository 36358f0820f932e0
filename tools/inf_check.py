import sys; sys.path.insert(0, ".")
import numpy as np
from conftest import gen_from
from paper_1609_01689_b200 import ci
from oracle import ref
h = gen_from((3072, 3, 256, 0.2, 0.4, 13, 0, 2000))
x = ci.random_block(h.dim, 4, 1)
x[100, 0] = np.inf
x[200, 1] = np.nan
y = ci.spmm(h, x)
yr = ref.RefMatrix(h).spmm(x, serial=True)
for c in range(2):
    print("col", c, "gpu nonfinite rows", int((~np.isfinite(y[:, c])).sum()), "ref nonfinite rows", int((~np.isfinite(yr[:, c])).sum()))
fin = np.isfinite(yr)
print("finite-ref entries that differ:", int((~np.isclose(y[fin], yr[fin], rtol=1e-12, atol=1e-12)).sum()))
