"""Timeline of CTA 0 of the sliced K1 on config 2 (CIEG_SLICED_TRACE)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
path = "/tmp/sliced_trace.bin"
os.environ["CIEG_SLICED_TRACE"] = path
import numpy as np
import torch
from paper_1609_01689_b200 import ci, configs
dev = ci.Device.default()
dev.set_spmm_mode("sliced")
dm = configs.CFG2.generate_device()
x = torch.from_numpy(ci.random_block(dm.dim, 16, 5)).cuda()
y = torch.empty_like(x)
for _ in range(3):
    dm.spmm_ptr(x.data_ptr(), y.data_ptr(), 16)
dev.synchronize()
raw = np.fromfile(path, dtype=np.int64)
t = raw[:4096].reshape(256, 16)
extra = raw[4096:]
hist = extra[:33]
if len(hist) and hist.sum():
    print("scatter pass bank-conflict degree histogram (CTA 0):", {i: int(v) for i, v in enumerate(hist) if v})
    print("mean wavefronts per pass: %.3f" % ((hist * np.arange(33)).sum() / hist.sum()))
if len(extra) > 41 and extra[41]:
    print("ticket waits (CTA 0): %d, mean %.0f cycles" % (extra[41], extra[40] / extra[41]))
n = int((t[:, 0] != 0).sum())
t = t[:n]
t0 = t[0, 0]
names = {0: "M.start", 1: "M.fullA", 2: "M.accE", 3: "M.issued", 8: "P.start", 4: "P.emptyA", 5: "P.zeroed",
         6: "P.scattered", 7: "P.arrived", 9: "R.top", 10: "R.acc", 11: "R.accF", 12: "R.recomb", 13: "R.done", 14: "T.accF", 15: "T.done"}
print("items traced", n)
print("item " + " ".join(f"{names[k]:>10s}" for k in sorted(names)))
for i in range(min(n, 40)):
    print(f"{i:4d} " + " ".join(f"{(t[i, k] - t0) if t[i, k] else -1:10d}" for k in sorted(names)))
d = np.diff(t[:, 0])
print("per item (cycles): M.start diff median", np.median(d))
for a_, b_, lab in ((8, 4, "P wait emptyA"), (4, 5, "P zero+bar"), (5, 6, "P scatter"), (0, 1, "M wait fullA"),
                    (1, 2, "M wait accE"), (2, 3, "M issue"), (11, 12, "R recombine"), (12, 13, "R rest"), (13, 10, "R yacc"), (9, 11, "R wait")):
    print(f"{lab:16s} median {np.median(t[2:, b_] - t[2:, a_]):8.0f}")
# steady-state gaps (items 4..n-2), including the back edges of each role's loop
s = slice(4, n - 1)
def med(a, b, nxt=False):
    return float(np.median((t[5:n, a] if nxt else t[s, a]) - t[s, b])) if n > 6 else 0.0
print("R: accF->recomb %.0f, recomb->done %.0f, done->acc %.0f, acc->next top %.0f, top->accF %.0f" % (
    med(12, 11), med(13, 12), med(10, 13), med(9, 10, True), med(11, 9)))
print("T: accF->done %.0f, done->next accF %.0f" % (med(15, 14), med(14, 15, True)))
print("M: start->fullA %.0f, fullA->accE %.0f, accE->issued %.0f, issued->next start %.0f" % (
    med(1, 0), med(2, 1), med(3, 2), med(0, 3, True)))
np.save("gpurun_out/sliced_trace_last.npy", t)
