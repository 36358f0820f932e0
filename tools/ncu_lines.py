"""Top CUDA source lines of an ncu --set full --import-source capture by
warp-stall samples, with the dominant stall reasons per line.
usage: python tools/ncu_lines.py REPORT.ncu-rep [N]"""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
hdr = rows[hi]
ix = {k: i for i, k in enumerate(hdr)}
reasons = [k for k in hdr if k.startswith("stall_") and "Not Issued" not in k]


def val(r, k):
    try:
        return int(float(r[ix[k]] or 0))
    except (ValueError, IndexError):
        return 0


recs = [r for r in rows[hi + 1:] if len(r) == len(hdr)]
tot_all = {k: sum(val(r, k) for r in recs) for k in reasons}
s = sum(tot_all.values())
print(f"== all lines: {s} samples")
for k, v in sorted(tot_all.items(), key=lambda x: -x[1])[:10]:
    print(f"   {k:24s} {v:9d} {100 * v / max(s, 1):5.1f}%")
print("== top lines")
for r in sorted(recs, key=lambda r: -sum(val(r, k) for k in reasons))[:top]:
    t = sum(val(r, k) for k in reasons)
    if t == 0:
        break
    br = sorted(((val(r, k), k[6:]) for k in reasons), reverse=True)[:3]
    print(f"  {r[ix['Line No']]:>5s} {t:8d} {100 * t / max(s, 1):5.1f}%  " + " ".join(f"{k}={v}" for v, k in br) +
          f"  | {r[ix['Source']].strip()[:80]}")
