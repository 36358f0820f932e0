"""Summarise an ncu source-page CSV: stall reasons per code region (split at
the first DMMA-containing block = consumer) and the top instructions."""
import csv, subprocess, sys
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[1]
ix = {k: i for i, k in enumerate(hdr)}
reasons = [k for k in hdr if k.startswith("stall_") and "Not Issued" not in k]
recs = []
for r in rows[2:]:
    if len(r) < len(hdr):
        continue
    recs.append(r)
# consumer region: from first DMMA-block label backwards is hard; use marker instructions
first_dmma = next(i for i, r in enumerate(recs) if "DMMA" in r[ix["Source"]])
# find the consumer entry: the BAR.ARV issued twice at consumer start precedes the DMMA loop
split = first_dmma
for i in range(first_dmma, -1, -1):
    if "BAR.ARV" in recs[i][ix["Source"]]:
        split = i
        break
def summarise(sub, name):
    tot = {k: 0 for k in reasons}
    for r in sub:
        for k in reasons:
            try:
                tot[k] += int(r[ix[k]] or 0)
            except ValueError:
                pass
    s = sum(tot.values())
    print(f"== {name}: {s} samples")
    for k, v in sorted(tot.items(), key=lambda x: -x[1])[:8]:
        print(f"   {k:22s} {v:8d} {100*v/max(s,1):5.1f}%")
summarise(recs[:split - 5], "producer (+prologue)")
summarise(recs[split - 5:], "consumer")
if len(sys.argv) > 2:
    top = int(sys.argv[2])
    def tot(r):
        s = 0
        for k in reasons:
            try:
                s += int(r[ix[k]] or 0)
            except ValueError:
                pass
        return s
    print("== top instructions (addr, total, long_sb, wait, barrier, source)")
    for i, r in sorted(enumerate(recs), key=lambda x: -tot(x[1]))[:top]:
        g = lambda k: r[ix[k]] if k in ix else "?"
        print(f"  {i:5d} {tot(r):7d} lsb={g('stall_long_sb'):>6s} wait={g('stall_wait'):>6s} bar={g('stall_barrier'):>6s} "
              f"ssb={g('stall_short_sb'):>6s} {'P' if i < split - 5 else 'C'} {r[ix['Source']][:70]}")
