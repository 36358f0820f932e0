"""Reduce an ncu `--metrics gpu__time_duration.sum --csv` launch list to
(id, kernel, duration_ns) plus a per-kernel summary (profiles/)."""
import collections, csv, sys

src, out_csv, out_txt, cmd = sys.argv[1], sys.argv[2], sys.argv[3], sys.argv[4]
rows = list(csv.reader(open(src)))
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hi]
ix = {k: i for i, k in enumerate(h)}
scale = {"ns": 1, "nsecond": 1, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6}
out = [("id", "kernel", "duration_ns")]
agg = collections.OrderedDict()
for r in rows[hi + 1:]:
    if len(r) < len(h) or r[ix["Metric Name"]] != "gpu__time_duration.sum":
        continue
    v = float(r[ix["Metric Value"]].replace(",", "")) * scale[r[ix["Metric Unit"]]]
    name = r[ix["Kernel Name"]]
    out.append((r[ix["ID"]], name, int(round(v))))
    short = name.replace("(anonymous namespace)::", "").replace("<unnamed>::", "").replace("unnamed>::", "").split("(")[0]
    a = agg.setdefault(short, [0, 0.0])
    a[0] += 1
    a[1] += v
with open(out_csv, "w", newline="") as f:
    csv.writer(f).writerows(out)
tot = sum(a[1] for a in agg.values())
lines = [f"# ncu launch list of: {cmd}",
         "# cold-cache, serialised per-launch times (gpu__time_duration.sum, --clock-control none)",
         f"# launches {len(out) - 1}, sum of kernel time {tot / 1e6:.3f} ms",
         f"{'kernel':58s} {'launches':>8s} {'total_ms':>10s} {'share':>6s} {'avg_us':>10s}"]
for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    lines.append(f"{k[:58]:58s} {c:8d} {t / 1e6:10.3f} {100 * t / tot:5.1f}% {t / c / 1e3:10.1f}")
open(out_txt, "w").write("\n".join(lines) + "\n")
print("\n".join(lines[:14]))
