"""Refresh profiles/traffic.json's "cfg2-spmm" entry from the ncu CSV of
tools/diag/sliced_prof.py (dram__bytes_read.sum, dram__bytes_write.sum,
gpu__time_duration.sum): the kernels of the LAST SpMM call in the capture.
usage: traffic_update.py CSV [source-note]"""
import collections, csv, io, json, os, sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
src = sys.argv[1]
txt = open(src).read()
rows = list(csv.DictReader(io.StringIO(txt[txt.index('"ID"'):])))
launches = collections.OrderedDict()
for r in rows:
    k = int(r["ID"])
    d = launches.setdefault(k, {"name": r["Kernel Name"]})
    d[r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
ids = sorted(launches)
# the last call = from the last digitize_kernel launch to the end
start = max(i for i in ids if "digitize_kernel" in launches[i]["name"])
call = [launches[i] for i in ids if i >= start]
def short(n):
    n = n.replace("<unnamed>::", "").replace("unnamed>::", "").replace("(anonymous namespace)::", "")
    n = n.split("(")[0].replace("void ", "").strip()
    return n
per = collections.OrderedDict()
for d in call:
    per[short(d["name"])] = [int(d["dram__bytes_read.sum"]), int(d["dram__bytes_write.sum"]), int(d["gpu__time_duration.sum"])]
rd = sum(v[0] for v in per.values())
wr = sum(v[1] for v in per.values())
path = os.path.join(REPO, "profiles", "traffic.json")
t = json.load(open(path))
old = t["cfg2-spmm"]
t["cfg2-spmm"] = {
    "kernel": "sliced (int8 tcgen05): " + " + ".join(per) + ", the m = 16 default (round 2, final)",
    "m": 16,
    "per_kernel": {k: v[:2] for k, v in per.items()},
    "per_kernel_ns_under_ncu": {k: v[2] for k, v in per.items()},
    "dram_bytes_read": rd,
    "dram_bytes_write": wr,
    "algorithmic_bytes_per_launch": old["algorithmic_bytes_per_launch"],
    "source": (sys.argv[2] if len(sys.argv) > 2 else src) +
              " (tools/evidence_r2.sh: ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum "
              "--clock-control none, last SpMM call of tools/diag/sliced_prof.py), round 2",
    "note": "four dense slice planes (64 KB per stored tile, zeros included) + the sparse lowest-slice lists streamed once by "
            "TMA; partner X digit slabs (L2 misses); the fixed-point Y (yint) written by integer reds and read / cleared by "
            "yint_to_y_kernel",
    "traffic_per_launch": rd + wr,
}
json.dump(t, open(path, "w"), indent=1)
print(json.dumps(t["cfg2-spmm"], indent=1))
