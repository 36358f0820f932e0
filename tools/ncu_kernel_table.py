"""Per-kernel table of an ncu --set full capture (several kernels): time,
DRAM bytes and bandwidth against the measured HBM peak, FP64-pipe
(DMMA + DFMA) utilisation, occupancy and registers. Used for the LOBPCG
block kernels in profiles/ (each kernel's bound from counters).
python tools/ncu_kernel_table.py rep.ncu-rep out.txt "<command>" """
import csv, io, json, os, subprocess, sys

rep, out, cmd = sys.argv[1], sys.argv[2], sys.argv[3]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, u = rows[0], rows[1]
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6, "usecond": 1e-6,
         "ms": 1e-3, "msecond": 1e-3, "nsecond": 1e-9, "s": 1.0, "second": 1.0}
peaks = json.load(open(os.path.join(os.path.dirname(__file__), "..", "MEASURED_PEAKS.json")))
hbm = None
for k, v in peaks.items():
    if "hbm" in k.lower() and isinstance(v, (int, float)):
        hbm = float(v)
        break


def val(r, k):
    if k not in h:
        return None
    s = r[h.index(k)].replace(",", "")
    try:
        return float(s) * scale.get(u[h.index(k)], 1.0)
    except ValueError:
        return None


keys = {"t": "gpu__time_duration.sum", "rd": "dram__bytes_read.sum", "wr": "dram__bytes_write.sum",
        "fp64": "TPC.TriageCompute.sm__pipe_fp64_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
        "tensor": "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
        "occ": "sm__warps_active.avg.pct_of_peak_sustained_active", "regs": "launch__registers_per_thread"}
lines = [f"# ncu --set full per-kernel table of: {cmd}",
         f"# HBM peak {hbm} GB/s (MEASURED_PEAKS.json); fp64/tensor = pipe-active % of elapsed",
         f"{'kernel':52s} {'us':>9s} {'GB':>7s} {'GB/s':>8s} {'%HBM':>6s} {'fp64%':>6s} {'tens%':>6s} {'occ%':>6s} {'regs':>5s}"]
for r in rows[2:]:
    name = r[h.index("Kernel Name")][:52]
    t = val(r, keys["t"]) or 0.0
    b = (val(r, keys["rd"]) or 0.0) + (val(r, keys["wr"]) or 0.0)
    gbs = b / t / 1e9 if t else 0.0
    f = lambda k: val(r, keys[k])
    lines.append(f"{name:52s} {t * 1e6:9.1f} {b / 1e9:7.3f} {gbs:8.0f} {100 * gbs / hbm if hbm else 0:6.1f} "
                 f"{(f('fp64') or 0):6.1f} {(f('tensor') or 0):6.1f} {(f('occ') or 0):6.1f} {int(f('regs') or 0):5d}")
open(out, "w").write("\n".join(lines) + "\n")
print("\n".join(lines))
