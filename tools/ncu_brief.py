"""Summarise one kernel of an ncu --set full capture for profiles/: the key
throughput / traffic / pipe metrics and the warp-stall split with the
hottest SASS lines. usage: ncu_brief.py report.ncu-rep out.txt [algorithmic_bytes]"""
import csv, io, subprocess, sys

rep, out_txt = sys.argv[1], sys.argv[2]
alg = float(sys.argv[3]) if len(sys.argv) > 3 else None
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, u, v = rows[0], rows[1], rows[2]
get = lambda k: (v[h.index(k)], u[h.index(k)]) if k in h else ("n/a", "")
keys = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_subpipe_imma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__issue_active.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
        "launch__shared_mem_per_block_dynamic", "sm__cycles_active.avg"]
lines = [f"# ncu --set full --import-source on --clock-control none: {rep.split('/')[-1]}"]
for k in keys:
    val, unit = get(k)
    lines.append(f"{k:70s} {val} {unit}")
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
try:
    rd = float(get("dram__bytes_read.sum")[0].replace(",", "")) * scale[get("dram__bytes_read.sum")[1]]
    wr = float(get("dram__bytes_write.sum")[0].replace(",", "")) * scale[get("dram__bytes_write.sum")[1]]
    lines.append(f"{'dram traffic per launch (read + write)':70s} {rd + wr:.4e} bytes")
    if alg:
        lines.append(f"{'algorithmic bytes per launch':70s} {alg:.4e} bytes")
        lines.append(f"{'traffic / algorithmic':70s} {(rd + wr) / alg:.3f}")
except Exception:
    pass
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
srows = list(csv.reader(io.StringIO(src)))
sh = srows[1]
data = srows[2:]
ix = {n: i for i, n in enumerate(sh)}
def f(r, k):
    try:
        return float(r[ix[k]].replace(",", ""))
    except Exception:
        return 0.0
stalls = [k for k in sh if k.startswith("stall_") and "Not" not in k]
tot = {k: sum(f(r, k) for r in data) for k in stalls}
s = sum(tot.values()) or 1.0
lines.append("")
lines.append("# warp-stall samples, all warps: " + ", ".join(f"{k[6:]} {100 * t / s:.1f}%" for t, k in
                                                       sorted(((t, k) for k, t in tot.items() if t), reverse=True)[:8]))
lines.append("# hottest SASS lines (samples, top two stall reasons)")
for r in sorted(data, key=lambda r: -f(r, "Warp Stall Sampling (All Samples)"))[:16]:
    st = sorted(((f(r, k), k) for k in stalls), reverse=True)[:2]
    lines.append(f"{r[1].strip()[:64]:64s} {int(f(r, 'Warp Stall Sampling (All Samples)')):8d}  " +
                 ", ".join(f"{k[6:]} {int(a)}" for a, k in st))
open(out_txt, "w").write("\n".join(lines) + "\n")
print("\n".join(lines[:30]))
