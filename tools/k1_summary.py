"""Summarise an ncu --set full capture of K1 (spmm_ws_kernel) for profiles/:
key throughput metrics, DRAM traffic vs algorithmic bytes, stall split."""
import csv, io, json, subprocess, sys

rep, out_txt, alg_bytes = sys.argv[1], sys.argv[2], float(sys.argv[3])
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, u, v = rows[0], rows[1], rows[2]
get = lambda k: (v[h.index(k)], u[h.index(k)]) if k in h else ("n/a", "")
keys = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum",
        "smsp__inst_executed.sum", "sm__cycles_active.avg", "launch__grid_size", "launch__block_size",
        "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic"]
lines = [f"# ncu --set full --import-source on --clock-control none -k regex:spmm_ws: {rep.split('/')[-1]}"]
for k in keys:
    val, unit = get(k)
    lines.append(f"{k:62s} {val} {unit}")
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
rd = float(get("dram__bytes_read.sum")[0].replace(",", "")) * scale[get("dram__bytes_read.sum")[1]]
wr = float(get("dram__bytes_write.sum")[0].replace(",", "")) * scale[get("dram__bytes_write.sum")[1]]
lines.append(f"{'dram traffic per launch (read + write)':62s} {rd + wr:.4e} bytes")
lines.append(f"{'algorithmic bytes per launch (DESIGN.md K1)':62s} {alg_bytes:.4e} bytes")
lines.append(f"{'traffic / algorithmic':62s} {(rd + wr) / alg_bytes:.3f}")
stalls = subprocess.run([sys.executable, "tools/ncu_stalls.py", rep, "12"], capture_output=True, text=True).stdout
lines.append("")
lines.append("# warp-stall samples (tools/ncu_stalls.py): producer warps vs consumer warps, top SASS lines")
lines += stalls.rstrip().splitlines()
open(out_txt, "w").write("\n".join(lines) + "\n")
print(json.dumps({"dram_read": rd, "dram_write": wr, "traffic": rd + wr, "algorithmic": alg_bytes}))
