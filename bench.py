#!/usr/bin/env python
"""bench.py -- the BASELINE.json headline on B200: fused symmetric SpMM
H.X + H^T.X GB/s (% of the measured HBM roofline) on config 2 (n = 2e6,
256-row tiles, fp32 H, fp64 X/Y, m = 16), plus the LOBPCG time-to-solution of
config 1 as a side record.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One step = one fused SpMM over the whole matrix with X resident in HBM
(value); e2e = the same SpMM through the C-ABI host call cieg_spmm_host with
pinned host X/U, H2D + kernel + D2H inside the timed region. H (6.4 GB) and
X/U (256 MB each) exceed the 126 MB L2, so no flush is needed between steps.
--impl reference times the UNMODIFIED reference ci::spmm (oracle/_ref,
OpenMP on all host cores) on the same matrix.
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

FP64_PEAK_TFLOPS = 37.0  # measured: tools/microbench/fp64_probe.cu (DFMA and DMMA both 37.0 TF/s)


def _bf16_peak():
    try:
        with open(os.path.join(REPO, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["bf16_tflops"])
    except Exception:
        return 2250.0


BF16_PEAK_TFLOPS = _bf16_peak()


def load_peaks():
    try:
        with open(os.path.join(REPO, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def load_traffic(workload):
    """dram bytes per launch from the committed ncu --set full capture."""
    p = os.path.join(REPO, "profiles", "traffic.json")
    try:
        with open(p) as f:
            e = json.load(f).get(workload)
        return int(e["traffic_per_launch"]) if e else None
    except Exception:
        return None


def roofline(gbs, tflops, hbm_peak, hbm_kind, nbytes, flops, workload, issued_flops=None, ms=None, kernel=None,
             int8_ops=None):
    """the roof is min(HBM, FP64). The bound is whichever
    the algorithmic intensity F/B selects against the ridge
    FP64_peak / HBM_peak (5.7 flop/B): cfg2 at m = 16 (7.4 flop/B) is
    FP64-bound, m <= 8 HBM-bound. Both fractions are reported."""
    ridge = FP64_PEAK_TFLOPS * 1e12 / (hbm_peak * 1e9)
    ai = flops / nbytes
    r = {"traffic": load_traffic(workload), "traffic_source": "profiles/traffic.json: ncu dram__bytes_read.sum + "
         "dram__bytes_write.sum summed over the kernels of one SpMM call (committed capture, not this run)",
         "bytes_per_launch": nbytes, "flops_per_launch": flops,
         "flop_per_byte": round(ai, 3), "ridge_flop_per_byte": round(ridge, 3),
         "hbm_achieved_gbs": round(gbs, 2), "hbm_peak_gbs": hbm_peak, "hbm_peak_kind": hbm_kind,
         "hbm_frac": round(gbs / hbm_peak, 4), "hbm_frac_nominal": round(gbs / 8000.0, 4),
         "fp64_achieved_tflops": round(tflops, 3), "fp64_peak_tflops": FP64_PEAK_TFLOPS,
         "fp64_peak_kind": "measured (tools/microbench/fp64_probe.cu: DFMA = DMMA m8n8k4 = 37.0 TF/s)",
         "fp64_frac": round(tflops / FP64_PEAK_TFLOPS, 4)}
    if issued_flops and ms:
        # what the FP64 tensor pipe actually executes: every work item is a
        # dense TD x TD tile times TD x 8 ceil(m / 8) slab (DMMA), zeros included
        it = issued_flops / (ms * 1e-3) / 1e12
        r.update({"fp64_issued_flops_per_launch": int(issued_flops), "fp64_issued_tflops": round(it, 3),
                  "fp64_issued_frac": round(it / FP64_PEAK_TFLOPS, 4)})
    if kernel == "sliced":
        # the int8 tensor-core K1: no FP64 pipe in the product; the bound is
        # HBM (its int8 tensor work is reported beside it)
        r.update({"bound": "hbm", "achieved": r["hbm_achieved_gbs"], "peak": hbm_peak, "unit": "GB/s",
                  "frac": r["hbm_frac"], "peak_kind": hbm_kind, "kernel": "sliced (int8 tcgen05, Ozaki slices)"})
        if int8_ops and ms:
            t = int8_ops / (ms * 1e-3) / 1e12
            r.update({"int8_tensor_ops_per_launch": int(int8_ops), "int8_tensor_tops": round(t, 1),
                      "int8_tensor_peak_tops": round(2 * BF16_PEAK_TFLOPS, 1),
                      "int8_tensor_peak_kind": "2x MEASURED_PEAKS bf16 (dense int8 = 2x bf16 rate)",
                      "int8_tensor_frac": round(t / (2 * BF16_PEAK_TFLOPS), 4)})
        return r
    if ai >= ridge:
        r.update({"bound": "tensor", "achieved": r["fp64_achieved_tflops"], "peak": FP64_PEAK_TFLOPS,
                  "unit": "TFLOP/s", "frac": r["fp64_frac"], "peak_kind": r["fp64_peak_kind"]})
    else:
        r.update({"bound": "hbm", "achieved": r["hbm_achieved_gbs"], "peak": hbm_peak, "unit": "GB/s",
                  "frac": r["hbm_frac"], "peak_kind": hbm_kind})
    return r


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.path = None

    def __enter__(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        time.sleep(0.25)
        return self

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        rows = []
        try:
            with open(self.path) as f:
                for line in f:
                    parts = [x.strip() for x in line.split(",")]
                    if len(parts) >= 7 and parts[0].replace(".", "").isdigit():
                        rows.append(parts)
        except Exception:
            pass
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [float(r[0]) for r in rows]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[3 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": float(rows[0][1]), "reasons": reasons,
                "samples": len(rows)}


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def gen_matrix(cfg, rank):
    t = time.time()
    h = cfg.generate(seed=cfg.seed + rank)
    return h, time.time() - t


# BASELINE config 2 (the headline workload). Raw parameters here so the
# reference arm can build it without importing the product package;
# ours() asserts that configs.CFG2 agrees.
CFG2_RAW = {"name": "cfg2-spmm", "n": 2_000_000, "sectors": 20, "tile": 256, "q": 0.4, "target_nnz": 0.8e9,
            "seed": 1, "m": 16, "precision": 0, "beta": 2000}


def spmm_config(world, p, nnz):
    """The config dict both arms print, byte for byte."""
    c = CFG2_RAW
    return {"workload": c["name"], "n": c["n"], "sectors": c["sectors"], "tile": c["tile"],
            "p_calibrated": float(f"{p:.10g}"), "q": c["q"], "seed": c["seed"], "nnz_stored": int(nnz),
            "m": c["m"], "h_values": "fp32", "x_y": "fp64",
            "l2": "inputs larger than L2 (H 6.4 GB, X/U 256 MB each); no flush",
            "parallelism": "single GPU" if world == 1 else f"row-block shards x{world} (X halo exchange)"}


def reference_arm(args):
    """--impl reference: the reference's own ci::spmm (oracle/_ref, the
    UNMODIFIED proj/src compiled here) on the host cores. The matrix is built
    by the oracle's generator (oracle/ref_gen.cpp) straight into the
    reference's ci::CsbMatrix -- the product library is never loaded."""
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    from oracle import ci_oracle, ref

    c = CFG2_RAW
    m = c["m"]
    p = ref.calibrated_p(c["n"], c["sectors"], c["tile"], c["q"], c["target_nnz"])
    gen = lambda nbk: ref.generate(c["n"], c["sectors"], c["tile"], p, c["q"], c["seed"], c["precision"],
                                   c["beta"], nbk=nbk)
    # every host core the process may use (torchrun exports OMP_NUM_THREADS=1)
    ref.set_threads(len(os.sched_getaffinity(0)))
    cores = ref.max_threads()
    nnz_full = ref.count_nnz(c["n"], c["sectors"], c["tile"], p, c["q"], c["seed"])
    # Bounded sample: the leading principal submatrix (whole CSB block rows)
    # sized so that warmup + steps stay within ~90 s of CPU time.
    probe = gen(1)
    nb = probe.nb_total
    probe = gen(max(1, nb // 16))
    xp = ci_oracle.random_block(probe.dim, m, 5)
    secs, _ = ref.spmm_timed(probe, xp, 2)
    rate = probe.nnz / max(secs[1], 1e-9)
    budget = 90.0 / max(1, args.steps + args.warmup)
    frac_nnz = min(1.0, budget * rate / nnz_full)
    nbk = max(1, min(nb, int(round(nb * frac_nnz))))
    del probe
    rm = gen(nbk)
    x = ci_oracle.random_block(rm.dim, m, 5)
    secs, _ = ref.spmm_timed(rm, x, args.warmup + args.steps)
    t = float(np.mean(secs[args.warmup:]))
    v = 4 if c["precision"] == 0 else 8
    nbytes = rm.nnz * (v + 4) + 2 * rm.dim * m * 8
    gbs = nbytes / t / 1e9
    desc = (f"ci::spmm (reference, OpenMP {cores} threads, timed inside the library) on the leading {rm.dim} rows "
            f"({rm.nnz} stored nnz, {100.0 * rm.nnz / nnz_full:.1f}% of config 2), m={m}")
    line = {
        "metric": "spmm_gbs", "value": round(gbs, 3), "unit": "GB/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(t * 1e3, 3), "higher_is_better": True,
        "scaling": "strong" if world > 1 else "weak",
        "vs_baseline": None, "dtype": "f64 (fp32 H promoted)", "data": "synthetic (seeded sector generator, BASELINE config 2)",
        "config": spmm_config(world, p, nnz_full),
        "impl": "reference",
        "cpu_baseline": {"value": round(gbs, 3), "unit": "GB/s", "cores": cores, "kind": "reference",
                         "sample": desc},
        "e2e": {"value": round(gbs, 3), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def _leading_block(h, nbk):
    """Leading principal submatrix made of the first nbk CSB block rows."""
    from paper_1609_01689_b200 import ci

    nblk = nbk * (nbk + 1) // 2
    e = int(h.entry_offsets[nblk])
    dim = int(h.block_boundaries[nbk])
    groups = None
    if h.groups is not None:
        groups = h.groups[h.groups <= dim]
        if groups[-1] != dim:
            groups = np.append(groups, np.uint32(dim))
    return ci.CsbMatrix(dim=dim, precision=h.precision, block_boundaries=h.block_boundaries[:nbk + 1].copy(),
                        entry_offsets=h.entry_offsets[:nblk + 1].copy(), rows=h.rows[:e], cols=h.cols[:e],
                        values=h.values[:e], groups=groups, beta=h.beta)


def cpu_baseline(h, m, x, y_gpu):
    """cpu_baseline record: the reference ci::spmm (oracle/_ref) on the FULL
    config-2 matrix, timed inside the library (3 calls), and the parity check
    of the GPU result against it (max relative difference)."""
    from oracle import ref

    if not ref.available():
        return None, None
    ref.set_threads(len(os.sched_getaffinity(0)))
    cores = ref.max_threads()
    rm = ref.RefMatrix(h)
    secs, y_ref = ref.spmm_timed(rm, x, 3)
    t = float(np.mean(secs[1:]))
    v = 4 if h.precision == 0 else 8
    gbs = (h.nnz_lower * (v + 4) + 2 * h.dim * m * 8) / t / 1e9
    scale = np.abs(y_ref).max(axis=0)
    max_rel = float((np.abs(y_gpu - y_ref).max(axis=0) / scale).max())
    rec = {"value": round(gbs, 3), "unit": "GB/s", "cores": cores, "kind": "reference",
           "sample": f"ci::spmm (oracle/_ref) on the full config-2 matrix ({h.dim} rows, {h.nnz_lower} nnz), m={m}, "
                     f"mean of calls 2-3 timed inside the library"}
    parity = {"max_rel": max_rel, "norm": "per column, relative to max |U_ref|",
              "vs": "ci::spmm (unmodified reference, oracle/_ref) on the full config-2 matrix, same X",
              "tolerance": 1e-13}
    return rec, parity


def lobpcg_record():
    """Config-1 LOBPCG time-to-solution (GPU) with the reference's iteration count."""
    from paper_1609_01689_b200 import ci, configs

    cfg = configs.CFG1
    h = cfg.generate()
    td = ci.extract_tile_diagonal(h)
    x0 = ci.random_block(h.dim, cfg.kt, 42)
    opt = ci.LobpcgOptions(k_want=cfg.k_want, tol=cfg.tol, preconditioner=td)
    ci.lobpcg_solve(h, x0, opt)  # warm
    times = []
    for _ in range(3):  # median of three solves (host-side timing)
        t0 = time.perf_counter()
        rep = ci.lobpcg_solve(h, x0, opt)
        times.append((time.perf_counter() - t0) * 1e3)
    ms = statistics.median(times)
    out = {"workload": cfg.name, "iterations": rep.iterations, "converged": rep.converged, "ms": round(ms, 2),
           "split_ms": {k: round(v, 2) for k, v in rep.timing_ms.items()},
           "eigenvalues": [float(v) for v in rep.eigenvalues]}
    try:
        from oracle import ref

        if ref.available():
            rm = ref.RefMatrix(h)
            rtd = ref.RefTileDiagonal(rm, h.groups)
            t0 = time.perf_counter()
            rr = ref.lobpcg_solve(rm, x0, cfg.k_want, cfg.tol, 500, rtd)
            out["reference"] = {"iterations": rr.iterations, "ms": round((time.perf_counter() - t0) * 1e3, 2),
                                "cores": ref.max_threads()}
            out["max_rel_eig_diff"] = float(np.max(np.abs(rep.eigenvalues - rr.eigenvalues) / np.abs(rr.eigenvalues)))
    except Exception as e:  # the record is informative only
        out["reference_error"] = str(e)
    return out


def lanczos_record():
    """Config-1 Lanczos baseline (lanczos.cpp:24-136) on the GPU vs the
    reference's CPU Lanczos, same start (ones on the first sector, the
    generator's lowest stratum), k_want 4, tol 1e-8."""
    from paper_1609_01689_b200 import ci, configs

    cfg = configs.CFG1
    h = cfg.generate()
    v0 = ci.lanczos_default_start(h.dim, h.dim // cfg.sectors)
    opt = ci.LanczosOptions(k_want=cfg.k_want, tol=cfg.tol, max_iter=500)
    ci.lanczos_solve(h, v0, opt)  # warm
    times = []
    for _ in range(3):  # median of three solves
        t0 = time.perf_counter()
        rep = ci.lanczos_solve(h, v0, opt)
        times.append((time.perf_counter() - t0) * 1e3)
    ms = statistics.median(times)
    out = {"workload": cfg.name + " (Lanczos)", "iterations": rep.iterations, "converged": rep.converged,
           "ms": round(ms, 2), "split_ms": {k: round(v, 2) for k, v in rep.timing_ms.items()},
           "eigenvalues": [float(v) for v in rep.eigenvalues]}
    try:
        from oracle import ref

        if ref.available():
            rm = ref.RefMatrix(h)
            t0 = time.perf_counter()
            rr = ref.lanczos_solve(rm, v0, cfg.k_want, cfg.tol, 500)
            out["reference"] = {"iterations": rr.iterations, "ms": round((time.perf_counter() - t0) * 1e3, 2),
                                "cores": ref.max_threads()}
            out["max_rel_eig_diff"] = float(np.max(np.abs(rep.eigenvalues - rr.eigenvalues) / np.abs(rr.eigenvalues)))
    except Exception as e:  # the record is informative only
        out["reference_error"] = str(e)
    return out


def sweep_record(dev):
    """BASELINE config 3: the config-1 matrix (fp64, L2-resident) at m = 1..64:
    device time per SpMM (CUDA events, 20 back-to-back calls after warm-up),
    algorithmic GB/s and flop/byte per m. The problem is L2-resident and
    launch-bound, so the same 20 calls are also captured in a CUDA graph and
    replayed (`graph_us`, launch overhead removed); both are labelled."""
    import torch

    from paper_1609_01689_b200 import _lib as L
    from paper_1609_01689_b200 import ci, configs

    cfg = configs.CFG1
    dm = cfg.generate_device(device=dev)
    tdev = torch.device("cuda", dev.index)
    lib = L.load()
    stream = torch.cuda.Stream(device=tdev)
    ci._check(lib.cieg_ctx_set_stream(dev.handle, ctypes.c_void_p(stream.cuda_stream)))
    out = []
    try:
        for m in configs.SWEEP_M:
            x = torch.from_numpy(ci.random_block(cfg.n, m, m)).to(tdev)
            y = torch.empty_like(x)
            torch.cuda.synchronize()
            with torch.cuda.stream(stream):
                for _ in range(3):
                    dm.spmm_ptr(x.data_ptr(), y.data_ptr(), m)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                for _ in range(20):
                    dm.spmm_ptr(x.data_ptr(), y.data_ptr(), m)
                e1.record(stream)
            e1.synchronize()
            us = e0.elapsed_time(e1) / 20 * 1e3
            graph_us = None
            try:
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=stream):
                    for _ in range(20):
                        dm.spmm_ptr(x.data_ptr(), y.data_ptr(), m)
                g.replay()
                torch.cuda.synchronize()
                e2, e3 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                with torch.cuda.stream(stream):
                    e2.record(stream)
                    g.replay()
                    e3.record(stream)
                e3.synchronize()
                graph_us = round(e2.elapsed_time(e3) / 20 * 1e3, 2)
            except Exception:  # capture unsupported here: report the plain number only
                graph_us = None
            b = configs.spmm_bytes(dm.nnz, cfg.n, m, 1)
            f = configs.spmm_flops(dm.nnz, cfg.n, m)
            out.append({"m": m, "us": round(us, 2), "graph_us": graph_us,
                        "gbs": round(b / (us * 1e-6) / 1e9, 1),
                        "graph_gbs": round(b / (graph_us * 1e-6) / 1e9, 1) if graph_us else None,
                        "flop_per_byte": round(f / b, 3), "gflops": round(f / (us * 1e-6) / 1e9, 1)})
    finally:
        ci._check(lib.cieg_ctx_set_stream(dev.handle, None))
    return {"workload": "cfg3-sweep (config-1 matrix, fp64 H, L2-resident; us = back-to-back launches, "
                        "graph_us = CUDA-graph replay)", "points": out}


def cfg4_record(dev):
    """BASELINE config 4 time-to-solution on one GPU (matrix generated on the
    GPU; preconditioned, k_want 8, block 16, tol 1e-6)."""
    import numpy as np

    from paper_1609_01689_b200 import ci, configs

    cfg = configs.CFG4
    t0 = time.time()
    dm = cfg.generate_device(device=dev)
    td = ci.tile_diagonal_from_matrix(dm)
    dm.prepare(cfg.kt)  # the sliced kernel's slice planes (one-time matrix setup, outside the solve)
    dev.synchronize()
    gen_s = time.time() - t0
    x0 = ci.random_block(cfg.n, cfg.kt, 42)
    t0 = time.perf_counter()
    rep = ci.lobpcg_solve(dm, x0, ci.LobpcgOptions(k_want=cfg.k_want, tol=cfg.tol, preconditioner=td))
    tts = time.perf_counter() - t0
    rr = np.array([r.relres for r in rep.history]).reshape(-1, cfg.kt)
    out = {"workload": cfg.name, "n": cfg.n, "nnz_stored": dm.nnz, "tts_s": round(tts, 3),
           "iterations": rep.iterations, "converged": rep.converged, "gen_on_gpu_s": round(gen_s, 2),
           "split_ms": {k: round(v, 1) for k, v in rep.timing_ms.items()}, "counters": vars(rep.counters),
           "max_final_relres": float(rr[-1, :cfg.k_want].max()), "eigenvalues": rep.eigenvalues.tolist()}
    # the paper's comparison: the Lanczos baseline on the same matrix
    # (ones on the first sector, k_want 8, tol 1e-6, <= 500 steps)
    del td
    t0 = time.perf_counter()
    la = ci.lanczos_solve(dm, ci.lanczos_default_start(cfg.n, cfg.n // cfg.sectors),
                          ci.LanczosOptions(k_want=cfg.k_want, tol=cfg.tol, max_iter=500))
    out["lanczos"] = {"tts_s": round(time.perf_counter() - t0, 3), "iterations": la.iterations,
                      "converged": la.converged, "split_ms": {k: round(v, 1) for k, v in la.timing_ms.items()},
                      "spmv_equivalents": la.counters.spmv_equivalents,
                      "max_rel_eig_diff_vs_lobpcg": float(np.max(np.abs(la.eigenvalues - rep.eigenvalues) /
                                                                 np.abs(rep.eigenvalues)))}
    return out


def cfg5_record(dev, rank, world):
    """BASELINE config 5 (n = 4e7, S = 2e10, k_want 8, block 16, tol 1e-6)
    sharded over the ranks: every rank generates its row block on its GPU
    (DeviceShard) and its local tile-diagonal preconditioner; X halos move
    point to point before each SpMM, Grams are all-reduced. Collective: all
    ranks call it. Times are max over ranks."""
    import torch
    import torch.distributed as dist

    from paper_1609_01689_b200 import ci, configs
    from paper_1609_01689_b200 import dist as D

    cfg = configs.CFG5
    scale = float(os.environ.get("CIEG_CFG5_SCALE", "1"))  # < 1 only to exercise the path on one GPU
    if scale != 1.0:
        import dataclasses

        n = int(cfg.n * scale) // cfg.sectors * cfg.sectors
        cfg = dataclasses.replace(cfg, name=f"{cfg.name} (scaled x{scale}, functional check)", n=n,
                                  target_nnz=cfg.target_nnz * scale)
    tdev = torch.device("cuda", dev.index)
    out = {"workload": cfg.name, "n": cfg.n, "gpus": world, "k_want": cfg.k_want, "block": cfg.kt, "tol": cfg.tol}
    try:
        # per-rank footprint: tile stream (8 B/entry, boundary tiles duplicated),
        # dense fp64 256 x 256 diagonal blocks, ~15 local n x 16 blocks
        local = cfg.n / world
        free, _ = torch.cuda.mem_get_info(tdev)
        tiles = cfg.expected_nnz() / world * 8 * 1.06
        blocks = local * 256 * 8
        if blocks > (free - tiles) / 4:  # the library then stores the diagonal blocks in fp32 (exact)
            blocks /= 2
        est = tiles + blocks + 15 * local * cfg.kt * 8
        ok = torch.tensor([1 if est < 0.92 * free else 0], device=tdev)
        dist.all_reduce(ok, op=dist.ReduceOp.MIN)
        if not int(ok.item()):
            out["skipped"] = f"needs ~{est / 1e9:.0f} GB per GPU, {free / 1e9:.0f} GB free"
            return out
        dist.barrier()
        t0 = time.time()
        rb = D.generated_row_bounds(cfg, world)
        sh = D.DeviceShard.generate(cfg, rb, dev)
        td = ci.tile_diagonal_from_matrix(sh.dm)
        dev.synchronize()
        dist.barrier()
        gen_s = time.time() - t0
        x0 = ci.random_block_rows(sh.row_lo, sh.row_hi, cfg.kt, 42)
        dist.barrier()
        t0 = time.perf_counter()
        rep = D.lobpcg_solve_dist(sh, x0, ci.LobpcgOptions(k_want=cfg.k_want, tol=cfg.tol), td)
        dist.barrier()
        tts = time.perf_counter() - t0
        del td
        # standalone sharded SpMMs at m = 16: K1 alone vs K1 + halo exchange
        m = 16
        xl = torch.from_numpy(ci.random_block_rows(sh.row_lo, sh.row_hi, m, 7)).to(tdev)
        hl, hh = sh.halo
        buf = torch.empty((hh - hl, m), dtype=torch.float64, device=tdev)
        y = torch.empty((sh.local_rows, m), dtype=torch.float64, device=tdev)
        stream = torch.cuda.Stream(device=tdev)
        torch.cuda.set_stream(stream)
        from paper_1609_01689_b200 import _lib as L

        lib = L.load()
        ci._check(lib.cieg_ctx_set_stream(dev.handle, ctypes.c_void_p(stream.cuda_stream)))
        xfull_ptr = buf.data_ptr() - 8 * hl * m

        def k1():
            sh.dm.spmm_ptr(xfull_ptr, y.data_ptr(), m)

        def step():
            D.halo_exchange(xl, sh.plan, buf, out_row0=hl)
            k1()

        def timed(fn, k=5):
            for _ in range(2):
                fn()
            torch.cuda.synchronize()
            dist.barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(k):
                fn()
            e1.record(stream)
            e1.synchronize()
            t = torch.tensor([e0.elapsed_time(e1) / k], device=tdev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            return float(t.item())

        ms_step, ms_k1 = timed(step), timed(k1)
        ci._check(lib.cieg_ctx_set_stream(dev.handle, None))
        torch.cuda.set_stream(torch.cuda.default_stream(tdev))
        nnz_t = torch.tensor([float(sh.dm.nnz)], device=tdev, dtype=torch.float64)
        dist.all_reduce(nnz_t)
        nnz_max = torch.tensor([float(sh.dm.nnz)], device=tdev, dtype=torch.float64)
        dist.all_reduce(nnz_max, op=dist.ReduceOp.MAX)
        split = torch.tensor([rep.timing_ms[k] for k in ("spmm", "rayleigh_ritz", "orthonormalization",
                                                          "preconditioner", "residual", "other", "total")],
                             device=tdev, dtype=torch.float64)
        dist.all_reduce(split, op=dist.ReduceOp.MAX)
        per_gpu_bytes = configs.spmm_bytes(int(nnz_max.item()), sh.local_rows, m, 0)
        peak, _ = load_peaks()
        per_gpu_gbs = per_gpu_bytes / (ms_k1 * 1e-3) / 1e9
        out.update({"tts_s": round(tts, 3), "iterations": rep.iterations, "converged": rep.converged,
                    "gen_on_gpu_s": round(gen_s, 2), "nnz_stored_total": int(nnz_t.item()),
                    "split_ms_max_over_ranks": dict(zip(("spmm", "rayleigh_ritz", "orthonormalization",
                                                         "preconditioner", "residual", "other", "total"),
                                                        [round(v, 1) for v in split.tolist()])),
                    "counters": vars(rep.counters), "eigenvalues": rep.eigenvalues.tolist(),
                    "spmm_m16": {"ms_k1": round(ms_k1, 3), "ms_with_halo_exchange": round(ms_step, 3),
                                 "comm_fraction": round(1 - ms_k1 / ms_step, 3),
                                 "per_gpu_gbs": round(per_gpu_gbs, 1),
                                 "per_gpu_hbm_frac": round(per_gpu_gbs / peak, 4),
                                 "halo_rows": hh - hl, "rows_per_gpu": sh.local_rows}})
    except Exception as e:  # reported in the line; the headline stands
        out["error"] = repr(e)[:400]
    return out


def widths_record(dev, dm, stream, n):
    """K1 on the config-2 matrix at the LOBPCG / Lanczos block widths, in the
    default mode and in each explicit kernel (owner-computes, DMMA single
    pass, sliced int8 tensor-core), device time per launch (median of 3 x 10
    launches)."""
    import torch

    from paper_1609_01689_b200 import configs

    out = []
    for m in (1, 4, 8, 16):
        x = torch.randn(n, m, dtype=torch.float64, device="cuda")
        y = torch.empty_like(x)
        row = {"m": m}
        for mode in ("auto", "owner", "single", "sliced"):
            dev.set_spmm_mode(mode)
            for _ in range(3):
                dm.spmm_ptr(x.data_ptr(), y.data_ptr(), m)
            times = []
            for _ in range(3):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                for _ in range(10):
                    dm.spmm_ptr(x.data_ptr(), y.data_ptr(), m)
                e1.record(stream)
                e1.synchronize()
                times.append(e0.elapsed_time(e1) / 10)
            t = sorted(times)[1]
            row[mode] = {"ms": round(t, 4),
                         "gbs": round(configs.spmm_bytes(dm.nnz, n, m, dm.precision) / (t * 1e-3) / 1e9, 1)}
        dev.set_spmm_mode("auto")
        row["auto_mode"] = dm.spmm_kernel(m)
        out.append(row)
        del x, y
    dev.set_spmm_mode("auto")
    return {"workload": "cfg2-spmm K1 by block width", "points": out}


def shard_modes_record(dev, dm, plan, row_bounds, rank, n, tdev, stream, m=8):
    """N > 1, config 2 at m = 8 on the same shards: owner-computes K1 after
    the X halo exchange vs the single pass, whose transposed partials for
    lower ranks' rows go back point to point (SURVEY.md 8(e) reduce-scatter)
    -- per step, max over ranks."""
    import torch
    import torch.distributed as dist

    from paper_1609_01689_b200 import ci, configs
    from paper_1609_01689_b200 import dist as D

    try:
        lo, hi = int(row_bounds[rank]), int(row_bounds[rank + 1])
        x_full = torch.from_numpy(ci.random_block(n, m, 8)).to(tdev)
        x_local = x_full[lo:hi].clone()
        y = torch.empty((hi - lo, m), dtype=torch.float64, device=tdev)
        pplan = D.PartialPlan(row_bounds, D.gather_partial_lo(D.partial_rows(dm.handle)[0], tdev), rank)

        def owner():
            D.halo_exchange(x_local, plan, x_full)
            dm.spmm_ptr(x_full.data_ptr(), y.data_ptr(), m)

        def single():
            D.halo_exchange(x_local, plan, x_full)
            D.spmm_single_pass(dm.handle, dev, x_full, y, pplan)

        def timed(fn, k=5):
            for _ in range(2):
                fn()
            torch.cuda.synchronize()
            dist.barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(k):
                fn()
            e1.record(stream)
            e1.synchronize()
            t = torch.tensor([e0.elapsed_time(e1) / k], device=tdev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            return float(t.item())

        ms_o, ms_s = timed(owner), timed(single)
        nnz = int(configs.CFG2.expected_nnz())
        nb = configs.spmm_bytes(nnz, n, m, 0)
        return {"m": m, "owner_ms": round(ms_o, 3), "single_pass_ms": round(ms_s, 3),
                "owner_gbs": round(nb / (ms_o * 1e-3) / 1e9, 1), "single_pass_gbs": round(nb / (ms_s * 1e-3) / 1e9, 1),
                "partial_rows_sent": pplan.send_rows(), "partial_rows_received": pplan.recv_rows()}
    except Exception as e:  # reported in the line; the headline stands
        return {"error": repr(e)[:400]}


def group_bounds(cfg):
    """Generator tile (= group) starts, the rule of generator.cpp make_grid."""
    out = []
    for s in range(cfg.sectors):
        a, b = cfg.n * s // cfg.sectors, cfg.n * (s + 1) // cfg.sectors
        out.extend(range(a, b, cfg.tile))
    return out + [cfg.n]


def ours(args):
    import torch

    from paper_1609_01689_b200 import ci, configs

    rank, world, local = dist_env()
    local = local % max(1, torch.cuda.device_count())
    if world > 1:
        import torch.distributed as dist

        # CIEG_DIST_BACKEND=gloo runs the N > 1 choreography with host-mediated
        # collectives (used to exercise several ranks on a single GPU)
        if os.environ.get("CIEG_DIST_BACKEND") == "gloo":
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    cfg = configs.CFG2
    raw = CFG2_RAW
    assert (cfg.name, cfg.n, cfg.sectors, cfg.tile, cfg.q, cfg.target_nnz, cfg.seed, cfg.m, cfg.precision,
            cfg.beta) == (raw["name"], raw["n"], raw["sectors"], raw["tile"], raw["q"], raw["target_nnz"],
                          raw["seed"], raw["m"], raw["precision"], raw["beta"]), "CFG2_RAW out of date"
    m = args.m or cfg.m
    dev = ci.Device(local)
    tdev = torch.device("cuda", local)
    h = None
    t0 = time.time()
    if world == 1:
        # the drop-in path: host CsbMatrix (also used by the CPU baseline) -> upload
        h, t_gen = gen_matrix(cfg, 0)
        t0 = time.time()
        dm = ci.DeviceMatrix(h, dev)
        row_bounds = [0, cfg.n]
    else:
        # row-block shards generated on each GPU (strong scaling of the same matrix)
        from paper_1609_01689_b200 import dist as D

        # panel-aligned cuts balanced by streamed entries (the documented sharding)
        row_bounds = [int(v) for v in D.generated_row_bounds(cfg, world)]
        t_gen = 0.0
        dm = cfg.generate_device(device=dev, rows=(row_bounds[rank], row_bounds[rank + 1]))
    t_up = time.time() - t0
    n = cfg.n
    lo, hi = row_bounds[rank], row_bounds[rank + 1]
    # one dedicated (non-default) stream carries the collectives and the
    # library's kernels, so both are ordered and the events time both
    stream = torch.cuda.Stream(device=tdev)
    torch.cuda.set_stream(stream)
    from paper_1609_01689_b200 import _lib as L

    lib = L.load()
    ci._check(lib.cieg_ctx_set_stream(dev.handle, ctypes.c_void_p(stream.cuda_stream)))
    x_full = torch.from_numpy(ci.random_block(n, m, 5)).to(tdev)
    x_local = x_full[lo:hi].clone()
    y = torch.empty((hi - lo, m), dtype=torch.float64, device=tdev)
    exchange = None
    if world > 1:
        from paper_1609_01689_b200 import dist as D

        # each rank's kernel reads X only on its halo: point-to-point halo
        # exchange (CIEG_EXCHANGE=allgather for the all-gather variant)
        gl, gh = D.gather_halos(dm.halo_lo, dm.halo_hi, tdev)
        plan = D.ExchangePlan(row_bounds, gl, gh, rank)
        mode = os.environ.get("CIEG_EXCHANGE", "halo")
        recv = plan.recv_rows() if mode == "halo" else n - (hi - lo)
        rt = torch.tensor([recv], dtype=torch.int64, device=tdev)
        dist.all_reduce(rt, op=dist.ReduceOp.MAX)
        exchange = {"kind": "halo point-to-point" if mode == "halo" else "all-gather",
                    "max_recv_rows_per_rank": int(rt.item()),
                    "recv_bytes_per_step_max": int(rt.item()) * m * 8, "rows_per_rank": hi - lo}
    torch.cuda.synchronize()

    def step():
        if world > 1:
            if exchange["kind"] == "all-gather":
                D.allgather_rows(x_local, row_bounds, x_full)
            else:
                D.halo_exchange(x_local, plan, x_full)
        dm.spmm_ptr(x_full.data_ptr(), y.data_ptr(), m)

    def barrier():
        if world > 1:
            import torch.distributed as dist

            dist.barrier()

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    l0 = dev.launches
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        ev0.record(stream)
        for _ in range(args.steps):
            step()
        ev1.record(stream)
        ev1.synchronize()
    torch.cuda.synchronize()
    barrier()
    launches = dev.launches - l0
    ms = ev0.elapsed_time(ev1) / args.steps
    kernel = dm.spmm_kernel(m) if world == 1 else "owner-computes shards"
    if world > 1:
        import torch.distributed as dist

        t = torch.tensor([ms], device=tdev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        nnz_t = torch.tensor([dm.nnz], device=tdev, dtype=torch.float64)
        dist.all_reduce(nnz_t)
    nnz_total = dm.nnz if world == 1 else None
    # algorithmic bytes of the whole distributed SpMM: every stored entry once,
    # X and U once (shards duplicate boundary tiles; those bytes are not counted)
    if world == 1:
        nbytes = configs.spmm_bytes(dm.nnz, n, m, dm.precision)
        flops = configs.spmm_flops(dm.nnz, n, m)
    else:
        nnz_total = ci.count_nnz(cfg.n, cfg.sectors, cfg.tile, cfg.p(), cfg.q, cfg.seed)
        nbytes = configs.spmm_bytes(nnz_total, n, m, 0)
        flops = configs.spmm_flops(nnz_total, n, m)
    gbs = nbytes / (ms * 1e-3) / 1e9
    widths = widths_record(dev, dm, stream, n) if world == 1 else None
    shard_modes = shard_modes_record(dev, dm, plan, row_bounds, rank, n, tdev, stream) if world > 1 else None
    ci._check(lib.cieg_ctx_set_stream(dev.handle, None))
    torch.cuda.set_stream(torch.cuda.default_stream(tdev))

    # e2e (rank 0 drives a full-matrix host call when world == 1; sharded runs
    # report the device-resident number end to end through all ranks)
    e2e = None
    if world == 1:
        # The headline: ci::spmm's own host call (the drop-in binds
        # cieg_spmm_host on the pageable std::vector of ci::BlockVectors):
        # pageable numpy X/U, H2D + K1 + D2H inside each timed call. The
        # pinned-buffer single call and the pipelined pinned batch
        # (cieg_spmm_host_batch, copies of neighbouring steps overlapping K1)
        # are reported beside it.
        pd = ctypes.POINTER(ctypes.c_double)
        own = torch.cuda.ExternalStream(dev.stream, device=tdev)
        ke = max(3, min(args.steps, 20))

        def timed(fn, reps):
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            w0 = time.perf_counter()
            e0.record(own)
            fn()
            e1.record(own)
            e1.synchronize()
            return e0.elapsed_time(e1) / reps, (time.perf_counter() - w0) * 1e3 / reps

        xpg = [ci.random_block(n, m, 6 + b) for b in range(2)]
        ypg = [np.empty_like(xpg[0]) for _ in range(2)]
        xpp = [ctypes.cast(a.ctypes.data, pd) for a in xpg]
        ypp = [ctypes.cast(a.ctypes.data, pd) for a in ypg]

        def pageable():
            for i in range(ke):
                ci._check(lib.cieg_spmm_host(dev.handle, dm.handle, xpp[i % 2], ypp[i % 2], m))

        pageable()  # warm (staging ring, page faults of the fresh numpy buffers)
        ms_e2e, wall_e2e = timed(pageable, ke)
        xhs = [torch.from_numpy(a).pin_memory() for a in xpg]
        yhs = [torch.empty_like(xhs[0]).pin_memory() for _ in range(2)]
        xp = [ctypes.cast(t.data_ptr(), pd) for t in xhs]
        yp = [ctypes.cast(t.data_ptr(), pd) for t in yhs]
        xs = (pd * ke)(*[xp[i % 2] for i in range(ke)])
        ys = (pd * ke)(*[yp[i % 2] for i in range(ke)])

        def batch():
            ci._check(lib.cieg_spmm_host_batch(dev.handle, dm.handle, xs, ys, m, ke))

        def single():
            for i in range(ke):
                ci._check(lib.cieg_spmm_host(dev.handle, dm.handle, xp[i % 2], yp[i % 2], m))

        batch()  # warm (allocates the second device buffers)
        ms_batch, _ = sorted((timed(batch, ke) for _ in range(3)), key=lambda t: t[0])[1]
        ms_single, _ = timed(single, ke)
        gb = lambda t: round(nbytes / (t * 1e-3) / 1e9, 3)
        e2e = {"value": gb(ms_e2e), "unit": "GB/s", "h2d_bytes_per_step": n * m * 8, "d2h_bytes_per_step": n * m * 8,
               "ms_per_step": round(ms_e2e, 4), "wall_ms_per_step": round(wall_e2e, 4), "steps": ke,
               "call": "cieg_spmm_host per step on pageable host X/U (ci::spmm's call in the drop-in; inside the "
                       "library the upload, the sliced kernels and the download are pipelined over row chunks "
                       "through pinned staging rings)",
               "pinned": {"value": gb(ms_single), "ms_per_step": round(ms_single, 4),
                          "call": "cieg_spmm_host per step, pinned host X/U (the same chunk pipeline, no staging copies)"},
               "pinned_batch": {"value": gb(ms_batch), "ms_per_step": round(ms_batch, 4),
                                "call": "cieg_spmm_host_batch (pinned; copies of neighbouring steps overlap K1)"}}
    else:
        # every rank: its rows of X from pinned host memory, the halo exchange
        # and K1, its rows of U back to pinned host memory (max over ranks)
        import torch.distributed as dist

        xh = torch.from_numpy(ci.random_block_rows(lo, hi, m, 9)).pin_memory()
        yh = torch.empty((hi - lo, m), dtype=torch.float64).pin_memory()
        torch.cuda.set_stream(stream)
        ci._check(lib.cieg_ctx_set_stream(dev.handle, ctypes.c_void_p(stream.cuda_stream)))

        def e2e_step():
            x_local.copy_(xh, non_blocking=True)
            step()
            yh.copy_(y, non_blocking=True)

        for _ in range(2):
            e2e_step()
        torch.cuda.synchronize()
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            e2e_step()
        e1.record(stream)
        e1.synchronize()
        te = torch.tensor([e0.elapsed_time(e1) / args.steps], device=tdev)
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
        ms_e2e = float(te.item())
        ci._check(lib.cieg_ctx_set_stream(dev.handle, None))
        torch.cuda.set_stream(torch.cuda.default_stream(tdev))
        e2e = {"value": round(nbytes / (ms_e2e * 1e-3) / 1e9, 3), "unit": "GB/s",
               "h2d_bytes_per_step": n * m * 8, "d2h_bytes_per_step": n * m * 8, "ms_per_step": round(ms_e2e, 4),
               "call": "per rank: pinned host rows of X -> device, halo exchange + K1, rows of U -> pinned host "
                       "(bytes summed over ranks; time max over ranks)"}
    tile_edge, ntiles, npanels = dm.tile_edge, dm.ntiles, dm.npanels
    if world == 1:  # the timed steps' input and output, for the parity check against the reference
        x_host, y_host = x_full.cpu().numpy(), y.cpu().numpy()
    del dm  # the records below build their own matrices
    torch.cuda.empty_cache()
    cfg5 = None
    if world > 1 and not args.no_cfg5:
        cfg5 = cfg5_record(dev, rank, world)  # collective: every rank
    peak, peak_kind = load_peaks()
    # owner-computes at m = 16: 2 items per off-diagonal tile + 1 per diagonal
    # tile (one per panel), each a dense tile x (TD x 16) slab product
    issued = ((2 * ntiles - npanels) * tile_edge * tile_edge * 8 * ((m + 7) // 8) * 2
              if world == 1 and m > 8 and kernel == "owner-computes" else None)
    # sliced: per stored tile and orientation, sum_s 128 x N_s x 128 int8 MACs,
    # N_s = 16 min(7, 8 - s) over the H slices s = 0..4 (sum 464); diagonal
    # tiles one orientation; 2 ops per MAC
    int8_ops = (2 * 128 * 464 * 128 * (2 * (ntiles - npanels) + npanels)
                if world == 1 and kernel == "sliced" else None)
    if rank != 0:
        if world > 1:
            import torch.distributed as dist

            dist.destroy_process_group()
        return 0
    line = {
        "metric": "spmm_gbs", "value": round(gbs, 3), "unit": "GB/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms, 4), "higher_is_better": True,
        "scaling": "strong" if world > 1 else "weak",
        "vs_baseline": None, "dtype": "f64 (fp32 H promoted exactly)",
        "data": "synthetic (seeded sector generator, BASELINE config 2)",
        "config": spmm_config(world, cfg.p(), nnz_total),
        "setup": {"device_tile_edge": tile_edge, "device_tiles": ntiles, "exchange": exchange,
                  "gen_s": round(t_gen, 1), "upload_s": round(t_up, 1)},
        "roofline": roofline(gbs, flops / (ms * 1e-3) / 1e12, peak, peak_kind, nbytes, flops, cfg.name,
                             issued_flops=issued, ms=ms, kernel=kernel, int8_ops=int8_ops),
        "spmm_kernel": kernel,
        "e2e": e2e,
        "gpu_launches": int(launches),
        "clocks": clk.summary(),
    }
    if widths is not None:
        line["widths"] = widths
    if shard_modes is not None:
        line["shard_modes_m8"] = shard_modes
    if world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"], line["parity"] = cpu_baseline(h, m, x_host, y_host)
    if world == 1 and not args.no_lobpcg:
        line["lobpcg"] = lobpcg_record()
        line["lanczos"] = lanczos_record()
        line["sweep"] = sweep_record(dev)
        if not args.no_cfg4:
            line["lobpcg_cfg4"] = cfg4_record(dev)
    if cfg5 is not None:
        line["lobpcg_cfg5"] = cfg5
    print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--m", type=int, default=0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-lobpcg", action="store_true")
    ap.add_argument("--no-cfg4", action="store_true")
    ap.add_argument("--no-cfg5", action="store_true", help="skip the sharded config-5 LOBPCG record (N > 1)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        return reference_arm(args)
    return ours(args)


if __name__ == "__main__":
    sys.exit(main())
