"""N > 1 path on the CPU: world-size-2 gloo processes run the sharding
choreography of paper_1609_01689_b200/dist.py -- the host shard plan
(cieg_shard_plan), the row all-gather and the Gram all-reduce helpers -- with
the numpy oracle standing in for the per-shard device kernels (test
infrastructure), and reproduce the single-process reference results."""
import os
import socket
import sys

import numpy as np
import pytest

from conftest import ROOT, gen_from


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, golden_path, out_q):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch
    import torch.distributed as dist

    from conftest import gen_from as gf
    from oracle import ci_oracle as O
    from paper_1609_01689_b200 import ci
    from paper_1609_01689_b200 import dist as D

    dist.init_process_group("gloo", rank=rank, world_size=world)
    res = {}
    try:
        g = dict(np.load(golden_path))
        h = gf(g["sector_f64_prec_params"])
        rb, hl, hh = D.row_partition(h, world)
        lo, hi = int(rb[rank]), int(rb[rank + 1])
        res["bounds"] = rb.tolist()
        # (1) all-gather of row-distributed X
        x = ci.random_block(h.dim, 5, 9)
        full = torch.zeros((h.dim, 5), dtype=torch.float64)
        D.allgather_rows(torch.from_numpy(x[lo:hi].copy()), rb, full)
        res["allgather_ok"] = bool(np.array_equal(full.numpy(), x))
        # (2) the shard's halo suffices: X rows outside [halo_lo, halo_hi) poisoned
        xp = full.numpy().copy()
        xp[: hl[rank]] = np.nan
        xp[hh[rank]:] = np.nan
        r, c, v, _, _ = O._global_entries(h)
        mine_row = (r >= lo) & (r < hi)
        mine_col = (c >= lo) & (c < hi) & (r != c)
        y = np.zeros((hi - lo, 5))
        np.add.at(y, r[mine_row] - lo, v[mine_row, None] * xp[c[mine_row]])
        np.add.at(y, c[mine_col] - lo, v[mine_col, None] * xp[r[mine_col]])
        res["halo_ok"] = bool(np.isfinite(y).all())
        res["shard_rows_ok"] = bool(np.allclose(y, O.spmm(h, x)[lo:hi], rtol=0, atol=1e-13))
        # (2b) the point-to-point halo exchange fills exactly the halo
        plan = D.ExchangePlan(rb, hl, hh, rank)
        hx = torch.full((h.dim, 5), float("nan"), dtype=torch.float64)
        D.halo_exchange(torch.from_numpy(x[lo:hi].copy()), plan, hx)
        hxn = hx.numpy()
        res["halo_exchange_ok"] = bool(np.array_equal(hxn[hl[rank]:hh[rank]], x[hl[rank]:hh[rank]]))
        res["halo_rows"] = plan.recv_rows()

        # (3) sharded LOBPCG: local rows, all-gathered SpMM input, all-reduced Grams
        def inner(a, b):
            t = torch.from_numpy(np.ascontiguousarray(O.block_inner(a, b)))
            D.allreduce_sum_(t)
            return t.numpy()

        def matvec(vloc):  # halo rows only, as the device path does
            f = torch.zeros((h.dim, vloc.shape[1]), dtype=torch.float64)
            D.halo_exchange(torch.from_numpy(np.ascontiguousarray(vloc)), plan, f)
            return O.spmm(h, f.numpy())[lo:hi]

        k, kt, tol, pre, seed = g["sector_f64_prec_meta"]
        x0 = ci.random_block(h.dim, int(kt), int(seed))[lo:hi]
        tiles_all = O.extract_tile_diagonal(h, h.groups)
        gb = h.groups.astype(np.int64)
        sel = [i for i in range(len(gb) - 1) if gb[i] >= lo and gb[i + 1] <= hi]
        tiles = [tiles_all[i] for i in sel]
        bounds = np.array([gb[sel[0]]] + [gb[i + 1] for i in sel]) - lo
        rep = O.lobpcg_solve(None, x0, int(k), float(tol), 500, tiles, bounds, matvec=matvec, inner=inner)
        res["iterations"] = rep.iterations
        res["eigenvalues"] = rep.eigenvalues.tolist()
        res["counters"] = rep.counters
    except Exception as e:  # pragma: no cover -- surfaced by the parent
        res["error"] = repr(e)
    finally:
        dist.destroy_process_group()
    out_q.put((rank, res))


def test_shard_plan_properties():
    from paper_1609_01689_b200 import configs, dist as D

    h = configs.CFG1.generate()
    for world in (1, 2, 3, 4, 8):
        rb, hl, hh = D.row_partition(h, world)
        assert rb[0] == 0 and rb[-1] == h.dim and np.all(np.diff(rb) > 0)
        assert set(rb.tolist()) <= set(h.groups.astype(np.int64).tolist())  # group aligned
        assert np.all(hl <= rb[:-1]) and np.all(hh >= rb[1:])
        # balanced by streamed entries within 20 % at this size
        from oracle import ci_oracle as O

        r, c, _, _, _ = O._global_entries(h)
        cost = np.bincount(r, minlength=h.dim) + np.bincount(c[r != c], minlength=h.dim)
        per = np.array([cost[rb[k]:rb[k + 1]].sum() for k in range(world)])
        assert per.max() <= 1.2 * per.mean() + cost.max() * 64


def test_gloo_world2_sharded_path(golden):
    import multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    gp = os.path.join(ROOT, "tests", "golden", "lobpcg.npz")
    procs = [ctx.Process(target=_worker, args=(r, 2, port, gp, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=600) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    g = golden("lobpcg")
    for rank in (0, 1):
        res = out[rank]
        assert "error" not in res, res.get("error")
        assert res["allgather_ok"] and res["halo_ok"] and res["shard_rows_ok"] and res["halo_exchange_ok"]
        assert res["iterations"] == int(g["sector_f64_prec_iterations"])
        assert res["counters"] == g["sector_f64_prec_counters"].tolist()
        np.testing.assert_allclose(res["eigenvalues"], g["sector_f64_prec_eigenvalues"], rtol=1e-10)
    assert out[0]["eigenvalues"] == out[1]["eigenvalues"]  # identical decisions on every rank


def _exchange_worker(rank, world, port, out_q):
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch
    import torch.distributed as dist

    from paper_1609_01689_b200 import ci, configs
    from paper_1609_01689_b200 import dist as D

    dist.init_process_group("gloo", rank=rank, world_size=world)
    res = {}
    try:
        h = configs.CFG1.generate()
        rb, hl, hh = D.row_partition(h, world)
        lo, hi = int(rb[rank]), int(rb[rank + 1])
        x = ci.random_block(h.dim, 3, 21)
        plan = D.ExchangePlan(rb, hl, hh, rank)
        gl, gh = D.gather_halos(int(hl[rank]), int(hh[rank]), torch.device("cpu"))
        res["gather_ok"] = gl.tolist() == hl.tolist() and gh.tolist() == hh.tolist()
        out = torch.full((h.dim, 3), float("nan"), dtype=torch.float64)
        D.halo_exchange(torch.from_numpy(x[lo:hi].copy()), plan, out)
        o = out.numpy()
        res["halo_ok"] = bool(np.array_equal(o[hl[rank]:hh[rank]], x[hl[rank]:hh[rank]]))
        res["outside_untouched"] = bool(np.isnan(o[: hl[rank]]).all() and np.isnan(o[hh[rank]:]).all())
        res["recv_rows"] = plan.recv_rows()
        res["send_rows"] = plan.send_rows()
    except Exception as e:  # pragma: no cover
        res["error"] = repr(e)
    finally:
        dist.destroy_process_group()
    out_q.put((rank, res))


@pytest.mark.parametrize("world", [3, 4])
def test_gloo_halo_exchange(world):
    """Point-to-point halo exchange (SURVEY.md 8(e) optimised variant) with
    several peers: every rank ends up with exactly X on its halo rows, rows
    outside the halo are never written, and the sent rows match the received
    ones across ranks."""
    import multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_exchange_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=600) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    for r in range(world):
        assert "error" not in out[r], out[r].get("error")
        assert out[r]["gather_ok"] and out[r]["halo_ok"] and out[r]["outside_untouched"]
    assert sum(out[r]["recv_rows"] for r in range(world)) == sum(out[r]["send_rows"] for r in range(world))


def _partial_worker(rank, world, port, out_q):
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch
    import torch.distributed as dist

    from paper_1609_01689_b200 import dist as D

    dist.init_process_group("gloo", rank=rank, world_size=world)
    res = {}
    try:
        # rows 0..99 in uneven shards; each rank's partial range reaches two shards down
        rb = [0, 17, 40, 71, 100][: world + 1]
        rb[-1] = 100
        plo = [max(0, rb[r] - 30) if r > 0 else 0 for r in range(world)]
        plan = D.PartialPlan(rb, plo, rank)
        gl = D.gather_partial_lo(plo[rank], torch.device("cpu"))
        res["gather_ok"] = gl.tolist() == plo
        lo, hi = rb[rank], rb[rank + 1]

        def f(r, rows, m=3):  # rank r's partial for global rows
            rows = np.asarray(rows, dtype=np.float64)[:, None]
            return r * 1000.0 + rows + 0.25 * np.arange(m)[None, :]

        yhalo = torch.from_numpy(f(rank, range(plo[rank], lo))) if lo > plo[rank] else torch.zeros((1, 3))
        y = torch.from_numpy(np.full((hi - lo, 3), 0.5))
        D.partial_reduce(yhalo, plan, y)
        want = np.full((hi - lo, 3), 0.5)
        for t in range(rank + 1, world):  # ascending peers
            a, b = max(lo, plo[t]), min(hi, rb[t])
            if b > a:
                want[a - lo:b - lo] += f(t, range(a, b))
        res["ok"] = bool(np.array_equal(y.numpy(), want))
        res["sent"] = plan.send_rows()
        res["recv"] = plan.recv_rows()
    except Exception as e:  # pragma: no cover
        import traceback

        res["error"] = repr(e) + traceback.format_exc()
    finally:
        dist.destroy_process_group()
    out_q.put((rank, res))


@pytest.mark.parametrize("world", [3, 4])
def test_gloo_partial_reduce(world):
    """Reverse exchange of the single-pass SpMM (transposed
    partials back to the row owners): every owner ends with its rows plus
    the partials of every higher rank, added in ascending rank order
    (exactly reproducible), and sent rows equal received rows overall."""
    import multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_partial_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=600) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    for r in range(world):
        assert "error" not in out[r], out[r].get("error")
        assert out[r]["gather_ok"] and out[r]["ok"]
    assert sum(out[r]["sent"] for r in range(world)) == sum(out[r]["recv"] for r in range(world))
