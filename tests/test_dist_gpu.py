"""The sharded GPU solver (cieg_lobpcg_solve_dist via dist.py): world 1 over
NCCL, and world 2 as two processes sharing the one available B200 with gloo
collectives (host-mediated: no kernel waits on another rank's kernel). Same
iteration count and eigenvalues as the reference."""
import os
import socket
import sys

import numpy as np
import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, backend, name, out_q):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch
    import torch.distributed as dist

    from conftest import gen_from
    from paper_1609_01689_b200 import ci
    from paper_1609_01689_b200 import dist as D

    torch.cuda.set_device(0)
    if backend == "nccl":
        dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", 0))
    else:
        dist.init_process_group("gloo", rank=rank, world_size=world)
    res = {}
    try:
        g = dict(np.load(os.path.join(ROOT, "tests", "golden", "lobpcg.npz")))
        h = gen_from(g[f"{name}_params"])
        k, kt, tol, pre, seed = g[f"{name}_meta"]
        dev = ci.Device(0)
        sm = D.ShardedMatrix(h, rank, world, dev)
        x0 = ci.random_block(h.dim, int(kt), int(seed))[sm.row_lo:sm.row_hi]
        prec = D.local_tile_diagonal(h, sm.row_lo, sm.row_hi, dev) if pre else None
        # sharded SpMM against the single-GPU kernel
        x = ci.random_block(h.dim, 7, 3)
        y = sm.spmm(torch.from_numpy(x[sm.row_lo:sm.row_hi].copy()).cuda()).cpu().numpy()
        yf = ci.spmm(h, x)[sm.row_lo:sm.row_hi]
        res["spmm_rel"] = float(np.abs(y - yf).max() / np.abs(yf).max())
        ys = sm.spmm(torch.from_numpy(x[sm.row_lo:sm.row_hi].copy()).cuda(), mode="single").cpu().numpy()
        res["spmm_single_rel"] = float(np.abs(ys - yf).max() / np.abs(yf).max())
        rep = D.lobpcg_solve_dist(sm, x0, ci.LobpcgOptions(k_want=int(k), tol=float(tol)), prec)
        res["iterations"] = rep.iterations
        res["eigenvalues"] = rep.eigenvalues.tolist()
        res["counters"] = [rep.counters.spmm_calls, rep.counters.spmv_equivalents,
                           rep.counters.precond_applications, rep.counters.orthogonalizations]
        res["rows"] = rep.trial_vectors.shape[0]
        if backend == "nccl":
            # the same solve with the collectives inside the library (the
            # context's own NCCL communicator, no Python hooks)
            D.nccl_init(dev)
            try:
                rn = D.lobpcg_solve_nccl(sm, x0, ci.LobpcgOptions(k_want=int(k), tol=float(tol)), prec)
            finally:
                D.nccl_finalize(dev)
            res["nccl_iterations"] = rn.iterations
            res["nccl_eigenvalues"] = rn.eigenvalues.tolist()
            res["nccl_counters"] = [rn.counters.spmm_calls, rn.counters.spmv_equivalents,
                                    rn.counters.precond_applications, rn.counters.orthogonalizations]
    except Exception as e:  # pragma: no cover
        import traceback

        res["error"] = repr(e) + traceback.format_exc()
    finally:
        dist.destroy_process_group()
    out_q.put((rank, res))


def _run(world, backend, name):
    import multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, backend, name, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    return out


@pytest.mark.timeout(400)
@pytest.mark.parametrize("world,backend", [(1, "nccl"), (2, "gloo")])
@pytest.mark.parametrize("name", ["sector_f64", "sector_f64_prec"])
def test_sharded_solver_matches_reference(golden, world, backend, name):
    out = _run(world, backend, name)
    g = golden("lobpcg")
    rows = 0
    for rank in range(world):
        res = out[rank]
        assert "error" not in res, res.get("error")
        assert res["spmm_rel"] < 1e-13
        assert res["spmm_single_rel"] < 1e-13
        assert res["iterations"] == int(g[f"{name}_iterations"])
        assert res["counters"] == g[f"{name}_counters"].tolist()
        np.testing.assert_allclose(res["eigenvalues"], g[f"{name}_eigenvalues"], rtol=1e-10)
        if backend == "nccl":  # the in-library NCCL data plane
            assert res["nccl_iterations"] == res["iterations"]
            assert res["nccl_counters"] == res["counters"]
            np.testing.assert_allclose(res["nccl_eigenvalues"], res["eigenvalues"], rtol=1e-13)
        rows += res["rows"]
    assert rows == int(g[f"{name}_params"][0])
    assert all(out[r]["eigenvalues"] == out[0]["eigenvalues"] for r in range(world))


def _gen_worker(rank, world, port, out_q):
    """GPU-generated shards (no host CSB), halo exchange, sharded solve."""
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch
    import torch.distributed as dist

    from paper_1609_01689_b200 import ci, configs
    from paper_1609_01689_b200 import dist as D

    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    res = {}
    try:
        cfg = configs.CFG1
        dev = ci.Device(0)
        rb = D.generated_row_bounds(cfg, world)
        sh = D.DeviceShard.generate(cfg, rb, dev)
        td = ci.tile_diagonal_from_matrix(sh.dm)
        x0 = ci.random_block_rows(sh.row_lo, sh.row_hi, cfg.kt, 42)
        rep = D.lobpcg_solve_dist(sh, x0, ci.LobpcgOptions(k_want=cfg.k_want, tol=cfg.tol), td)
        res["iterations"] = rep.iterations
        res["eigenvalues"] = rep.eigenvalues.tolist()
        res["rows"] = rep.trial_vectors.shape[0]
        res["halo"] = sh.halo
        res["bounds"] = rb.tolist()
    except Exception as e:  # pragma: no cover
        import traceback

        res["error"] = repr(e) + traceback.format_exc()
    finally:
        dist.destroy_process_group()
    out_q.put((rank, res))


@pytest.mark.timeout(400)
def test_generated_shards_solver_matches_single_gpu():
    """The config-5 path at config-1 size: every rank generates its rows on
    the GPU, builds its local preconditioner from them, and the sharded solve
    reproduces the single-GPU solve from the same start."""
    import multiprocessing as mp

    from paper_1609_01689_b200 import ci, configs

    cfg = configs.CFG1
    single = ci.lobpcg_solve(cfg.generate_device(), ci.random_block(cfg.n, cfg.kt, 42),
                             ci.LobpcgOptions(k_want=cfg.k_want, tol=cfg.tol,
                                              preconditioner=ci.tile_diagonal_from_matrix(cfg.generate_device())))
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gen_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    for r in range(2):
        assert "error" not in out[r], out[r].get("error")
        assert out[r]["iterations"] == single.iterations
        np.testing.assert_allclose(out[r]["eigenvalues"], single.eigenvalues, rtol=1e-10)
    assert out[0]["rows"] + out[1]["rows"] == cfg.n
    assert out[0]["eigenvalues"] == out[1]["eigenvalues"]


from conftest import single_pass_shards as _single_pass_shards  # noqa: E402


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("mat", ["f64_t64", "f32_t128"])
@pytest.mark.parametrize("m", [1, 5, 16])
def test_single_pass_shards_match_reference(world, mat, m):
    """each shard reads its stored tiles once; the transposed
    partials for lower shards' rows are reduced at their owners. The
    assembled product equals the reference's spmm."""
    from conftest import gen_from

    from oracle import ci_oracle as O
    from paper_1609_01689_b200 import ci

    params = {"f64_t64": (20_000, 10, 64, 0.05, 0.5, 1, 1, 2000),
              "f32_t128": (30_000, 3, 256, 0.02, 0.4, 77, 0, 2000)}[mat]
    h = gen_from(params)
    x = ci.random_block(h.dim, m, 11 + m)
    y = _single_pass_shards(h, world, m, x)
    want = O.spmm(h, x)
    assert np.abs(y - want).max() / np.abs(want).max() < 1e-13


def test_single_pass_shards_nonfinite():
    """Inf / NaN rows feeding other shards' rows through the partials: the
    receiving owner's fix-up adds those terms (same pattern as the reference)."""
    from conftest import gen_from

    from oracle import ci_oracle as O
    from paper_1609_01689_b200 import ci

    h = gen_from((3072, 3, 256, 0.2, 0.4, 13, 0, 2000))
    x = ci.random_block(h.dim, 4, 5)
    x[2100, 1] = np.inf
    x[1030, 2] = np.nan
    x[2900, 3] = -np.inf
    y = _single_pass_shards(h, 2, 4, x)
    yo = O.spmm(h, x)
    for mask in (np.isnan, np.isposinf, np.isneginf):
        assert np.array_equal(mask(y), mask(yo))
    fin = np.isfinite(yo)
    np.testing.assert_allclose(y[fin], yo[fin], rtol=1e-12, atol=1e-12)


def _small_groups_worker(rank, world, port, out_q):
    """A matrix whose 16-row groups merge into device panels: the shard cuts
    must fall on panel boundaries; the sharded solve matches one GPU."""
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch
    import torch.distributed as dist

    from paper_1609_01689_b200 import ci
    from paper_1609_01689_b200 import dist as D

    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    res = {}
    try:
        h = ci.generate_sector_matrix(1926, 2, 16, 0.3, 0.4, 91, 1, 256, band=1)
        dev = ci.Device(0)
        sm = D.ShardedMatrix(h, rank, world, dev)
        x0 = ci.random_block(h.dim, 6, 5)
        rep = D.lobpcg_solve_dist(sm, x0[sm.row_lo:sm.row_hi], ci.LobpcgOptions(k_want=3, tol=1e-8))
        one = ci.lobpcg_solve(h, x0, ci.LobpcgOptions(k_want=3, tol=1e-8))
        res["iterations"] = (rep.iterations, one.iterations)
        res["eig_rel"] = float(np.abs(rep.eigenvalues - one.eigenvalues).max() / np.abs(one.eigenvalues).max())
        res["bounds"] = [int(b) for b in sm.row_bounds]
    except Exception as e:  # pragma: no cover
        import traceback

        res["error"] = repr(e) + traceback.format_exc()
    finally:
        dist.destroy_process_group()
    out_q.put((rank, res))


@pytest.mark.timeout(400)
def test_sharded_solver_small_groups():
    import multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_small_groups_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    for r in range(2):
        assert "error" not in out[r], out[r].get("error")
        it, it1 = out[r]["iterations"]
        assert it == it1
        assert out[r]["eig_rel"] < 1e-10


def test_spmm_partial_arguments():
    """cieg_spmm_partial: a shard with partial rows needs the partial buffer
    (loud failure without it); on an unsharded matrix it is the single pass
    with no partial rows (cieg_matrix_partial_rows gives an empty range)."""
    import ctypes as C

    import torch

    from conftest import gen_from
    from oracle import ci_oracle as O
    from paper_1609_01689_b200 import _lib, ci
    from paper_1609_01689_b200 import dist as D

    h = gen_from((20_000, 10, 64, 0.05, 0.5, 1, 1, 2000))
    dev = ci.Device.default()
    lib = _lib.load()
    rb, hl, hh = D.row_partition(h, 2)
    sm = D.ShardedMatrix(h, 1, 2, dev, plan=(rb, hl, hh))
    plo, phi = D.partial_rows(sm.handle)
    assert plo < phi == sm.row_lo
    x = torch.from_numpy(ci.random_block(h.dim, 3, 1)).cuda()
    y = torch.empty((sm.local_rows, 3), dtype=torch.float64, device="cuda")
    with pytest.raises(ci.Error):
        ci._check(lib.cieg_spmm_partial(dev.handle, sm.handle, C.c_void_p(x.data_ptr()), C.c_void_p(y.data_ptr()),
                                        3, None))
    dm = ci.DeviceMatrix(h)
    assert D.partial_rows(dm.handle) == (0, 0)
    yf = torch.empty((h.dim, 3), dtype=torch.float64, device="cuda")
    ci._check(lib.cieg_spmm_partial(dev.handle, dm.handle, C.c_void_p(x.data_ptr()), C.c_void_p(yf.data_ptr()), 3,
                                    None))
    dev.synchronize()
    want = O.spmm(h, x.cpu().numpy())
    assert np.abs(yf.cpu().numpy() - want).max() <= 1e-13 * np.abs(want).max()
