"""Row-block sharding of the LOBPCG path over several GPUs,
one process per GPU with torch.distributed for the plumbing.

* Partition: ``row_partition`` (cieg_shard_plan) cuts the rows at group
  boundaries, balanced by the entries each owner streams. Every rank owns its
  rows of H's owner work lists (row parts and the transposed parts of tiles
  (I, P) landing in its rows -- owner-computes needs no reduce-scatter of
  transposed partials; tiles on a shard boundary are held by both owners) and
  its rows of every block vector and tile-diagonal group.
* SpMM: the rank's rows of X are all-gathered (one NCCL broadcast per rank
  into the full-length X; uneven row counts), then the local owner-computes
  kernel writes the rank's rows of U.
* Grams: a local partial over the rank's rows, then an all-reduce; all ranks
  then take identical control-flow decisions (the solver loop is the same
  C++ code as the single-GPU path, driven through cieg_lobpcg_solve_dist's
  collective hooks).

The collective helpers here work on CUDA (NCCL) and CPU (gloo) tensors alike,
so the N > 1 choreography is covered by world-size-2 gloo tests on the CPU.
"""
from __future__ import annotations

import ctypes as C
from typing import Optional

import numpy as np
import torch
import torch.distributed as dist

from . import _lib, ci


def row_partition(h: ci.CsbMatrix, world: int, tile_edge: int = 0):
    """cieg_shard_plan: (row_bounds[world+1], halo_lo[world], halo_hi[world])."""
    lib = _lib.load()
    v = h.view()
    rb = np.zeros(world + 1, np.uint32)
    hl = np.zeros(world, np.uint32)
    hh = np.zeros(world, np.uint32)
    g = None if h.groups is None else np.ascontiguousarray(h.groups, dtype=np.uint32)
    ci._check(lib.cieg_shard_plan(C.byref(v), None if g is None else ci._ptr(g, C.c_uint32),
                                  0 if g is None else len(g) - 1, tile_edge, world, ci._ptr(rb, C.c_uint32),
                                  ci._ptr(hl, C.c_uint32), ci._ptr(hh, C.c_uint32)))
    return rb.astype(np.int64), hl.astype(np.int64), hh.astype(np.int64)


def allgather_rows(x_local: torch.Tensor, row_bounds, out: torch.Tensor, group=None) -> torch.Tensor:
    """out[row_bounds[r]:row_bounds[r+1]] = rank r's x_local, on every rank
    (one broadcast per rank: uneven row counts, no padding copies)."""
    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    lo, hi = int(row_bounds[rank]), int(row_bounds[rank + 1])
    out[lo:hi].copy_(x_local)
    for r in range(world):
        a, b = int(row_bounds[r]), int(row_bounds[r + 1])
        if b > a:
            src = r if group is None else dist.get_global_rank(group, r)
            dist.broadcast(out[a:b], src=src, group=group)
    return out


def allreduce_sum_(t: torch.Tensor, group=None) -> torch.Tensor:
    dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return t


class _CudaView:
    """Zero-copy torch view of a raw device pointer (__cuda_array_interface__)."""

    def __init__(self, ptr: int, shape):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": "<f8", "data": (int(ptr), False),
                                         "version": 3, "strides": None}


def _view(ptr: int, shape, device) -> torch.Tensor:
    return torch.as_tensor(_CudaView(ptr, shape), device=device)


class ShardedMatrix:
    """This rank's part of H resident on its GPU (cieg_matrix_upload_shard)."""

    def __init__(self, h: ci.CsbMatrix, rank: int, world: int, device: ci.Device, tile_edge: int = 0,
                 plan=None):
        self.h = h
        self.rank, self.world = rank, world
        self.device = device
        self.row_bounds, self.halo_lo, self.halo_hi = plan if plan is not None else row_partition(h, world, tile_edge)
        self.row_lo, self.row_hi = int(self.row_bounds[rank]), int(self.row_bounds[rank + 1])
        lib = _lib.load()
        v = h.view()
        g = np.ascontiguousarray(h.groups, dtype=np.uint32) if h.groups is not None else None
        handle = C.c_void_p()
        ci._check(lib.cieg_matrix_upload_shard(device.handle, C.byref(v), None if g is None else ci._ptr(g, C.c_uint32),
                                               0 if g is None else len(g) - 1, tile_edge, self.row_lo, self.row_hi,
                                               C.byref(handle)))
        self.handle = handle
        import weakref

        self._fin = weakref.finalize(self, lib.cieg_matrix_destroy, handle)

    @property
    def local_rows(self) -> int:
        return self.row_hi - self.row_lo

    def spmm(self, x_local: torch.Tensor, group=None) -> torch.Tensor:
        """Rows [row_lo, row_hi) of H X from the rank's rows of X."""
        m = x_local.shape[1]
        full = torch.empty((self.h.dim, m), dtype=torch.float64, device=x_local.device)
        allgather_rows(x_local, self.row_bounds, full, group)
        y = torch.empty((self.local_rows, m), dtype=torch.float64, device=x_local.device)
        torch.cuda.current_stream().synchronize()
        ci._check(_lib.load().cieg_spmm(self.device.handle, self.handle, C.c_void_p(full.data_ptr()),
                                        C.c_void_p(y.data_ptr()), m))
        self.device.synchronize()
        return y


def local_tile_diagonal(h: ci.CsbMatrix, row_lo: int, row_hi: int, device: ci.Device) -> ci.TileDiagonal:
    g = np.ascontiguousarray(h.groups, dtype=np.uint32)
    v = h.view()
    handle = C.c_void_p()
    ci._check(_lib.load().cieg_precond_from_csb_range(device.handle, C.byref(v), ci._ptr(g, C.c_uint32), len(g) - 1,
                                                      row_lo, row_hi, C.byref(handle)))
    lb = g[(g >= row_lo) & (g <= row_hi)].astype(np.int64) - row_lo
    return ci.TileDiagonal(handle, lb.astype(np.uint32), device)


def lobpcg_solve_dist(sm: ShardedMatrix, x0_local: np.ndarray, options: ci.LobpcgOptions,
                      precond: Optional[ci.TileDiagonal] = None, group=None) -> ci.SolveReport:
    """Sharded ci::lobpcg_solve. x0_local = the rank's rows of X0. The report's
    trial vectors are the rank's rows; eigenvalues/history are global."""
    lib = _lib.load()
    dev = sm.device
    tdev = torch.device("cuda", dev.index)
    # One dedicated stream carries both the library's kernels and the
    # collectives issued from the hooks, so they are ordered without host syncs.
    torch_stream = torch.cuda.Stream(device=tdev)
    prev_stream = torch.cuda.current_stream(tdev)
    torch.cuda.set_stream(torch_stream)
    ci._check(lib.cieg_ctx_set_stream(dev.handle, C.c_void_p(torch_stream.cuda_stream)))
    rb = sm.row_bounds
    dim = sm.h.dim

    def _allreduce(_user, buf, count):
        try:
            host = np.ctypeslib.as_array(buf, (count,))
            t = torch.from_numpy(host.copy()).to(tdev)
            allreduce_sum_(t, group)
            host[:] = t.cpu().numpy()
            return 0
        except Exception:  # noqa: BLE001 -- report through the status code
            return 1

    def _allgather(_user, xptr, m, fullptr):
        try:
            nloc = sm.local_rows
            xl = _view(xptr, (nloc, m), tdev)
            full = _view(fullptr, (dim, m), tdev)
            allgather_rows(xl, rb, full, group)
            return 0
        except Exception:  # noqa: BLE001
            return 1

    hooks = _lib.DistHooks()
    hooks.user = None
    hooks.allreduce_sum = _lib.ALLREDUCE_FN(_allreduce)
    hooks.allgather_rows = _lib.ALLGATHER_FN(_allgather)
    opt = _lib.LobpcgOptionsC()
    opt.k_want, opt.tol, opt.max_iter = options.k_want, options.tol, options.max_iter
    opt.precond_config = options.precond_config.c()
    x0 = ci._f64(x0_local)
    rep = C.c_void_p()
    try:
        ci._check(lib.cieg_lobpcg_solve_dist(dev.handle, sm.handle, ci._ptr(x0), x0.shape[1],
                                             precond.handle if precond is not None else None, C.byref(opt),
                                             C.byref(hooks), C.byref(rep)))
    finally:
        lib.cieg_ctx_set_stream(dev.handle, None)
        torch.cuda.set_stream(prev_stream)
    return ci._read_report(lib, rep, sm.local_rows)
