"""Row-block sharding of the LOBPCG path over several GPUs,
one process per GPU with torch.distributed for the plumbing.

* Partition: ``row_partition`` (cieg_shard_plan) cuts the rows at group
  boundaries, balanced by the entries each owner streams. Every rank owns its
  rows of H's owner work lists (row parts and the transposed parts of tiles
  (I, P) landing in its rows -- owner-computes needs no reduce-scatter of
  transposed partials; tiles on a shard boundary are held by both owners) and
  its rows of every block vector and tile-diagonal group.
* SpMM: each rank's owner kernel reads X only on its halo rows
  [halo_lo, halo_hi) (cieg_matrix_rows), so before K1 every rank receives
  exactly the rows of its halo that other ranks own, point to point
  (``halo_exchange``: batched isend/irecv, SURVEY.md 8(e) "optimised
  variant"), then writes its rows of U. For the block-banded sector matrices
  the halo is the +-2-sector band, so the exchanged volume stays flat as the
  rank count grows, where an all-gather (``allgather_rows``, kept for
  comparison) moves (G-1)/G of X to every rank.
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


class ExchangePlan:
    """Who sends which owned rows to whom: recvs[(peer, a, b)] = peer's rows
    [a, b) inside this rank's halo, sends[(peer, a, b)] = this rank's rows
    inside peer's halo. Built from every rank's row bounds and halo."""

    def __init__(self, row_bounds, halo_lo, halo_hi, rank: int):
        world = len(row_bounds) - 1
        self.rank = rank
        self.lo, self.hi = int(row_bounds[rank]), int(row_bounds[rank + 1])
        self.sends, self.recvs = [], []
        for s in range(world):
            if s == rank:
                continue
            a, b = max(self.lo, int(halo_lo[s])), min(self.hi, int(halo_hi[s]))
            if b > a:
                self.sends.append((s, a, b))
            a, b = max(int(row_bounds[s]), int(halo_lo[rank])), min(int(row_bounds[s + 1]), int(halo_hi[rank]))
            if b > a:
                self.recvs.append((s, a, b))

    def recv_rows(self) -> int:
        return sum(b - a for _, a, b in self.recvs)

    def send_rows(self) -> int:
        return sum(b - a for _, a, b in self.sends)


def gather_halos(halo_lo: int, halo_hi: int, device, group=None):
    """Every rank's (halo_lo, halo_hi), from each rank's own matrix."""
    world = dist.get_world_size(group)
    mine = torch.tensor([halo_lo, halo_hi], dtype=torch.int64, device=device)
    allh = [torch.zeros(2, dtype=torch.int64, device=device) for _ in range(world)]
    dist.all_gather(allh, mine, group=group)
    hs = torch.stack(allh).cpu().numpy()
    return hs[:, 0], hs[:, 1]


def halo_exchange(x_local: torch.Tensor, plan: ExchangePlan, out: torch.Tensor, group=None,
                  out_row0: int = 0) -> torch.Tensor:
    """X[a:b] into out for every row this rank's SpMM reads: own rows copied,
    peers' rows received point to point (one batched isend/irecv round).
    out[i] holds global row out_row0 + i (a halo-sized buffer: out_row0 =
    halo_lo; a full-length one: 0)."""
    if out_row0:
        lo = plan.lo - out_row0
        sub = ExchangePlan.__new__(ExchangePlan)
        sub.rank, sub.lo, sub.hi = plan.rank, lo, lo + (plan.hi - plan.lo)
        sub.sends = [(p, a - out_row0, b - out_row0) for p, a, b in plan.sends]
        sub.recvs = [(p, a - out_row0, b - out_row0) for p, a, b in plan.recvs]
        plan = sub
    out[plan.lo:plan.hi].copy_(x_local)
    if out.is_cuda and dist.get_backend(group) == "gloo":
        # gloo moves host tensors only (single-GPU multi-rank runs): stage
        xh = x_local.cpu()
        hb = {(a, b): torch.empty((b - a,) + tuple(out.shape[1:]), dtype=out.dtype) for _, a, b in plan.recvs}
        ops = [dist.P2POp(dist.irecv, hb[(a, b)], peer if group is None else dist.get_global_rank(group, peer), group)
               for peer, a, b in plan.recvs]
        ops += [dist.P2POp(dist.isend, xh[a - plan.lo:b - plan.lo].contiguous(),
                           peer if group is None else dist.get_global_rank(group, peer), group)
                for peer, a, b in plan.sends]
        if ops:
            for w in dist.batch_isend_irecv(ops):
                w.wait()
        for (a, b), t in hb.items():
            out[a:b].copy_(t)
        return out
    ops = []
    for peer, a, b in plan.recvs:
        g = peer if group is None else dist.get_global_rank(group, peer)
        ops.append(dist.P2POp(dist.irecv, out[a:b], g, group))
    for peer, a, b in plan.sends:
        g = peer if group is None else dist.get_global_rank(group, peer)
        ops.append(dist.P2POp(dist.isend, x_local[a - plan.lo:b - plan.lo], g, group))
    if ops:
        for w in dist.batch_isend_irecv(ops):
            w.wait()
    return out


class PartialPlan:
    """The reverse of the halo exchange for the single-pass SpMM
    (cieg_spmm_partial): every rank holds transposed partial sums for rows
    [part_lo, row_lo) owned by lower ranks. sends[(peer, a, b)] = rows of
    peer inside this rank's partial range; recvs[(peer, a, b)] = this rank's
    rows inside peer's partial range (peers above this rank)."""

    def __init__(self, row_bounds, part_lo, rank: int):
        world = len(row_bounds) - 1
        self.rank = rank
        self.lo, self.hi = int(row_bounds[rank]), int(row_bounds[rank + 1])
        self.part_lo = int(part_lo[rank])
        self.sends, self.recvs = [], []
        for s in range(world):
            if s < rank:  # rows of a lower owner inside my partial range
                a, b = max(int(row_bounds[s]), self.part_lo), min(int(row_bounds[s + 1]), self.lo)
                if b > a:
                    self.sends.append((s, a, b))
            elif s > rank:  # my rows inside a higher rank's partial range
                a, b = max(self.lo, int(part_lo[s])), min(self.hi, int(row_bounds[s]))
                if b > a:
                    self.recvs.append((s, a, b))

    def recv_rows(self) -> int:
        return sum(b - a for _, a, b in self.recvs)

    def send_rows(self) -> int:
        return sum(b - a for _, a, b in self.sends)


def gather_partial_lo(part_lo: int, device, group=None):
    world = dist.get_world_size(group)
    mine = torch.tensor([part_lo], dtype=torch.int64, device=device)
    allp = [torch.zeros(1, dtype=torch.int64, device=device) for _ in range(world)]
    dist.all_gather(allp, mine, group=group)
    return torch.cat(allp).cpu().numpy()


def partial_reduce(yhalo: torch.Tensor, plan: PartialPlan, y_local: torch.Tensor, group=None) -> torch.Tensor:
    """Send this rank's partial rows to their owners and add the partials
    received for its own rows: point to point (one batched isend/irecv
    round), added in ascending peer order -- deterministic for a fixed
    partition. yhalo[i] holds global row plan.part_lo + i."""
    staged = y_local.is_cuda and dist.get_backend(group) == "gloo"  # gloo moves host tensors only
    src = yhalo.cpu() if staged else yhalo
    bufs = [(peer, a, b, torch.empty((b - a,) + tuple(y_local.shape[1:]), dtype=y_local.dtype,
                                      device="cpu" if staged else y_local.device))
            for peer, a, b in sorted(plan.recvs)]
    ops = [dist.P2POp(dist.irecv, t, peer if group is None else dist.get_global_rank(group, peer), group)
           for peer, a, b, t in bufs]
    ops += [dist.P2POp(dist.isend, src[a - plan.part_lo:b - plan.part_lo].contiguous(),
                       peer if group is None else dist.get_global_rank(group, peer), group)
            for peer, a, b in plan.sends]
    if ops:
        for w in dist.batch_isend_irecv(ops):
            w.wait()
    for peer, a, b, t in bufs:  # ascending peer order
        y_local[a - plan.lo:b - plan.lo] += t.to(y_local.device)
    return y_local


def spmm_single_pass(handle, device: ci.Device, x_full: torch.Tensor, y_local: torch.Tensor, plan: PartialPlan,
                     group=None) -> torch.Tensor:
    """H X on a shard in the single pass (cieg_spmm_partial): the local rows
    plus the transposed partials the higher ranks send (x_full: globally
    addressed, halo rows filled)."""
    m = x_full.shape[1]
    yhalo = torch.empty((max(plan.lo - plan.part_lo, 1), m), dtype=torch.float64, device=y_local.device)
    torch.cuda.current_stream().synchronize()
    ci._check(_lib.load().cieg_spmm_partial(device.handle, handle, C.c_void_p(x_full.data_ptr()),
                                            C.c_void_p(y_local.data_ptr()), m, C.c_void_p(yhalo.data_ptr())))
    device.synchronize()
    return partial_reduce(yhalo, plan, y_local, group)


def partial_rows(handle):
    lo, hi = C.c_uint32(), C.c_uint32()
    ci._check(_lib.load().cieg_matrix_partial_rows(handle, C.byref(lo), C.byref(hi)))
    return lo.value, hi.value


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
        self.plan = ExchangePlan(self.row_bounds, self.halo_lo, self.halo_hi, rank)

    @property
    def local_rows(self) -> int:
        return self.row_hi - self.row_lo

    @property
    def dim(self) -> int:
        return self.h.dim

    @property
    def halo(self):
        return int(self.halo_lo[self.rank]), int(self.halo_hi[self.rank])

    def spmm(self, x_local: torch.Tensor, group=None, exchange: str = "halo", mode: str = "owner") -> torch.Tensor:
        """Rows [row_lo, row_hi) of H X from the rank's rows of X (the halo
        rows of X arrive point to point; exchange="allgather" for the
        all-gather variant). mode="single": the single pass, whose
        transposed partials for lower ranks' rows go back point to point
        (collective: every rank calls it)."""
        m = x_local.shape[1]
        full = torch.empty((self.h.dim, m), dtype=torch.float64, device=x_local.device)
        if exchange == "halo":
            halo_exchange(x_local, self.plan, full, group)
        else:
            allgather_rows(x_local, self.row_bounds, full, group)
        y = torch.empty((self.local_rows, m), dtype=torch.float64, device=x_local.device)
        if mode == "single":
            if getattr(self, "partial_plan", None) is None:
                plo = gather_partial_lo(partial_rows(self.handle)[0], x_local.device, group)
                self.partial_plan = PartialPlan(self.row_bounds, plo, self.rank)
            return spmm_single_pass(self.handle, self.device, full, y, self.partial_plan, group)
        torch.cuda.current_stream().synchronize()
        ci._check(_lib.load().cieg_spmm(self.device.handle, self.handle, C.c_void_p(full.data_ptr()),
                                        C.c_void_p(y.data_ptr()), m))
        self.device.synchronize()
        return y


class DeviceShard:
    """This rank's shard generated on its GPU (cieg_generate_device with a
    row range): no host CSB anywhere -- the config-5 path (2e10 entries).
    Collective: every rank must construct its shard (halos are exchanged)."""

    def __init__(self, dm: ci.DeviceMatrix, row_bounds, group=None):
        self.dm = dm
        self.device = dm.device
        self.handle = dm.handle
        self.dim = dm.dim
        self.rank = dist.get_rank(group)
        self.row_bounds = np.asarray(row_bounds, dtype=np.int64)
        self.row_lo, self.row_hi = dm.row_lo, dm.row_hi
        assert self.row_lo == self.row_bounds[self.rank] and self.row_hi == self.row_bounds[self.rank + 1]
        tdev = torch.device("cuda", dm.device.index)
        self.halo_lo_all, self.halo_hi_all = gather_halos(dm.halo_lo, dm.halo_hi, tdev, group)
        self.plan = ExchangePlan(self.row_bounds, self.halo_lo_all, self.halo_hi_all, self.rank)

    @classmethod
    def generate(cls, cfg, row_bounds, device: ci.Device, group=None, seed: Optional[int] = None) -> "DeviceShard":
        rank = dist.get_rank(group)
        dm = cfg.generate_device(device=device, rows=(int(row_bounds[rank]), int(row_bounds[rank + 1])), seed=seed)
        return cls(dm, row_bounds, group)

    @property
    def local_rows(self) -> int:
        return self.row_hi - self.row_lo

    @property
    def halo(self):
        return int(self.dm.halo_lo), int(self.dm.halo_hi)


def generated_row_bounds(cfg, world: int):
    """Row cuts for GPU-generated shards on the device panel grid
    (cieg_generated_panels: small groups merge into panels), balanced by the
    generator's expected streamed entries per row (edge sectors couple to
    fewer neighbours than interior ones)."""
    gb = ci.generated_panels(cfg.n, cfg.sectors, cfg.tile, precision=cfg.precision, beta=cfg.beta)
    # expected row weight: sectors within the +-2 band around the row's sector
    sec = np.minimum((gb[:-1] * cfg.sectors) // cfg.n, cfg.sectors - 1)
    neigh = np.array([min(s + 2, cfg.sectors - 1) - max(s - 2, 0) + 1 for s in sec], dtype=np.float64)
    w = neigh * np.diff(gb)
    cum = np.concatenate([[0.0], np.cumsum(w)])
    bounds = [0]
    for k in range(1, world):
        i = int(np.argmin(np.abs(cum - cum[-1] * k / world)))
        bounds.append(max(int(gb[i]), bounds[-1] + 1))
    bounds.append(cfg.n)
    return np.asarray(bounds, dtype=np.int64)


def local_tile_diagonal(h: ci.CsbMatrix, row_lo: int, row_hi: int, device: ci.Device) -> ci.TileDiagonal:
    g = np.ascontiguousarray(h.groups, dtype=np.uint32)
    v = h.view()
    handle = C.c_void_p()
    ci._check(_lib.load().cieg_precond_from_csb_range(device.handle, C.byref(v), ci._ptr(g, C.c_uint32), len(g) - 1,
                                                      row_lo, row_hi, C.byref(handle)))
    lb = g[(g >= row_lo) & (g <= row_hi)].astype(np.int64) - row_lo
    return ci.TileDiagonal(handle, lb.astype(np.uint32), device)


def lobpcg_solve_dist(sm, x0_local: np.ndarray, options: ci.LobpcgOptions,
                      precond: Optional[ci.TileDiagonal] = None, group=None,
                      single_pass: bool = True) -> ci.SolveReport:
    """Sharded ci::lobpcg_solve on a ShardedMatrix (host CSB uploaded by
    rows) or a DeviceShard (generated on the GPU). x0_local = the rank's rows
    of X0. The report's trial vectors are the rank's rows; eigenvalues,
    history and counters are global (identical on every rank).
    single_pass: SpMMs of the single-pass widths (the SpMM mode's rule) use
    the single pass with the partials reduced at their owners; False keeps
    every SpMM owner-computes."""
    lib = _lib.load()
    dev = sm.device
    tdev = torch.device("cuda", dev.index)
    # One dedicated stream carries both the library's kernels and the
    # collectives issued from the hooks, so they are ordered without host syncs.
    torch_stream = torch.cuda.Stream(device=tdev)
    prev_stream = torch.cuda.current_stream(tdev)
    torch.cuda.set_stream(torch_stream)
    ci._check(lib.cieg_ctx_set_stream(dev.handle, C.c_void_p(torch_stream.cuda_stream)))
    hlo, hhi = sm.halo

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
        # fullptr is globally indexed and backed on the halo rows only:
        # view exactly those and exchange point to point
        try:
            nloc = sm.local_rows
            xl = _view(xptr, (nloc, m), tdev)
            halo_buf = _view(fullptr + 8 * hlo * m, (hhi - hlo, m), tdev)
            halo_exchange(xl, sm.plan, halo_buf, group, out_row0=hlo)
            return 0
        except Exception:  # noqa: BLE001
            return 1

    # single-pass SpMM widths: transposed partials back to their owners
    plo = gather_partial_lo(partial_rows(sm.handle)[0], tdev, group)
    pplan = PartialPlan(sm.row_bounds, plo, dist.get_rank(group))

    def _partials(_user, yhptr, m, yptr):
        try:
            yl = _view(yptr, (sm.local_rows, m), tdev)
            yh = _view(yhptr, (max(pplan.lo - pplan.part_lo, 1), m), tdev)
            partial_reduce(yh, pplan, yl, group)
            return 0
        except Exception:  # noqa: BLE001
            return 1

    hooks = _lib.DistHooks()
    hooks.user = None
    hooks.allreduce_sum = _lib.ALLREDUCE_FN(_allreduce)
    hooks.allgather_rows = _lib.ALLGATHER_FN(_allgather)
    hooks.reduce_partials = _lib.PARTIALS_FN(_partials) if single_pass else _lib.PARTIALS_FN()
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


def nccl_init(dev: "ci.Device", group=None) -> None:
    """Give the device context its own NCCL communicator over the ranks of
    `group` (rank 0 creates the id, torch.distributed broadcasts it): the
    library's in-library data plane (cieg_lobpcg_solve_nccl)."""
    lib = _lib.load()
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    uid = (C.c_uint8 * 128)()
    if rank == 0:
        ci._check(lib.cieg_nccl_unique_id(uid))
    box = [bytes(uid)]
    dist.broadcast_object_list(box, src=0, group=group)
    uid = (C.c_uint8 * 128).from_buffer_copy(box[0])
    ci._check(lib.cieg_ctx_nccl_init(dev.handle, uid, world, rank))


def nccl_finalize(dev: "ci.Device") -> None:
    ci._check(_lib.load().cieg_ctx_nccl_finalize(dev.handle))


def lobpcg_solve_nccl(sm, x0_local: np.ndarray, options: ci.LobpcgOptions,
                      precond: Optional[ci.TileDiagonal] = None) -> ci.SolveReport:
    """lobpcg_solve_dist with the collectives inside the library (the
    context's NCCL communicator, nccl_init): Gram all-reduces on the device
    before the single D2H, the X halo exchange and the single-pass partial
    reduction as grouped ncclSend/ncclRecv -- no Python callback in the
    iteration. Same results as lobpcg_solve_dist."""
    lib = _lib.load()
    dev = sm.device
    opt = _lib.LobpcgOptionsC()
    opt.k_want, opt.tol, opt.max_iter = options.k_want, options.tol, options.max_iter
    opt.precond_config = options.precond_config.c()
    x0 = ci._f64(x0_local)
    rep = C.c_void_p()
    ci._check(lib.cieg_lobpcg_solve_nccl(dev.handle, sm.handle, ci._ptr(x0), x0.shape[1],
                                         precond.handle if precond is not None else None, C.byref(opt),
                                         C.byref(rep)))
    return ci._read_report(lib, rep, sm.local_rows)
