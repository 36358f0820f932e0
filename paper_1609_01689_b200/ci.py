"""Host-side mirror of the reference's ``ci::`` solver/operator API
(/root/reference/proj/include/ci/), backed by the sm_100a kernels of
libcieg.so through the C ABI in include/cieg.h.

Names, argument meaning and error behaviour follow the reference:

=============================  ===============================================
this module                    reference
=============================  ===============================================
CsbMatrix                      ci::CsbMatrix (csb.hpp:33-60)
spmm(h, x)                     ci::spmm (csb.hpp:83, csb.cpp:182-193)
block_inner(x, y)              ci::block_inner (block_vectors.hpp:60)
linear_combination(y, g)       ci::linear_combination (block_vectors.hpp:64)
add_linear_combination(y,x,g)  ci::add_linear_combination (block_vectors.hpp:68)
column_norms(x)                ci::column_norms (block_vectors.hpp:75)
random_block(n, k, seed)       ci::random_block (block_vectors.hpp:72)
PrecondConfig / ShiftPlan      ci::PrecondConfig / ci::ShiftPlan (precond.hpp:16-40)
choose_shifts(...)             ci::choose_shifts (precond.hpp:47-48)
extract_tile_diagonal(h, g)    ci::extract_tile_diagonal (hamiltonian.hpp:65)
apply_preconditioner(...)      ci::apply_preconditioner (precond.hpp:53-54)
LobpcgOptions / SolveReport    ci::LobpcgOptions / ci::SolveReport (lobpcg.hpp:34-60)
lobpcg_solve(h, x0, opt)       ci::lobpcg_solve (lobpcg.hpp:67-68)
write_history_csv(rep, os)     ci::write_history_csv (lobpcg.hpp:102)
save_csb / load_csb            ci::save_csb / ci::load_csb (csb.hpp:105-106)
=============================  ===============================================

Errors are raised as the reference's exception types (errors.hpp:9-32).
There is no CPU fallback: every compute call goes through libcieg.so on a
CUDA device and raises if the library or the device is unavailable.
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import io
import struct
import weakref
from typing import Callable, Optional, Sequence

import numpy as np

from . import _lib

# --------------------------------------------------------------------- errors


class Error(RuntimeError):
    """ci::Error (errors.hpp:9-12)."""


class DimensionMismatch(Error):
    pass


class ConfigError(Error):
    pass


class SubspaceCollapse(Error):
    pass


class FormatError(Error):
    pass


class IndefiniteGram(Error):
    pass


class BetaTooLarge(Error):
    pass


class CudaError(Error):
    pass


_STATUS = {1: DimensionMismatch, 2: ConfigError, 3: SubspaceCollapse, 4: FormatError,
           5: IndefiniteGram, 6: CudaError, 7: Error, 8: BetaTooLarge}


def _check(status: int) -> None:
    if status:
        msg = _lib.load().cieg_last_error().decode()
        raise _STATUS.get(status, Error)(msg)


def _ptr(a: np.ndarray, ctype=C.c_double):
    return a.ctypes.data_as(C.POINTER(ctype))


def _f64(x) -> np.ndarray:
    return np.ascontiguousarray(x, dtype=np.float64)


# --------------------------------------------------------------------- device

class Device:
    """One CUDA device + stream (cieg_ctx)."""

    _default: dict[int, "Device"] = {}

    def __init__(self, index: int = 0):
        lib = _lib.load()
        h = C.c_void_p()
        _check(lib.cieg_ctx_create(index, C.byref(h)))
        self.index = index
        self.handle = h
        self._fin = weakref.finalize(self, lib.cieg_ctx_destroy, h)

    @classmethod
    def default(cls, index: int = 0) -> "Device":
        d = cls._default.get(index)
        if d is None:
            d = cls._default[index] = Device(index)
        return d

    def synchronize(self) -> None:
        _check(_lib.load().cieg_ctx_synchronize(self.handle))

    def set_stream(self, stream: int) -> None:
        """Launch on an external CUDA stream (a cudaStream_t as int; 0 or
        None = back to the context's own stream). cieg_ctx_set_stream."""
        _check(_lib.load().cieg_ctx_set_stream(self.handle, C.c_void_p(stream) if stream else None))

    def set_exact_order(self, exact: bool) -> None:
        """True: the preconditioner's FOM follows the reference's operation
        order bit for bit; False (default): tensor-core products and parallel
        fixed-order reductions."""
        _check(_lib.load().cieg_ctx_set_exact_order(self.handle, 1 if exact else 0))

    SPMM_MODES = {"auto": 0, "owner": 1, "single": 2, "sliced": 3}

    def set_spmm_mode(self, mode: str) -> None:
        """SpMM mode: "auto" (default: single pass for widths <= 8 on
        unsharded matrices), "owner" (owner-computes) or "single" (single
        pass). cieg_ctx_set_spmm_mode."""
        if mode not in self.SPMM_MODES:
            raise ValueError(f"unknown SpMM mode {mode!r}")
        _check(_lib.load().cieg_ctx_set_spmm_mode(self.handle, self.SPMM_MODES[mode]))

    @property
    def stream(self) -> int:
        return int(_lib.load().cieg_ctx_stream(self.handle) or 0)

    @property
    def launches(self) -> int:
        return int(_lib.load().cieg_ctx_launch_count(self.handle))


# --------------------------------------------------------------------- matrix

@dataclasses.dataclass(eq=False)
class CsbMatrix:
    """Flattened ci::CsbMatrix: lower-triangle CSB blocks, block (I, J<=I) at
    linear index I(I+1)/2+J, entries sorted by (row, col) with 16-bit
    block-local offsets. ``groups`` (optional) holds the GroupPartition ranges
    (group = tile) used for the device panel plan and the preconditioner."""

    dim: int
    precision: int  # 0 single, 1 double
    block_boundaries: np.ndarray  # u32, nb + 1
    entry_offsets: np.ndarray  # u64, nb(nb+1)/2 + 1
    rows: np.ndarray  # u16
    cols: np.ndarray  # u16
    values: np.ndarray  # f32 / f64
    groups: Optional[np.ndarray] = None  # u32 bounds
    beta: int = 2000
    _keepalive: object = None

    @property
    def nnz_lower(self) -> int:
        return int(self.entry_offsets[-1])

    def block_count(self) -> int:
        return len(self.block_boundaries) - 1

    def view(self) -> _lib.CsbView:
        v = _lib.CsbView()
        v.dim = self.dim
        v.nb = self.block_count()
        v.precision = self.precision
        v.block_boundaries = _ptr(self.block_boundaries, C.c_uint32)
        v.entry_offsets = _ptr(self.entry_offsets, C.c_uint64)
        v.rows = _ptr(self.rows, C.c_uint16)
        v.cols = _ptr(self.cols, C.c_uint16)
        v.values = self.values.ctypes.data_as(C.c_void_p)
        return v

    def coo(self):
        """Global (row, col, value) triplets of the stored lower triangle."""
        nb = self.block_count()
        counts = np.diff(self.entry_offsets.astype(np.int64))
        bi = np.repeat(np.concatenate([np.full(i + 1, i) for i in range(nb)]), counts)
        bj = np.repeat(np.concatenate([np.arange(i + 1) for i in range(nb)]), counts)
        bb = self.block_boundaries.astype(np.int64)
        r = bb[bi] + self.rows.astype(np.int64)
        c = bb[bj] + self.cols.astype(np.int64)
        return r, c, self.values.astype(np.float64)

    def to_dense(self) -> np.ndarray:
        """ci::to_dense (csb.cpp:220-237); refuses dim > 5000."""
        if self.dim > 5000:
            raise DimensionMismatch("to_dense is a test oracle; dim > 5000")
        r, c, v = self.coo()
        m = np.zeros((self.dim, self.dim))
        m[r, c] = v
        m[c, r] = v
        return m


def generate_sector_matrix(n: int, sectors: int, tile: int, p: float, q: float, seed: int = 1,
                           precision: int = 0, beta: int = 2000, band: int = 2) -> CsbMatrix:
    """The BASELINE.json sector generator (generator.cpp)."""
    lib = _lib.load()
    prm = gen_params(n, sectors, tile, p, q, seed, precision, beta, band)
    h = C.c_void_p()
    _check(lib.cieg_generate_csb(C.byref(prm), C.byref(h)))
    try:
        return _copy_host_csb(lib, h, precision, beta)
    finally:
        lib.cieg_host_csb_destroy(h)


def _copy_host_csb(lib, h, precision, beta) -> CsbMatrix:
    v = _lib.CsbView()
    nnz = C.c_uint64()
    _check(lib.cieg_host_csb_view(h, C.byref(v), C.byref(nnz)))
    gb = C.POINTER(C.c_uint32)()
    ng = C.c_uint32()
    _check(lib.cieg_host_csb_groups(h, C.byref(gb), C.byref(ng)))
    nb = v.nb
    nblk = nb * (nb + 1) // 2
    as_np = np.ctypeslib.as_array
    vals_t = C.c_float if precision == 0 else C.c_double
    nz = int(nnz.value)
    # Copy out so the matrix owns its memory (the generator object is freed).
    mat = CsbMatrix(
        dim=v.dim, precision=v.precision,
        block_boundaries=as_np(v.block_boundaries, (nb + 1,)).copy(),
        entry_offsets=as_np(v.entry_offsets, (nblk + 1,)).copy(),
        rows=as_np(v.rows, (nz,)).copy() if nz else np.zeros(0, np.uint16),
        cols=as_np(v.cols, (nz,)).copy() if nz else np.zeros(0, np.uint16),
        values=(as_np(C.cast(v.values, C.POINTER(vals_t)), (nz,)).copy() if nz
                else np.zeros(0, np.float32 if precision == 0 else np.float64)),
        groups=as_np(gb, (ng.value + 1,)).copy(),
        beta=beta)
    return mat


def gen_params(n, sectors, tile, p, q, seed=1, precision=0, beta=2000, band=2) -> _lib.GenParams:
    prm = _lib.GenParams()
    prm.n, prm.sectors, prm.tile, prm.band = n, sectors, tile, band
    prm.p, prm.q, prm.seed, prm.precision, prm.beta = p, q, seed, precision, beta
    return prm


def generated_panels(n, sectors, tile, p=0.5, q=0.5, precision=0, beta=2000, band=2, tile_edge=0) -> np.ndarray:
    """The device panel grid cieg_generate_device plans (panel starts, n
    last): shard row ranges must be unions of whole panels."""
    prm = gen_params(n, sectors, tile, p, q, precision=precision, beta=beta, band=band)
    lib = _lib.load()
    cnt = C.c_uint32()
    _check(lib.cieg_generated_panels(C.byref(prm), tile_edge, None, 0, C.byref(cnt)))
    out = np.zeros(cnt.value + 1, np.uint32)
    _check(lib.cieg_generated_panels(C.byref(prm), tile_edge, _ptr(out, C.c_uint32), len(out), C.byref(cnt)))
    return out.astype(np.int64)


def expected_nnz(n, sectors, tile, p, q, band=2) -> float:
    prm = gen_params(n, sectors, tile, p, q, band=band)
    return float(_lib.load().cieg_gen_expected_nnz(C.byref(prm)))


def count_nnz(n, sectors, tile, p, q, seed, band=2) -> int:
    """Exact stored-entry count of generate_sector_matrix(...) without building it."""
    prm = gen_params(n, sectors, tile, p, q, seed=seed, band=band)
    return int(_lib.load().cieg_gen_count_nnz(C.byref(prm)))


def avg_row_nnz(n, sectors, tile, p, q, band=2) -> float:
    prm = gen_params(n, sectors, tile, p, q, band=band)
    return float(_lib.load().cieg_gen_avg_row_nnz(C.byref(prm)))


def random_block(dim: int, width: int, seed: int) -> np.ndarray:
    """ci::random_block (block_vectors.cpp:162-174)."""
    out = np.empty((dim, width), dtype=np.float64)
    _check(_lib.load().cieg_random_block(dim, width, seed, _ptr(out)))
    return out


def random_block_rows(row_lo: int, row_hi: int, width: int, seed: int) -> np.ndarray:
    """Rows [row_lo, row_hi) of random_block(dim, width, seed) (a shard's X0)."""
    out = np.empty((row_hi - row_lo, width), dtype=np.float64)
    _check(_lib.load().cieg_random_block_rows(row_lo, row_hi, width, seed, _ptr(out)))
    return out


# CSB1 binary format (csb.cpp:256-331)

def save_csb(h: CsbMatrix, path: str) -> None:
    nb = h.block_count()
    groups = 0 if h.groups is None else len(h.groups) - 1
    with open(path, "wb") as f:
        f.write(b"CSB1")
        f.write(struct.pack("<IQIIQQQ", 0 if h.precision == 0 else 1, h.dim, h.beta, nb, h.nnz_lower,
                            groups, 0))
        f.write(np.asarray(h.block_boundaries, dtype="<u4").tobytes())
        vdt = "<f4" if h.precision == 0 else "<f8"
        rec = np.dtype([("r", "<u2"), ("c", "<u2"), ("v", vdt)])
        for b in range(nb * (nb + 1) // 2):
            e0, e1 = int(h.entry_offsets[b]), int(h.entry_offsets[b + 1])
            f.write(struct.pack("<Q", e1 - e0))
            if e1 > e0:
                a = np.empty(e1 - e0, dtype=rec)
                a["r"], a["c"], a["v"] = h.rows[e0:e1], h.cols[e0:e1], h.values[e0:e1]
                f.write(a.tobytes())


def load_csb(path: str) -> CsbMatrix:
    with open(path, "rb") as f:
        data = f.read()
    if data[:4] != b"CSB1":
        raise FormatError(f"bad magic; not a CSB1 file: {path}")
    try:
        prec, dim, beta, nb, nnz, groups, tiles = struct.unpack_from("<IQIIQQQ", data, 4)
    except struct.error as e:
        raise FormatError("truncated CSB file") from e
    if prec > 1:
        raise FormatError("bad precision tag")
    off = 4 + struct.calcsize("<IQIIQQQ")
    bb = np.frombuffer(data, dtype="<u4", count=nb + 1, offset=off).astype(np.uint32)
    off += 4 * (nb + 1)
    if bb[0] != 0 or bb[-1] != dim:
        raise FormatError("inconsistent block boundaries")
    vdt = "<f4" if prec == 0 else "<f8"
    rec = np.dtype([("r", "<u2"), ("c", "<u2"), ("v", vdt)])
    nblk = nb * (nb + 1) // 2
    offs = np.zeros(nblk + 1, dtype=np.uint64)
    parts = []
    for b in range(nblk):
        if off + 8 > len(data):
            raise FormatError("truncated CSB file")
        (cnt,) = struct.unpack_from("<Q", data, off)
        off += 8
        if off + cnt * rec.itemsize > len(data):
            raise FormatError("truncated CSB file")
        parts.append(np.frombuffer(data, dtype=rec, count=cnt, offset=off))
        off += cnt * rec.itemsize
        offs[b + 1] = offs[b] + cnt
    if int(offs[-1]) != nnz:
        raise FormatError("entry count disagrees with header")
    allr = np.concatenate(parts) if parts else np.zeros(0, dtype=rec)
    return CsbMatrix(dim=int(dim), precision=int(prec), block_boundaries=bb, entry_offsets=offs,
                     rows=allr["r"].astype(np.uint16), cols=allr["c"].astype(np.uint16),
                     values=allr["v"].astype(np.float32 if prec == 0 else np.float64), beta=int(beta))


class DeviceMatrix:
    """H re-tiled and resident in HBM (cieg_mat)."""

    def __init__(self, h: Optional[CsbMatrix], device: Optional[Device] = None, tile_edge: int = 0,
                 _handle: Optional[C.c_void_p] = None, cuts: Optional[Sequence[int]] = None,
                 _parent: Optional["DeviceMatrix"] = None):
        self.device = device or Device.default()
        self._parent = _parent  # a leading view borrows its parent's tile stream
        lib = _lib.load()
        if _handle is None:
            v = h.view()
            handle = C.c_void_p()
            gptr, ng = None, 0
            if h.groups is not None:
                g = np.ascontiguousarray(h.groups, dtype=np.uint32)
                gptr, ng = _ptr(g, C.c_uint32), len(g) - 1
            cu = np.ascontiguousarray(cuts if cuts is not None else [], dtype=np.uint32)
            _check(lib.cieg_matrix_upload_cuts(self.device.handle, C.byref(v), gptr, ng, tile_edge,
                                               _ptr(cu, C.c_uint32), len(cu), C.byref(handle)))
        else:
            handle = _handle
        self.handle = handle
        self._fin = weakref.finalize(self, lib.cieg_matrix_destroy, handle)
        info = [C.c_uint32(), C.c_uint64(), C.c_uint32(), C.c_uint64(), C.c_uint32(), C.c_int(), C.c_uint64()]
        _check(lib.cieg_matrix_info(handle, *[C.byref(x) for x in info]))
        (self.dim, self.nnz, self.npanels, self.ntiles, self.tile_edge, self.precision,
         self.tile_bytes) = [x.value for x in info]
        rows = [C.c_uint32() for _ in range(4)]
        _check(lib.cieg_matrix_rows(handle, *[C.byref(x) for x in rows]))
        self.row_lo, self.row_hi, self.halo_lo, self.halo_hi = [x.value for x in rows]

    @classmethod
    def generate(cls, n, sectors, tile, p, q, seed=1, precision=0, beta=2000, band=2,
                 device: Optional[Device] = None, tile_edge: int = 0, rows=None) -> "DeviceMatrix":
        """The BASELINE generator run on the GPU (cieg_generate_device): the
        tile stream is written in HBM directly, bit-identical to uploading
        generate_sector_matrix(...). `rows` = (row_lo, row_hi) for a shard."""
        dev = device or Device.default()
        prm = gen_params(n, sectors, tile, p, q, seed, precision, beta, band)
        lo, hi = (0, 0) if rows is None else rows
        handle = C.c_void_p()
        _check(_lib.load().cieg_generate_device(dev.handle, C.byref(prm), tile_edge, lo, hi, C.byref(handle)))
        return cls(None, dev, _handle=handle)

    def leading(self, dim: int) -> "DeviceMatrix":
        """H[0:dim, 0:dim] as a matrix of its own sharing this matrix's tile
        stream (cieg_matrix_leading_view); dim must be a device panel
        boundary (upload with cuts=[dim, ...] to make it one)."""
        handle = C.c_void_p()
        _check(_lib.load().cieg_matrix_leading_view(self.device.handle, self.handle, int(dim), C.byref(handle)))
        return DeviceMatrix(None, self.device, _handle=handle, _parent=self)

    def groups(self) -> np.ndarray:
        b = C.POINTER(C.c_uint32)()
        ng = C.c_uint32()
        _check(_lib.load().cieg_matrix_groups(self.handle, C.byref(b), C.byref(ng)))
        return np.ctypeslib.as_array(b, (ng.value + 1,)).copy() if ng.value else np.zeros(0, np.uint32)

    def export(self):
        """(tile_off, tile_pi, tile_pj, idx, val) of the device tile stream."""
        to = np.zeros(self.ntiles + 1, np.uint64)
        pi = np.zeros(self.ntiles, np.uint32)
        pj = np.zeros(self.ntiles, np.uint32)
        _check(_lib.load().cieg_matrix_export(self.handle, _ptr(to, C.c_uint64), None, None, None, None))
        slots = int(to[-1])
        idx = np.zeros(slots, np.uint32)
        val = np.zeros(slots, np.float32 if self.precision == 0 else np.float64)
        _check(_lib.load().cieg_matrix_export(self.handle, _ptr(to, C.c_uint64), _ptr(pi, C.c_uint32),
                                              _ptr(pj, C.c_uint32), _ptr(idx, C.c_uint32),
                                              val.ctypes.data_as(C.c_void_p)))
        return to, pi, pj, idx, val

    def spmm_host(self, x: np.ndarray) -> np.ndarray:
        x = _f64(x)
        if x.ndim != 2 or x.shape[0] != self.dim:
            raise DimensionMismatch("spmm: vector dim != matrix dim")
        y = np.empty((self.row_hi - self.row_lo, x.shape[1]))  # a shard returns its own rows
        _check(_lib.load().cieg_spmm_host(self.device.handle, self.handle, _ptr(x), _ptr(y), x.shape[1]))
        return y

    def spmm_host_batch(self, xs: Sequence[np.ndarray]) -> list:
        """Independent products H X_i through host memory with the copies of
        neighbouring products overlapping K1 (cieg_spmm_host_batch). Pass
        pinned arrays for full overlap."""
        xs = [_f64(x) for x in xs]
        if not xs:
            return []
        m = xs[0].shape[1]
        if any(x.shape != (self.dim, m) for x in xs):
            raise DimensionMismatch("spmm: vector dim != matrix dim")
        ys = [np.empty((self.row_hi - self.row_lo, m)) for _ in xs]
        pd = C.POINTER(C.c_double)
        xa = (pd * len(xs))(*[_ptr(x) for x in xs])
        ya = (pd * len(ys))(*[_ptr(y) for y in ys])
        _check(_lib.load().cieg_spmm_host_batch(self.device.handle, self.handle, xa, ya, m, len(xs)))
        return ys

    def spmm_ptr(self, x_ptr: int, y_ptr: int, m: int) -> None:
        """Device-pointer SpMM on the device's stream (row-major n x m)."""
        _check(_lib.load().cieg_spmm(self.device.handle, self.handle, C.c_void_p(x_ptr), C.c_void_p(y_ptr), m))

    SPMM_KERNELS = {1: "owner-computes", 2: "single pass", 3: "sliced"}

    def spmm_kernel(self, m: int) -> str:
        """The K1 kernel the device's current mode runs at width m here."""
        out = C.c_int()
        _check(_lib.load().cieg_spmm_effective_mode(self.device.handle, self.handle, m, C.byref(out)))
        return self.SPMM_KERNELS.get(out.value, str(out.value))

    def prepare(self, m: int = 16) -> str:
        """Build the device data of the K1 kernel for width m now (the sliced
        kernel's slice planes, otherwise built by the first SpMM); returns the
        kernel's name."""
        return self.spmm_kernel(m)


_UPLOADS: "weakref.WeakKeyDictionary[CsbMatrix, DeviceMatrix]" = weakref.WeakKeyDictionary()


def device_matrix(h: CsbMatrix, device: Optional[Device] = None) -> DeviceMatrix:
    """Upload-once cache: a CsbMatrix is re-tiled to HBM on first use."""
    dm = _UPLOADS.get(h)
    if dm is None or (device is not None and dm.device is not device):
        dm = _UPLOADS[h] = DeviceMatrix(h, device)
    return dm


def spmm(h: CsbMatrix, x: np.ndarray) -> np.ndarray:
    """U = (L + L^T - diag L) X -- ci::spmm."""
    x = _f64(x)
    if x.ndim != 2 or x.shape[0] != h.dim:
        raise DimensionMismatch("spmm: vector dim != matrix dim")
    return device_matrix(h).spmm_host(x)


# ------------------------------------------------------------ block kernels

class _DevArray:
    """Minimal device buffer for the host-array convenience wrappers."""

    def __init__(self, host: np.ndarray):
        import torch  # device memory plumbing only

        self.t = torch.from_numpy(np.ascontiguousarray(host, dtype=np.float64)).to("cuda")

    @property
    def ptr(self) -> C.c_void_p:
        return C.c_void_p(self.t.data_ptr())

    def host(self) -> np.ndarray:
        return self.t.cpu().numpy()


def _dev(d: Optional[Device]) -> Device:
    return d or Device.default()


def block_inner(x: np.ndarray, y: np.ndarray, device: Optional[Device] = None) -> np.ndarray:
    """X^T Y (column-major Eigen layout in, numpy out) -- ci::block_inner."""
    x, y = _f64(x), _f64(y)
    if x.shape[0] != y.shape[0]:
        raise DimensionMismatch("block_inner: row counts differ")
    dev = _dev(device)
    dx, dy = _DevArray(x), _DevArray(y)
    kx, ky = x.shape[1], y.shape[1]
    out = np.zeros(kx * ky)
    dev.synchronize()
    _check(_lib.load().cieg_block_inner(dev.handle, x.shape[0], dx.ptr, kx, dy.ptr, ky, _ptr(out)))
    return out.reshape(ky, kx).T.copy()


def linear_combination(y: np.ndarray, g: np.ndarray, device: Optional[Device] = None) -> np.ndarray:
    """Y G -- ci::linear_combination."""
    y, g = _f64(y), _f64(g)
    if g.shape[0] != y.shape[1]:
        raise DimensionMismatch("linear_combination: G rows != block width")
    dev = _dev(device)
    dy = _DevArray(y)
    do = _DevArray(np.zeros((y.shape[0], g.shape[1])))
    gc = np.asfortranarray(g)
    dev.synchronize()
    _check(_lib.load().cieg_linear_combination(dev.handle, y.shape[0], dy.ptr, y.shape[1],
                                               gc.ctypes.data_as(C.POINTER(C.c_double)), g.shape[1], do.ptr))
    dev.synchronize()
    return do.host()


def add_linear_combination(y: np.ndarray, x: np.ndarray, g: np.ndarray, device: Optional[Device] = None) -> None:
    """Y += X G in place -- ci::add_linear_combination."""
    x, g = _f64(x), _f64(g)
    if x.shape[0] != y.shape[0]:
        raise DimensionMismatch("add_linear_combination: dims")
    if g.shape != (x.shape[1], y.shape[1]):
        raise DimensionMismatch("add_linear_combination: G shape")
    dev = _dev(device)
    dy, dx = _DevArray(y), _DevArray(x)
    gc = np.asfortranarray(g)
    dev.synchronize()
    _check(_lib.load().cieg_add_linear_combination(dev.handle, y.shape[0], dy.ptr, y.shape[1], dx.ptr, x.shape[1],
                                                   gc.ctypes.data_as(C.POINTER(C.c_double))))
    dev.synchronize()
    y[...] = dy.host()


def column_norms(x: np.ndarray, device: Optional[Device] = None) -> np.ndarray:
    """Per-column norms -- ci::column_norms."""
    x = _f64(x)
    dev = _dev(device)
    dx = _DevArray(x)
    out = np.zeros(x.shape[1])
    dev.synchronize()
    _check(_lib.load().cieg_column_norms(dev.handle, x.shape[0], dx.ptr, x.shape[1], _ptr(out)))
    return out


# ------------------------------------------------------------ preconditioner

@dataclasses.dataclass
class PrecondConfig:
    """ci::PrecondConfig (precond.hpp:16-28) with its defaults."""

    inner_iters: int = 3
    small_block_cutoff: int = 64
    engage_after: int = 3
    relres_gate: float = 1e-1
    near_converged_factor: float = 10.0
    far_threshold: float = 1e-2
    column_floor_factor: float = 100.0

    def c(self) -> _lib.PrecondConfigC:
        s = _lib.PrecondConfigC()
        for f in dataclasses.fields(self):
            setattr(s, f.name, getattr(self, f.name))
        return s

    def as_array(self) -> np.ndarray:
        return np.array([getattr(self, f.name) for f in dataclasses.fields(self)], dtype=np.float64)


@dataclasses.dataclass
class ShiftPlan:
    mu: np.ndarray
    engage: np.ndarray  # bool


def choose_shifts(theta, res_norm, x_norm, relres, iteration: int, tol: float,
                  config: PrecondConfig = PrecondConfig()) -> ShiftPlan:
    """ci::choose_shifts (precond.cpp:13-55)."""
    th, rn, xn, rr = (_f64(a) for a in (theta, res_norm, x_norm, relres))
    k = len(th)
    mu = np.zeros(k)
    en = np.zeros(k, dtype=np.int32)
    cfg = config.c()
    _check(_lib.load().cieg_choose_shifts(k, _ptr(th), _ptr(rn), _ptr(xn), _ptr(rr), iteration, tol,
                                          C.byref(cfg), _ptr(mu), _ptr(en, C.c_int)))
    return ShiftPlan(mu=mu, engage=en.astype(bool))


class TileDiagonal:
    """ci::TileDiagonal resident on the device (cieg_prec)."""

    def __init__(self, handle: C.c_void_p, bounds: np.ndarray, device: Device):
        self.handle = handle
        self.bounds = bounds
        self.device = device
        self._fin = weakref.finalize(self, _lib.load().cieg_precond_destroy, handle)

    def group_count(self) -> int:
        return len(self.bounds) - 1

    @classmethod
    def from_blocks(cls, bounds, blocks: Sequence[np.ndarray], device: Optional[Device] = None) -> "TileDiagonal":
        dev = _dev(device)
        b = np.ascontiguousarray(bounds, dtype=np.uint32)
        flat = np.concatenate([np.asfortranarray(x, dtype=np.float64).ravel(order="F") for x in blocks]) \
            if len(blocks) else np.zeros(0)
        v = _lib.TileDiagView()
        v.dim, v.ngroups = int(b[-1]), len(b) - 1
        v.bounds = _ptr(b, C.c_uint32)
        v.blocks = _ptr(flat)
        h = C.c_void_p()
        _check(_lib.load().cieg_precond_upload(dev.handle, C.byref(v), C.byref(h)))
        return cls(h, b, dev)


def extract_tile_diagonal(h: CsbMatrix, groups=None, device: Optional[Device] = None) -> TileDiagonal:
    """ci::extract_tile_diagonal (hamiltonian.cpp:178-203)."""
    dev = _dev(device)
    g = np.ascontiguousarray(h.groups if groups is None else groups, dtype=np.uint32)
    v = h.view()
    handle = C.c_void_p()
    _check(_lib.load().cieg_precond_from_csb(dev.handle, C.byref(v), _ptr(g, C.c_uint32), len(g) - 1,
                                             C.byref(handle)))
    return TileDiagonal(handle, g, dev)


def tile_diagonal_from_matrix(dm: DeviceMatrix) -> TileDiagonal:
    """Tile diagonal built on the device from the matrix's diagonal tiles
    (cieg_precond_from_matrix; shard-local for a shard)."""
    handle = C.c_void_p()
    _check(_lib.load().cieg_precond_from_matrix(dm.device.handle, dm.handle, C.byref(handle)))
    g = dm.groups().astype(np.int64)
    lb = g[(g >= dm.row_lo) & (g <= dm.row_hi)] - dm.row_lo
    return TileDiagonal(handle, lb.astype(np.uint32), dm.device)


def apply_preconditioner(tiles: TileDiagonal, r: np.ndarray, plan: ShiftPlan,
                         config: PrecondConfig = PrecondConfig()) -> np.ndarray:
    """ci::apply_preconditioner (precond.cpp:160-207)."""
    r = _f64(r)
    if len(plan.mu) != r.shape[1] or len(plan.engage) != r.shape[1]:
        raise DimensionMismatch("apply_preconditioner: plan width != residual width")
    if tiles.group_count() > 0 and int(tiles.bounds[-1]) != r.shape[0]:
        raise DimensionMismatch("apply_preconditioner: tiles do not cover the basis")
    dev = tiles.device
    dr = _DevArray(r)
    dw = _DevArray(np.zeros_like(r))
    mu = _f64(plan.mu)
    en = np.ascontiguousarray(plan.engage, dtype=np.int32)
    cfg = config.c()
    dev.synchronize()
    _check(_lib.load().cieg_precond_apply(dev.handle, tiles.handle, dr.ptr, r.shape[1], _ptr(mu),
                                          _ptr(en, C.c_int), C.byref(cfg), dw.ptr))
    dev.synchronize()
    return dw.host()


# -------------------------------------------------------------------- LOBPCG

@dataclasses.dataclass
class HistoryRow:
    iteration: int
    column: int
    relres: float
    theta: float


@dataclasses.dataclass
class OperationCounters:
    spmm_calls: int = 0
    spmv_equivalents: int = 0
    precond_applications: int = 0
    orthogonalizations: int = 0


@dataclasses.dataclass
class SolveReport:
    eigenvalues: np.ndarray
    eigenvectors: np.ndarray
    trial_vectors: np.ndarray
    history: list
    counters: OperationCounters
    converged: bool
    iterations: int
    norm_estimate: float
    timing_ms: dict


@dataclasses.dataclass
class IterationView:
    iteration: int
    X: np.ndarray
    theta: np.ndarray
    relres: np.ndarray


@dataclasses.dataclass
class LobpcgOptions:
    """ci::LobpcgOptions (lobpcg.hpp:54-61)."""

    k_want: int = 8
    tol: float = 1e-6
    max_iter: int = 500
    preconditioner: Optional[TileDiagonal] = None
    precond_config: PrecondConfig = dataclasses.field(default_factory=PrecondConfig)
    observer: Optional[Callable[[IterationView], None]] = None


_TIMING_KEYS = ("spmm", "rayleigh_ritz", "orthonormalization", "preconditioner", "residual", "other", "total")


def lobpcg_solve(h, x0: np.ndarray, options: LobpcgOptions = LobpcgOptions(),
                 device: Optional[Device] = None) -> SolveReport:
    """ci::lobpcg_solve (lobpcg.cpp:216-387) on the GPU. `h` is a CsbMatrix
    (uploaded once) or an already resident DeviceMatrix."""
    x0 = _f64(x0)
    if x0.shape[0] != h.dim:
        raise DimensionMismatch("lobpcg: X0 dim != matrix dim")
    if x0.shape[1] < options.k_want:
        raise ConfigError("lobpcg: trial width below k_want")
    lib = _lib.load()
    dm = h if isinstance(h, DeviceMatrix) else device_matrix(h, device)
    dev = dm.device
    opt = _lib.LobpcgOptionsC()
    opt.k_want, opt.tol, opt.max_iter = options.k_want, options.tol, options.max_iter
    opt.precond_config = options.precond_config.c()
    cb = _lib.OBSERVER()
    if options.observer is not None:
        user_obs = options.observer

        def _obs(_user, it, xp, n, kt, thp, rrp):
            X = np.ctypeslib.as_array(xp, (n, kt)).copy()
            th = np.ctypeslib.as_array(thp, (kt,)).copy()
            rr = np.ctypeslib.as_array(rrp, (kt,)).copy()
            user_obs(IterationView(it, X, th, rr))

        cb = _lib.OBSERVER(_obs)
    rep = C.c_void_p()
    prec = options.preconditioner.handle if options.preconditioner is not None else None
    _check(lib.cieg_lobpcg_solve(dev.handle, dm.handle, _ptr(x0), x0.shape[1], prec, C.byref(opt), cb, None,
                                 C.byref(rep)))
    return _read_report(lib, rep, h.dim)


def _read_report(lib, rep, nrows: int) -> SolveReport:
    try:
        conv, iters, kw, kt = C.c_int(), C.c_int(), C.c_uint32(), C.c_uint32()
        ne, nh = C.c_double(), C.c_uint64()
        _check(lib.cieg_report_summary(rep, C.byref(conv), C.byref(iters), C.byref(ne), C.byref(kw), C.byref(kt),
                                       C.byref(nh)))
        cnt = np.zeros(4, dtype=np.uint64)
        _check(lib.cieg_report_counters(rep, _ptr(cnt, C.c_uint64)))
        ev = np.zeros(kw.value)
        _check(lib.cieg_report_eigenvalues(rep, _ptr(ev)))
        trial = np.zeros((nrows, kt.value))
        _check(lib.cieg_report_trial_vectors(rep, _ptr(trial)))
        n = nh.value
        hi, hc = np.zeros(n, np.int32), np.zeros(n, np.int32)
        hr, ht = np.zeros(n), np.zeros(n)
        _check(lib.cieg_report_history(rep, _ptr(hi, C.c_int), _ptr(hc, C.c_int), _ptr(hr), _ptr(ht)))
        tm = np.zeros(7)
        _check(lib.cieg_report_timing(rep, _ptr(tm)))
    finally:
        lib.cieg_report_destroy(rep)
    hist = [HistoryRow(int(a), int(b), float(c), float(d)) for a, b, c, d in zip(hi, hc, hr, ht)]
    return SolveReport(eigenvalues=ev, eigenvectors=trial[:, :kw.value].copy(), trial_vectors=trial,
                       history=hist, counters=OperationCounters(*[int(x) for x in cnt]),
                       converged=bool(conv.value), iterations=int(iters.value), norm_estimate=float(ne.value),
                       timing_ms=dict(zip(_TIMING_KEYS, tm.tolist())))


@dataclasses.dataclass
class LanczosOptions:
    """ci::LanczosOptions (lanczos.hpp:14-22); observer(m, basis (n x m),
    alpha, beta) at every checkpoint."""
    k_want: int = 8
    tol: float = 1e-6
    max_iter: int = 500
    observer: Optional[Callable] = None


def lanczos_checkpoint(m: int) -> bool:
    """ci::lanczos_checkpoint (lanczos.cpp:11-15)."""
    return bool(_lib.load().cieg_lanczos_checkpoint(int(m)))


def lanczos_default_start(n: int, stratum_end: int) -> np.ndarray:
    """ci::lanczos_default_start (lanczos.cpp:17-22) for a basis whose lowest
    stratum is rows [0, stratum_end)."""
    out = np.zeros(n)
    _check(_lib.load().cieg_lanczos_default_start(n, stratum_end, _ptr(out)))
    return out


def lanczos_solve(h, v0: np.ndarray, options: LanczosOptions = LanczosOptions(),
                  device: Optional[Device] = None) -> SolveReport:
    """ci::lanczos_solve (lanczos.cpp:24-136) on the GPU: K1 SpMV per step,
    two-pass full reorthogonalisation against the HBM-resident basis. `h` is
    a CsbMatrix (uploaded once) or a resident DeviceMatrix. The observer is
    called at every checkpoint as observer(m, basis, alpha, beta) with the
    (n x m) Lanczos basis, like LanczosOptions::observer."""
    v0 = np.ascontiguousarray(v0, dtype=np.float64).reshape(-1)
    if v0.shape[0] != h.dim:
        raise DimensionMismatch("lanczos: v0 dim != matrix dim")
    if not np.any(v0):
        raise ConfigError("lanczos: v0 must be nonzero")
    if options.k_want < 1:
        raise ConfigError("lanczos: k_want must be >= 1")
    lib = _lib.load()
    dm = h if isinstance(h, DeviceMatrix) else device_matrix(h, device)
    opt = _lib.LanczosOptionsC()
    lib.cieg_lanczos_options_default(C.byref(opt))
    opt.k_want, opt.tol, opt.max_iter = options.k_want, options.tol, options.max_iter
    if options.observer is not None:
        user_obs = options.observer

        def _obs(_user, m, ap, bp, basis_ptr, n):
            a = np.ctypeslib.as_array(ap, (m,)).copy()
            b = np.ctypeslib.as_array(bp, (m,)).copy()
            basis = np.ctypeslib.as_array(basis_ptr, (m, n)).T.copy()  # column-major n x m
            user_obs(m, basis, a, b)

        opt.observer = _lib.LANCZOS_OBSERVER(_obs)
    rep = C.c_void_p()
    _check(lib.cieg_lanczos_solve(dm.device.handle, dm.handle, _ptr(v0), C.byref(opt), C.byref(rep)))
    return _read_report(lib, rep, h.dim)


# ------------------------------------------- lobpcg.hpp public helpers

@dataclasses.dataclass
class SubspaceCoefficients:
    """ci::SubspaceCoefficients (lobpcg.hpp:73-80): Ritz coefficients g over
    the [X W P] basis and the segment widths."""
    g: np.ndarray
    x_width: int
    w_width: int
    p_width: int


def orthonormalize(y: np.ndarray, drop_tol: float = 1e-8, against: Optional[np.ndarray] = None,
                   device: Optional[Device] = None) -> np.ndarray:
    """ci::orthonormalize (lobpcg.cpp:89-119) on the GPU: projection against
    `against` (twice), rank-revealing column selection, CholQR twice. The
    result may be narrower than y."""
    y = _f64(y)
    if against is not None:
        against = _f64(against)
        if against.shape[0] != y.shape[0]:
            raise DimensionMismatch("orthonormalize: row counts differ")
    dev = _dev(device)
    dy = _DevArray(y)
    da = _DevArray(against) if against is not None and against.shape[1] else None
    kout = C.c_uint32()
    dev.synchronize()
    _check(_lib.load().cieg_orthonormalize(dev.handle, dy.ptr, y.shape[0], y.shape[1], float(drop_tol),
                                           da.ptr if da else None, da.t.shape[1] if da else 0, C.byref(kout)))
    k = kout.value
    return dy.host().reshape(-1)[: y.shape[0] * k].reshape(y.shape[0], k).copy()


def rayleigh_ritz(y_basis: np.ndarray, hy: np.ndarray, k_trial: int, x_width: int = -1, w_width: int = 0,
                  p_width: int = 0, device: Optional[Device] = None):
    """ci::rayleigh_ritz (lobpcg.cpp:121-145): (theta[k_trial], SubspaceCoefficients)."""
    y, hyy = _f64(y_basis), _f64(hy)
    if hyy.shape != y.shape:
        raise DimensionMismatch("rayleigh_ritz: HY shape mismatch")
    m = y.shape[1]
    if k_trial > m:
        raise DimensionMismatch("rayleigh_ritz: k_trial exceeds basis width")
    dev = _dev(device)
    dy, dh = _DevArray(y), _DevArray(hyy)
    theta = np.zeros(k_trial)
    g = np.zeros(m * k_trial)
    dev.synchronize()
    _check(_lib.load().cieg_rayleigh_ritz(dev.handle, dy.ptr, dh.ptr, y.shape[0], m, k_trial, _ptr(theta), _ptr(g)))
    return theta.tolist(), SubspaceCoefficients(g.reshape(k_trial, m).T.copy(), m if x_width < 0 else x_width,
                                                w_width, p_width)


def residual_norms(h, x: np.ndarray, theta, norm_est: Optional[float] = None,
                   device: Optional[Device] = None) -> list:
    """ci::residual_norms (lobpcg.cpp:147-169) on the GPU."""
    x = _f64(x)
    th = np.ascontiguousarray(theta, dtype=np.float64)
    if x.shape[1] != th.shape[0]:
        raise DimensionMismatch("residual_norms: theta width mismatch")
    dm = h if isinstance(h, DeviceMatrix) else device_matrix(h, device)
    dx = _DevArray(x)
    out = np.zeros(x.shape[1])
    dm.device.synchronize()
    _check(_lib.load().cieg_residual_norms(dm.device.handle, dm.handle, dx.ptr, x.shape[1], _ptr(th),
                                           float(norm_est) if norm_est is not None else 0.0, _ptr(out)))
    return out.tolist()


# ---------------------------------------------------- guess.hpp (starting blocks)

def pad_from_subspace(x1: np.ndarray, dim: int) -> np.ndarray:
    """ci::pad_from_subspace (guess.cpp:14-23)."""
    x1 = _f64(x1)
    out = np.zeros((dim, x1.shape[1]))
    _check(_lib.load().cieg_pad_from_subspace(_ptr(x1), x1.shape[0], x1.shape[1], int(dim), _ptr(out)))
    return out


@dataclasses.dataclass
class MultilevelOptions:
    """ci::MultilevelOptions (guess.hpp:47-54); the levels are given as the
    list of truncated dimensions (leading blocks of H)."""
    k_want: int = 8
    k_trial: int = 12
    tol: float = 1e-6
    max_iter: int = 500
    seed: int = 1


@dataclasses.dataclass
class LevelReport:
    """ci::LevelReport (guess.hpp:31-37); `dim` identifies the level."""
    dim: int
    iterations: int
    converged: bool
    seconds: float


@dataclasses.dataclass
class MultilevelResult:
    guess: np.ndarray
    levels: list


def multilevel_guess(h, level_dims: Sequence[int], options: MultilevelOptions = MultilevelOptions(),
                     device: Optional[Device] = None) -> MultilevelResult:
    """ci::multilevel_guess (guess.cpp:66-117) on the GPU. The truncated
    problems are the leading blocks H[0:d, 0:d] for d in level_dims
    (ascending, below dim) -- for a basis ordered by quanta stratum these are
    exactly the reference's lower-Nmax Hamiltonians. A CsbMatrix is uploaded
    with the level dimensions as mandatory panel cuts."""
    dims = np.ascontiguousarray(list(level_dims), dtype=np.uint32)
    dm = h if isinstance(h, DeviceMatrix) else DeviceMatrix(h, device, cuts=dims)
    o = _lib.MultilevelOptionsC()
    _lib.load().cieg_multilevel_options_default(C.byref(o))
    o.k_want, o.k_trial, o.tol, o.max_iter, o.seed = (options.k_want, options.k_trial, options.tol,
                                                      options.max_iter, options.seed)
    guess = np.zeros((dm.dim, options.k_trial))
    kout = C.c_uint32()
    lv = (_lib.LevelReportC * max(1, len(dims)))()
    _check(_lib.load().cieg_multilevel_guess(dm.device.handle, dm.handle, _ptr(dims, C.c_uint32), len(dims),
                                             C.byref(o), _ptr(guess), C.byref(kout), lv))
    k = kout.value
    g = guess.reshape(-1)[: dm.dim * k].reshape(dm.dim, k).copy()
    return MultilevelResult(g, [LevelReport(int(r.dim), int(r.iterations), bool(r.converged), float(r.seconds))
                                for r in list(lv)[: len(dims)]])


_BVEC = b"BVEC"


def save_vectors(x: np.ndarray, path: str) -> None:
    """ci::save_vectors (guess.cpp:119-133): "BVEC", u64 dim, u32 width,
    column-major little-endian doubles."""
    x = _f64(x)
    with open(path, "wb") as f:
        f.write(_BVEC)
        f.write(struct.pack("<QI", x.shape[0], x.shape[1]))
        f.write(np.asfortranarray(x).astype("<f8").tobytes(order="F"))


def load_guess_file(path: str, dim: int, k: int, device: Optional[Device] = None) -> np.ndarray:
    """ci::load_guess_file (guess.cpp:135-163): first k columns, orthonormalized."""
    try:
        f = open(path, "rb")
    except OSError:
        raise FormatError("cannot open: " + path)
    with f:
        magic = f.read(4)
        if magic != _BVEC:
            raise FormatError("bad magic; not a BVEC file: " + path)
        hdr = f.read(12)
        if len(hdr) < 12:
            raise FormatError("truncated BVEC header: " + path)
        fdim, width = struct.unpack("<QI", hdr)
        if fdim != dim:
            raise DimensionMismatch(f"vector file dimension {fdim} != basis dimension {dim}")
        if width < k:
            raise DimensionMismatch(f"vector file holds {width} columns, need {k}")
        raw = f.read(8 * dim * k)
        if len(raw) < 8 * dim * k:
            raise FormatError("truncated BVEC payload: " + path)
    x = np.frombuffer(raw, dtype="<f8").reshape(k, dim).T.astype(np.float64)
    return orthonormalize(x, device=device)


def write_history_csv(report: SolveReport, os: io.TextIOBase) -> None:
    """ci::write_history_csv (lobpcg.cpp:389-397): ``iter,col,relres,theta`` %.17g."""
    os.write("iter,col,relres,theta\n")
    for r in report.history:
        os.write("%d,%d,%.17g,%.17g\n" % (r.iteration, r.column, r.relres, r.theta))
