import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) CUDA device")
    config.addinivalue_line("markers", "slow: full BASELINE-scale case (minutes)")


def pytest_collection_modifyitems(config, items):
    try:
        import torch

        has_gpu = torch.cuda.is_available()
    except Exception:
        has_gpu = False
    if has_gpu:
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)


@pytest.fixture(scope="session")
def golden():
    cache = {}

    def load(name):
        if name not in cache:
            cache[name] = dict(np.load(os.path.join(GOLDEN, name + ".npz")))
        return cache[name]

    return load


def gen_from(params):
    from paper_1609_01689_b200 import ci

    n, s, t, p, q, seed, prec, beta = params
    return ci.generate_sector_matrix(int(n), int(s), int(t), float(p), float(q), int(seed), int(prec), int(beta))


@pytest.fixture(scope="session")
def ref_lib():
    from oracle import ref

    if not ref.available():
        pytest.skip("oracle/_ref not built (needs /root/reference at build time)")
    return ref


def multilevel_operator(g):
    """The operator multilevel_guess sees in tests/golden/multilevel.npz: the
    Nmax-4 4He Hamiltonian (the leading block of the Nmax-6 one) followed by
    a diagonal filler up to the Nmax-6 dimension. The level solves read only
    the leading block and the guess is zero-padded below it, so the filler
    never enters the result (make_golden.py: make_multilevel)."""
    from paper_1609_01689_b200 import ci

    full = int(g["full_dim"])
    bb = g["sub_block_boundaries"].astype(np.uint32)
    nb = len(bb) - 1
    eo = g["sub_entry_offsets"].astype(np.uint64)
    sub = int(bb[-1])
    fill = full - sub
    rows = np.concatenate([g["sub_rows"], np.arange(fill, dtype=np.uint16)])
    cols = np.concatenate([g["sub_cols"], np.arange(fill, dtype=np.uint16)])
    vals = np.concatenate([g["sub_values"], np.full(fill, 100.0, dtype=g["sub_values"].dtype)])
    # block row nb: blocks (nb, 0..nb-1) empty, (nb, nb) the filler diagonal
    eo_new = np.concatenate([eo, np.full(nb, eo[-1], dtype=np.uint64), [eo[-1] + fill]]).astype(np.uint64)
    groups = np.concatenate([g["sub_groups"].astype(np.uint32), [full]]).astype(np.uint32)
    return ci.CsbMatrix(dim=full, precision=int(g["sub_precision"]), block_boundaries=np.append(bb, np.uint32(full)),
                        entry_offsets=eo_new, rows=rows, cols=cols, values=vals, groups=groups)


def single_pass_shards(h, world, m, x):
    """Every shard of a world-`world` partition in this process: the
    single-pass kernel (cieg_spmm_partial) per shard, then the reverse
    exchange done on the host exactly as dist.partial_reduce orders it."""
    import ctypes as C

    import torch

    from paper_1609_01689_b200 import _lib, ci
    from paper_1609_01689_b200 import dist as D

    dev = ci.Device.default()
    rb, hl, hh = D.row_partition(h, world)
    xs = torch.from_numpy(x).cuda()
    ys, halos = [], []
    for r in range(world):
        sm = D.ShardedMatrix(h, r, world, dev, plan=(rb, hl, hh))
        plo, phi = D.partial_rows(sm.handle)
        assert phi == sm.row_lo and plo <= phi
        y = torch.empty((sm.local_rows, m), dtype=torch.float64, device="cuda")
        yh = torch.full((max(phi - plo, 1), m), float("nan"), dtype=torch.float64, device="cuda")
        torch.cuda.synchronize()  # the fill runs on torch's stream, the library on its own
        ci._check(_lib.load().cieg_spmm_partial(dev.handle, sm.handle, C.c_void_p(xs.data_ptr()),
                                                C.c_void_p(y.data_ptr()), m, C.c_void_p(yh.data_ptr())))
        dev.synchronize()
        ys.append(y.cpu().numpy())
        halos.append((plo, yh.cpu().numpy()[: phi - plo]))
    out = np.zeros((h.dim, m))
    for r in range(world):
        lo, hi = int(rb[r]), int(rb[r + 1])
        yr = ys[r].copy()
        for t in range(r + 1, world):
            plo, yh = halos[t]
            a, b = max(lo, plo), min(hi, int(rb[t]))
            if b > a:
                yr[a - lo:b - lo] += yh[a - plo:b - plo]
        out[lo:hi] = yr
    return out
