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
