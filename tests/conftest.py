import gzip
import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the sm_100a kernels)")
    config.addinivalue_line("markers", "slow: long CPU test")


def _build_once():
    from paper_2301_03598_b200 import build as b

    b.build()
    import oracle

    if not os.path.exists(oracle.PORT_SO):
        oracle.build(with_ref=False)
    if not os.path.exists(oracle.REF_SO) and os.path.isdir(oracle.REF_SRC):
        oracle.build(with_ref=True)


_build_once()


@pytest.fixture(scope="session")
def sk():
    import paper_2301_03598_b200 as m

    m.lib()
    return m


@pytest.fixture(scope="session")
def port():
    import oracle

    return oracle.Oracle("port")


@pytest.fixture(scope="session")
def ref():
    import oracle

    if not oracle.have_reference():
        pytest.skip("reference build (oracle/_ref) not present")
    return oracle.Oracle("reference")


@pytest.fixture(scope="session")
def golden_schedules():
    with gzip.open(os.path.join(GOLDEN, "schedules.json.gz"), "rt") as f:
        return json.load(f)["entries"]


@pytest.fixture(scope="session")
def golden_arrays():
    return dict(np.load(os.path.join(GOLDEN, "executor.npz")))


@pytest.fixture(scope="session")
def torch_cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch
