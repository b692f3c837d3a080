import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the sm_100a kernels)")
    config.addinivalue_line("markers", "slow: larger parity cases")


@pytest.fixture(scope="session")
def golden():
    with open(os.path.join(ROOT, "tests", "golden", "golden.json")) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def port():
    from oracle.pyoracle import Port
    return Port()


@pytest.fixture(scope="session")
def ref():
    """The compiled reference (oracle/_ref). Built here by __graft_entry__.build();
    the prebuilt .so travels to the GPU box with the snapshot."""
    from oracle.pyoracle import REF_SO, Ref
    if not os.path.exists(REF_SO):
        pytest.skip("oracle/_ref not built (needs /root/reference at build time)")
    return Ref()


@pytest.fixture(scope="session")
def ctx():
    """A B200 context. On a GPU box a missing library or device is a failure,
    never a silent skip."""
    import paper_2506_22668_b200 as sf
    c = sf.Context(0)
    yield c
    c.close()


def hex_to_u64(xs):
    return np.array([int(x, 16) for x in xs], dtype=np.uint64)


def toy_graph_arrays(dim=2):
    """test_helpers.hpp:73-91 toy graph."""
    edges = np.array([[0, 1], [1, 2], [2, 3], [3, 4], [4, 0], [1, 3], [1, 5]], np.uint64)
    feats = (0.1 * (np.arange(6 * dim, dtype=np.float32) + 1)).astype(np.float32).reshape(6, dim)
    return edges, feats
