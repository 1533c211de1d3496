import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) device")
    config.addinivalue_line("markers", "slow: benchmark-shape host work (seconds)")


def _has_gpu() -> bool:
    try:
        import ctypes
        cudart = ctypes.CDLL("libcudart.so.12")
        n = ctypes.c_int(0)
        return cudart.cudaGetDeviceCount(ctypes.byref(n)) == 0 and n.value > 0
    except OSError:
        return False


HAS_GPU = _has_gpu()


def pytest_collection_modifyitems(config, items):
    if HAS_GPU:
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


@pytest.fixture(scope="session")
def small_graph():
    import paper_2602_21597_b200 as m
    return m.Graph.synthetic("small", 1)


@pytest.fixture(scope="session")
def small_oracle_graph(small_graph):
    import oracle as O
    info = small_graph.info()
    return O.OracleGraph(info["n_entities"], info["n_relations"], small_graph.triples(0),
                         small_graph.triples(1), small_graph.triples(2))
