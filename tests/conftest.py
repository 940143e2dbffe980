import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU")
    config.addinivalue_line("markers", "slow: long-running")
    # BIFATTN_TEST_LIB=<path>: run the suite against a variant build of the same
    # sources (e.g. the -DBIFATTN_CHECKS device-bounds-check build)
    lib = os.environ.get("BIFATTN_TEST_LIB")
    if lib:
        import paper_2403_08845_b200 as ba

        ba.load_library(lib)


def pytest_collection_modifyitems(config, items):
    import torch

    if torch.cuda.is_available():
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)
