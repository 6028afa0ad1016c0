import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def golden():
    import numpy as np
    import json
    d = os.path.join(ROOT, "tests", "golden")
    g = dict(np.load(os.path.join(d, "golden_ref.npz")))
    with open(os.path.join(d, "golden_meta.json")) as fh:
        meta = json.load(fh)
    return g, meta


@pytest.fixture(scope="session")
def ref_available():
    from oracle import sorsvd_oracle as O
    return os.path.exists(O.REF_LIB_PATH)
