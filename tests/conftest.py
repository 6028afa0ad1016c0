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


@pytest.fixture(scope="session")
def parity_log():
    """Append one JSON record per call to $SORSVD_PARITY_OUT/parity.jsonl (the
    per-sigma error vectors committed under profiles/); no-op when unset."""
    import json
    out = os.environ.get("SORSVD_PARITY_OUT")

    def rec(name, **data):
        if not out:
            return
        os.makedirs(out, exist_ok=True)
        clean = {}
        for k, v in data.items():
            if hasattr(v, "tolist"):
                v = v.tolist()
            clean[k] = v
        with open(os.path.join(out, "parity.jsonl"), "a") as fh:
            fh.write(json.dumps({"test": name, **clean}) + "\n")
    return rec
