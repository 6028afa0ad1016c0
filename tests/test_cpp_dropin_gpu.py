"""GPU: run the C++ drop-in test (reference types in, reference exceptions out)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu


def test_cpp_dropin_runs_on_gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    exe = os.path.join(ROOT, "tests", "cpp", "_build", "test_dropin")
    if not os.path.exists(exe):
        pytest.skip("tests/cpp/_build/test_dropin not built (needs /root/reference at build time)")
    out = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    print(out.stdout)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "OK" in out.stdout
