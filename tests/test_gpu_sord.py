"""GPU: SORD matrix files streamed into and out of HBM through
pinned double buffers: bit-exact against the numpy restatement of the format,
FP32 rounding on the device, multi-chunk streaming, and a decomposition of a
loaded matrix."""
import numpy as np
import pytest

from oracle import sorsvd_oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1804_00462_b200 as P
    return P


@pytest.mark.parametrize("chunk_mb", [None, "1"])
def test_sord_load_save_roundtrip(P, tmp_path, monkeypatch, chunk_mb):
    import torch
    ctx = P.Context(0)
    if chunk_mb:
        ctx.set_option(P.Context.OPT_SORD_CHUNK_MB, int(chunk_mb))  # many chunks: both staging buffers cycle
    a = O.gaussian_matrix(1531, 389, 21)
    p = str(tmp_path / "a.sord")
    O.write_sord(p, a)
    d = P.load_sord(p, ctx=ctx)
    assert d.dtype == torch.float64 and tuple(d.shape) == a.shape
    np.testing.assert_array_equal(d.cpu().numpy(), a)
    f = P.load_sord(p, dtype=torch.float32, ctx=ctx)
    np.testing.assert_array_equal(f.cpu().numpy(), a.astype(np.float32))
    q = str(tmp_path / "b.sord")
    P.save_sord(q, d * 2.0, ctx=ctx)
    np.testing.assert_array_equal(O.read_sord(q), 2.0 * a)
    assert open(q, "rb").read() == open(p, "rb").read()[:24] + (2.0 * a).astype("<f8").tobytes()


def test_sord_decompose_loaded_matrix(P, tmp_path):
    a = O.gen_lowrank_decay(900, 600, 30, lambda j: 2.0 ** (-j / 3), 1e-6, 9)
    p = str(tmp_path / "c.sord")
    O.write_sord(p, a)
    d = P.load_sord(p)
    f = P.sor_svd_power(d, 20, P.SketchConfig(24, 1, 5))
    g = P.sor_svd_power(a, 20, P.SketchConfig(24, 1, 5))
    np.testing.assert_array_equal(f.sigma.cpu().numpy(), g.sigma)


def test_sord_errors(P, tmp_path):
    p = tmp_path / "x.sord"
    p.write_bytes(b"SORD" + np.array([2], "<u4").tobytes() + np.array([2, 2], "<u8").tobytes() + bytes(32))
    with pytest.raises(P.ParameterError):
        P.load_sord(str(p))
    with pytest.raises(P.ParameterError):
        P.load_sord(str(tmp_path / "missing.sord"))
