"""CPU: the C-ABI library loads, exports every symbol include/*.h declares,
and its host-side helpers (random.hpp / sketch.hpp mirrors) agree with the
oracle. No device compute here."""
import ctypes
import glob
import os
import re

import numpy as np
import pytest

from oracle import sorsvd_oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_functions():
    names = set()
    for h in glob.glob(os.path.join(ROOT, "include", "*.h")):
        src = open(h).read()
        src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
        for mt in re.finditer(r"^\s*[A-Za-z_][\w\s\*]*?\b(sorsvd_\w+)\s*\(", src, flags=re.M):
            names.add(mt.group(1))
    return names


@pytest.fixture(scope="module")
def lib():
    from paper_1804_00462_b200 import _capi
    if not os.path.exists(_capi.LIB_PATH):
        from paper_1804_00462_b200 import build as B
        B.build()
    return _capi.lib()


def test_exports_every_declared_symbol(lib):
    names = _declared_functions()
    assert len(names) >= 19, names
    for n in names:
        assert hasattr(lib, n), n
    from paper_1804_00462_b200 import _capi
    assert names == {s[0] for s in _capi.SIGNATURES}


def test_library_is_sm100a():
    from paper_1804_00462_b200 import _capi
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _capi.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_gaussian_matrix_matches_reference_stream(lib):
    import paper_1804_00462_b200 as P
    for (r, c, s) in [(7, 5, 123), (3, 3, 0), (1, 9, 2**64 - 1), (301, 77, 42)]:
        for nt in (1, 3, 8):
            assert np.array_equal(P.gaussian_matrix(r, c, s, nthreads=nt), O.gaussian_matrix(r, c, s))
    big = P.gaussian_matrix(1000, 333, 5)  # multi-threaded path, odd split points
    assert np.array_equal(big, O.gaussian_matrix(1000, 333, 5))
    # thread counts whose even-rounded chunk undershoots the total: the last chunk must run
    # to the end (1100 x 64 on 3 threads left the final pair unwritten)
    for (r, c, nt) in [(1100, 64, 3), (1100, 64, 0), (1025, 64, 7), (800, 100, 5), (70001, 1, 3), (4000, 100, 16)]:
        assert np.array_equal(P.gaussian_matrix(r, c, 9, nthreads=nt), O.gaussian_matrix(r, c, 9)), (r, c, nt)


def test_sub_seed_and_flops(lib):
    import paper_1804_00462_b200 as P
    for s in (0, 1, 42, 2**63):
        for t in range(4):
            assert P.sub_seed(s, t) == O.sub_seed(s, t)
    assert P.flop_estimate(1000, 1000, 38, 20, 0, P.FlopVariant.sor_3pass) == 239813744
    for v in range(4):
        assert P.flop_estimate(4000, 4000, 100, 100, 1, v) == O.flop_estimate(4000, 4000, 100, 100, 1, v)
    with pytest.raises(P.ParameterError):
        P.flop_estimate(-1, 4, 2, 1, 0, 0)


def test_validate_sketch_codes(lib):
    import paper_1804_00462_b200 as P
    for args in [(1, 5, 1, 1, 0), (5, 5, 0, 1, 0), (5, 5, 3, 2, 0), (5, 5, 2, 5, 0), (5, 5, 1, 2, -1)]:
        with pytest.raises(P.ParameterError):
            P.validate_sketch(*args)
    P.validate_sketch(5, 5, 2, 4, 0)


def test_context_without_gpu_fails_loudly(lib):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_1804_00462_b200 as P
    with pytest.raises(P.CudaError):
        P.Context(0)
    with pytest.raises(P.CudaError):
        P.sor_svd_power(np.ones((10, 8)), 2, P.SketchConfig(3, 0, 1))


def test_cpp_dropin_header_compiles_against_reference():
    """include/sorsvd_b200.hpp is a drop-in on the reference's own types; the
    test binary (tests/cpp) is built against the unmodified reference headers."""
    path = os.path.join(ROOT, "tests", "cpp", "_build", "test_dropin")
    if not os.path.isdir("/root/reference/proj/include") and not os.path.exists(path):
        pytest.skip("reference headers absent and test binary not prebuilt")
    if os.path.isdir("/root/reference/proj/include"):
        import subprocess
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "tests", "cpp")], check=True)
    assert os.path.exists(path)


def test_sord_header_cpu(tmp_path):
    # SORD files: header parsing through the C ABI needs no GPU
    import paper_1804_00462_b200 as P
    a = O.gaussian_matrix(37, 11, 3)
    p = str(tmp_path / "a.sord")
    O.write_sord(p, a)
    assert P.sord_header(p) == (37, 11)
    np.testing.assert_array_equal(O.read_sord(p), a)
    bad = tmp_path / "bad.sord"
    bad.write_bytes(b"NOPE" + open(p, "rb").read()[4:])
    with pytest.raises(P.ParameterError):
        P.sord_header(str(bad))
    short = tmp_path / "short.sord"
    short.write_bytes(open(p, "rb").read()[:-8])
    with pytest.raises(P.ShapeError):
        P.sord_header(str(short))


def test_gaussian_rows_is_a_slice_of_the_full_draw():
    """sorsvd_gaussian_rows (counter-based stream, random.hpp:27-55): any row block equals the same rows of
    gaussian_matrix, for odd / even offsets and every thread count (the Box-Muller pairs straddle rows)."""
    import ctypes
    import paper_1804_00462_b200 as P
    from oracle import sorsvd_oracle as O
    lib = P._capi.lib()
    for cols, total, seed in [(7, 41, 5), (20, 30000, 6), (1, 9, 7), (33, 5001, 8)]:
        full = O.gaussian_matrix(total, cols, seed)
        for row0, rows in [(0, total), (1, total - 1), (3, 17), (total - 5, 5), (total // 2 + 1, total // 3)]:
            rows = min(rows, total - row0)
            for nt in (1, 3, 16):
                out = np.full((rows, cols), np.nan)
                assert lib.sorsvd_gaussian_rows(cols, row0, rows, seed, out.ctypes.data_as(P._capi.c_dp), nt) == 0
                assert np.array_equal(out, full[row0:row0 + rows]), (cols, total, row0, rows, nt)


def test_default_build_keeps_34_digit_products():
    """The shipped library is the 34-product cut of the Ozaki passes (pairs t + u >= 5, error below FP64's own
    rounding); the 28-product cut is a build option (SORSVD_OZ_LEVEL0=6) and must not ship by accident."""
    from paper_1804_00462_b200 import _capi
    assert _capi.lib().sorsvd_ozaki_products() == 34
