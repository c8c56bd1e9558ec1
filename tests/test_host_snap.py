"""Host-side snapping of fp32 inputs (runtime/host_snap.cpp, fi_host_snap_f32):
fi_plan_run_host converts input panels on host cores before they cross PCIe,
so its result must equal the device conversion (runtime/convert.cu) bit for
bit. Here (no GPU) it is checked against a numpy restatement of that
conversion: f16 = IEEE RNE after the reference's saturation of finite
|x| >= 2^16 to +-65504 (anvil::round_to_f16, matrix.hpp:67-80), bf16 = IEEE
RNE, NaN -> 0x7FFF. tests/test_gpu_host_snap.py compares with the device."""
import numpy as np
import pytest

SPECIALS = np.array([0.0, -0.0, 1.0, -1.0, 0.1, 1e-8, -1e-8, 5.9604645e-08, 2.9802322e-08, 2.9802326e-08,
                     6.1035156e-05, 6.097555e-05, 65504.0, -65504.0, 65519.99, 65520.0, -65520.0, 65535.99,
                     65536.0, -65536.0, 1e10, -1e30, 3.4028235e38, -3.4028235e38, np.inf, -np.inf, np.nan,
                     1.0009765625, 1.00048828125, 1.001464843750, 3.3895314e38, 1.1754944e-38, 1e-45,
                     -2.5e-41, 255.5, 256.5, 257.5], dtype=np.float32)


def ref_f16(x):
    x = np.asarray(x, dtype=np.float32)
    a = np.abs(x)
    with np.errstate(invalid="ignore", over="ignore"):
        sat = (a >= 65536.0) & (a <= np.finfo(np.float32).max)
        y = np.where(sat, np.copysign(np.float32(65504.0), x), x).astype(np.float16).view(np.uint16)
    return np.where(np.isnan(x), np.uint16(0x7FFF), y).astype(np.uint16)


def ref_bf16(x):
    u = np.asarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    r = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16).astype(np.uint16)
    return np.where(np.isnan(np.asarray(x, dtype=np.float32)), np.uint16(0x7FFF), r).astype(np.uint16)


def payload_nans():
    return np.array([0x7FC00000, 0xFFC00000, 0x7F800001, 0xFF800001, 0x7FBFFFFF, 0x7FFFFFFF],
                    dtype=np.uint32).view(np.float32)


@pytest.mark.parametrize("elem,ref", [("f16", ref_f16), ("bf16", ref_bf16)])
def test_specials(fi, elem, ref):
    x = np.concatenate([SPECIALS, -SPECIALS, payload_nans()])
    got = fi.host_snap(x, elem)
    np.testing.assert_array_equal(got, ref(x))


@pytest.mark.parametrize("elem,ref", [("f16", ref_f16), ("bf16", ref_bf16)])
@pytest.mark.parametrize("n", [1, 15, 16, 17, 1000, 4099])
def test_random_bits_and_lengths(fi, elem, ref, n):
    """Arbitrary bit patterns (every exponent, subnormals, NaN payloads) and
    lengths around the 16-element vector step; offsets exercise the
    alignment head of the streaming stores."""
    rng = np.random.default_rng(n)
    x = rng.integers(0, 2**32, size=n + 7, dtype=np.uint64).astype(np.uint32).view(np.float32)
    for off in (0, 1, 3, 7):
        np.testing.assert_array_equal(fi.host_snap(x[off:off + n], elem), ref(x[off:off + n]))


def test_grid_values_round_trip(fi, oracle):
    """Values already on the f16 grid (what the reference's fills produce after
    round_to_f16) are unchanged; the oracle's round_elem agrees."""
    a = oracle.fill(64, 64, 3, False)
    r = oracle.round_elem(a, "f16")
    np.testing.assert_array_equal(fi.host_snap(r, "f16").view(np.float16).astype(np.float32), r)
    np.testing.assert_array_equal(fi.host_snap(a, "f16").view(np.float16).astype(np.float32), r)


def test_avx2_path_in_a_subprocess(fi):
    """The AVX-512 fast path is the default where the CPU has it; the AVX2 path
    (FI_HOST_SNAP_AVX2=1, read once per process) must agree bit for bit."""
    import os
    import subprocess
    import sys
    code = ("import sys; sys.path.insert(0, 'tests'); sys.path.insert(0, '.');"
            "import numpy as np, paper_2003_06324_b200 as fi, test_host_snap as t;"
            "rng = np.random.default_rng(5);"
            "x = np.concatenate([t.SPECIALS, -t.SPECIALS, t.payload_nans(),"
            " rng.integers(0, 2**32, size=100003, dtype=np.uint64).astype(np.uint32).view(np.float32)]);"
            "assert (fi.host_snap(x, 'f16') == t.ref_f16(x)).all();"
            "assert (fi.host_snap(x, 'bf16') == t.ref_bf16(x)).all(); print('ok')")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, "-c", code], cwd=root, capture_output=True, text=True,
                         env={**os.environ, "FI_HOST_SNAP_AVX2": "1"}, timeout=300)
    assert out.returncode == 0 and "ok" in out.stdout, out.stderr
