"""Device-side exhaustive check of the glibc 2.39 ports (csrc/glibc_math.cuh)
as the DEVICE compiles them (_rn intrinsics, __fma_rn in the FMA variant):
every one of the 2^32 float inputs of logf, sinf, cosf and the fused sincosf
is fingerprinted on the GPU (smpc_libm_hash) and compared with the same
fingerprint of the host libm (tests/golden/libm_hash.json, which
tests/test_glibc_math.py pins to this image's libm). Any single differing
output changes its bucket's sum, so equality means bitwise equality on all
inputs up to a 2^-64 collision chance per bucket."""
import ctypes
import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

HASHES = os.path.join(os.path.dirname(__file__), "golden", "libm_hash.json")
ROWS = ["logf", "sinf", "cosf", "sincosf.sin", "sincosf.cos"]


@pytest.fixture(scope="module")
def lib():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2409_07563_b200 import _lib
    return _lib.load()


@pytest.mark.parametrize("variant", ["fma", "generic"])
def test_device_libm_ports_exhaustive(lib, variant):
    host = np.array(json.load(open(HASHES))[variant], np.uint64).reshape(3, 256)
    out = np.zeros(5 * 256, np.uint64)
    rc = lib.smpc_libm_hash(0, 1 if variant == "fma" else 0, out.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)))
    assert rc == 0
    out = out.reshape(5, 256)
    want = host[[0, 1, 2, 1, 2]]
    for r, name in enumerate(ROWS):
        bad = np.nonzero(out[r] != want[r])[0]
        assert bad.size == 0, f"{name}: input top bytes {[hex(b) for b in bad[:8]]} differ from the host libm"


@pytest.mark.parametrize("variant", ["fma", "generic"])
def test_fast_math_matches_exact(lib, variant):
    """The unchecked rollout loop's branch-free math: sincosf (all 2^32
    floats, |x| < 120 equal to the exact port, NaN beyond -> exact replay),
    wrap_angle (all 2^32), float division (2^32 random pairs) and the
    importance term's double division with a precomputed divisor reciprocal
    (2^31 random pairs) equal the exact device ops wherever they do not
    return NaN."""
    out = np.zeros(16, np.uint64)
    rc = lib.smpc_fast_math_check(0, 1 if variant == "fma" else 0, out.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)))
    assert rc == 0
    print("fast-path pairs: div", out[4], "ddiv", out[5], "first mismatches", [hex(int(v)) for v in out[6:]])
    assert out[0] == 0 and out[1] == 0 and out[2] == 0 and out[3] == 0, out
    assert out[4] > (1 << 29) and out[5] > (1 << 28)
