"""CPU: the device ports of glibc 2.39 logf/sinf/cosf (csrc/glibc_math.cuh,
host build) equal this host's libm on every one of the 2^32 float inputs,
for both glibc ifunc variants (FMA build vs generic build selected with
GLIBC_TUNABLES=glibc.cpu.hwcaps=-AVX2,-FMA). The device compiles the same
source with explicit _rn intrinsics, so the device results follow; the GPU
tests confirm them on the sampler's whole uniform domain and in rollouts."""
import json
import os
import subprocess

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "native", "check_glibc_math.cpp")
HASHES = os.path.join(HERE, "golden", "libm_hash.json")


@pytest.fixture(scope="module")
def checker(tmp_path_factory):
    exe = str(tmp_path_factory.mktemp("gm") / "check_glibc_math")
    subprocess.run(["g++", "-O2", "-std=c++17", "-ffp-contract=off", "-fno-builtin", "-pthread", SRC, "-o", exe],
                   check=True)
    return exe


def run(exe, fma, env=None, stride=1):
    threads = str(max(1, os.cpu_count() or 1))
    r = subprocess.run([exe, str(stride), threads, "1" if fma else "0"], capture_output=True, text=True,
                       env={**os.environ, **(env or {})}, timeout=600)
    return r.returncode, r.stdout.strip(), r.stderr


def _hash(tmp_path, name):
    return [int(v) for v in open(tmp_path / name).read().split()]


def test_fma_variant_matches_default_libm_all_floats(checker, tmp_path):
    rc, out, err = run(checker, fma=True, env={"SMPC_LIBM_HASH_OUT": str(tmp_path / "fma.txt")})
    assert rc == 0, out + err
    # the committed fingerprint the device-side exhaustive check compares with
    # (tests/test_gpu_libm.py) is this host libm's
    assert _hash(tmp_path, "fma.txt") == json.load(open(HASHES))["fma"]


def test_generic_variant_matches_generic_libm_all_floats(checker, tmp_path):
    rc, out, err = run(checker, fma=False, env={"GLIBC_TUNABLES": "glibc.cpu.hwcaps=-AVX2,-FMA",
                                                "SMPC_LIBM_HASH_OUT": str(tmp_path / "generic.txt")})
    assert rc == 0, out + err
    assert _hash(tmp_path, "generic.txt") == json.load(open(HASHES))["generic"]


def test_variants_really_differ(checker):
    """The two variants differ on some inputs, so selecting the right one matters."""
    rc, out, err = run(checker, fma=False, stride=1)
    assert rc == 1 and "sinf mismatch" in err
