"""CPU: the device ports of glibc 2.39 logf/sinf/cosf (csrc/glibc_math.cuh,
host build) equal this host's libm on every one of the 2^32 float inputs,
for both glibc ifunc variants (FMA build vs generic build selected with
GLIBC_TUNABLES=glibc.cpu.hwcaps=-AVX2,-FMA). The device compiles the same
source with explicit _rn intrinsics, so the device results follow; the GPU
tests confirm them on the sampler's whole uniform domain and in rollouts."""
import os
import subprocess

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "native", "check_glibc_math.cpp")


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


def test_fma_variant_matches_default_libm_all_floats(checker):
    rc, out, err = run(checker, fma=True)
    assert rc == 0, out + err


def test_generic_variant_matches_generic_libm_all_floats(checker):
    rc, out, err = run(checker, fma=False, env={"GLIBC_TUNABLES": "glibc.cpu.hwcaps=-AVX2,-FMA"})
    assert rc == 0, out + err


def test_variants_really_differ(checker):
    """The two variants differ on some inputs, so selecting the right one matters."""
    rc, out, err = run(checker, fma=False, stride=1)
    assert rc == 1 and "sinf mismatch" in err
