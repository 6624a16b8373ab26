"""CPU: the user-model plugin API (include/smpc_b200_plugin.cuh) — an
out-of-tree model + cost (tests/native/user_model.cu) compiles into its own
shared object against the public header only, and its launcher table carries
the library's ABI version, argument-block size and the functors' dims.
(The GPU half, tests/test_gpu_plugin.py, runs controllers on it.)"""
import ctypes
import os
import subprocess

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
SRC = os.path.join(HERE, "native", "user_model.cu")
LIB = os.path.join(HERE, "native", "libuser_model.so")


def build_user_model(force: bool = False) -> str:
    """nvcc the out-of-tree plugin (sm_100a) next to its source."""
    import glob
    deps = [SRC] + glob.glob(os.path.join(ROOT, "include", "*")) + glob.glob(
        os.path.join(ROOT, "paper_2409_07563_b200", "csrc", "*.cuh")) + [
        os.path.join(ROOT, "paper_2409_07563_b200", "csrc", "launch.h")]
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < max(os.path.getmtime(d) for d in deps):
        subprocess.run(["nvcc", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo",
                        "-fmad=false", "-Xcompiler", "-fPIC", "-shared", "-I", os.path.join(ROOT, "include"), "-I",
                        os.path.join(ROOT, "paper_2409_07563_b200", "csrc"), SRC, "-o", LIB], check=True)
    return LIB


def load_user_model():
    from paper_2409_07563_b200._lib import SmpcModelOps
    lib = ctypes.CDLL(build_user_model())
    lib.user_di_ops.restype = SmpcModelOps
    lib.user_di_ops.argtypes = [ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double)]
    lib.spring_ops.restype = SmpcModelOps
    lib.spring_ops.argtypes = [ctypes.c_float, ctypes.c_float, ctypes.c_float]
    return lib


def test_plugin_table_carries_abi_and_dims():
    if subprocess.run(["which", "nvcc"], capture_output=True).returncode != 0 and not os.path.exists(LIB):
        pytest.skip("nvcc not available")
    from paper_2409_07563_b200 import scenario as S
    lib = load_user_model()
    t = (ctypes.c_double * 4)(1.0, -1.0, 0.0, 0.0)
    w = (ctypes.c_double * 4)(1.0, 1.0, 0.1, 0.1)
    ops = lib.user_di_ops(t, w)
    assert ops.abi_version == S.ABI_VERSION
    assert (ops.n_x, ops.n_u, ops.n_y) == (4, 2, 4)
    assert ops.name == b"user_double_integrator"
    assert ops.user_bytes >= 64 and all([ops.rollout, ops.update, ops.combine, ops.generate, ops.plant_step])
    sp = lib.spring_ops(2.0, 0.5, 3.0)
    assert (sp.n_x, sp.n_u, sp.n_y) == (2, 1, 2) and sp.name == b"spring_mass"
    assert sp.args_bytes == ops.args_bytes > 0
