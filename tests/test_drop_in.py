"""Drop-in: the reference's own closed loop (smpc::Plant::run_control_loop,
plant.cpp:133-181) driven by smpc::gpu::GpuMppiController (the header-only
adapter paper_2409_07563_b200/cpp/smpc_gpu_controller.hpp, deriving from the
reference's smpc::Controller) and by the reference's MppiController, from
one scenario JSON in the reference's schema.

The test binary links the unmodified reference library (oracle/_ref) and the
C-ABI library; it is built here by __graft_entry__.build() (the reference
headers exist only in this container) and travels to the GPU box prebuilt.
"""
import json
import os
import subprocess

import numpy as np
import pytest

from paper_2409_07563_b200 import scenario as S

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "build", "drop_in_plant")
BIN_PLUGIN = os.path.join(ROOT, "build", "drop_in_plugin")
PLUGIN_LIB = os.path.join(ROOT, "tests", "native", "libuser_model.so")


def build_drop_in():
    """Compile tests/native/drop_in_plant.cpp (needs /root/reference headers)."""
    ref_inc = "/root/reference/proj/core/include"
    if not os.path.isdir(ref_inc):
        return False
    nj = "/opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty"
    os.makedirs(os.path.dirname(BIN), exist_ok=True)
    cmd = ["g++", "-std=c++20", "-O2", "-I", os.path.join(ROOT, "oracle", "shim"), "-I", nj, "-I", ref_inc,
           "-I", os.path.join(ROOT, "include"), os.path.join(ROOT, "tests", "native", "drop_in_plant.cpp"),
           "-o", BIN, "-L", os.path.join(ROOT, "oracle", "_ref"), "-lsmpc_ref",
           "-L", os.path.join(ROOT, "paper_2409_07563_b200"), "-lsmpc_b200",
           "-Wl,-rpath,$ORIGIN/../oracle/_ref:$ORIGIN/../paper_2409_07563_b200", "-pthread"]
    subprocess.run(cmd, check=True)
    # a user model on both sides: reference subclasses + the out-of-tree device plugin
    cmd = [c if c != os.path.join(ROOT, "tests", "native", "drop_in_plant.cpp")
           else os.path.join(ROOT, "tests", "native", "drop_in_plugin.cpp") for c in cmd]
    cmd[cmd.index("-o") + 1] = BIN_PLUGIN
    subprocess.run(cmd + ["-ffp-contract=off", "-ldl"], check=True)
    return True


def test_adapter_compiles_against_reference_headers(oracle_built):
    if not os.path.isdir("/root/reference/proj/core/include"):
        pytest.skip("reference headers not present (GPU box)")
    assert build_drop_in() and os.path.exists(BIN)


def _scenario_files(tmp_path):
    out = {}
    cp = S.cartpole_scenario(num_samples=2048, horizon=100, seed=1)
    cp.initial_state = {"THETA": 0.1}
    out["cartpole"] = cp
    di = S.di_swarm_scenario(num_samples=4096, horizon=60, seed=7)
    out["di"] = di
    nav = S.diff_drive_nav_scenario(num_samples=1000, horizon=56, seed=42)
    path = str(tmp_path / "nav.costmap")
    nav.costmap.save(path)
    nav.cost_params = dict(nav.cost_params, costmap_path=path)
    out["nav"] = nav
    files = {}
    for k, sc in out.items():
        p = tmp_path / f"{k}.json"
        p.write_text(sc.to_json())
        files[k] = str(p)
    return files


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["cartpole", "di", "nav"])
def test_reference_plant_drives_gpu_controller(tmp_path, name):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    if not os.path.exists(BIN):
        pytest.skip("drop-in binary not built (needs /root/reference at build time)")
    f = _scenario_files(tmp_path)[name]
    r = subprocess.run([BIN, f, "0.3"], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr
    lines = [json.loads(ln) for ln in r.stdout.splitlines() if ln.startswith("{")]
    ref, gpu = lines[0], lines[1]
    assert ref["impl"] == "reference" and gpu["impl"] == "b200"
    # first solve: identical baseline, U*[0] within the FP32 tolerance
    assert gpu["rho"] == ref["rho"]
    assert abs(gpu["eta"] - ref["eta"]) <= 1e-9 * max(1.0, ref["eta"])
    assert np.allclose(gpu["u0"], ref["u0"], rtol=1e-4, atol=1e-5)
    # closed loop through the reference Plant: same number of solves, states close
    assert gpu["solves"] == ref["solves"]
    xr, xg = np.array(ref["x"]), np.array(gpu["x"])
    assert xr.shape == xg.shape
    assert np.allclose(xg[:5], xr[:5], rtol=1e-4, atol=1e-5)
    assert abs(gpu["accumulated_cost"] - ref["accumulated_cost"]) <= 1e-3 * max(1.0, abs(ref["accumulated_cost"]))


@pytest.mark.gpu
def test_reference_plant_drives_user_model_plugin():
    """The user's own DynamicsModel / CostFunction subclasses (spring-mass)
    run by the unmodified reference MppiController, and the same model's
    device twin (out-of-tree plugin, include/smpc_b200_plugin.cuh) run by
    GpuMppiController: identical first solve (the Philox noise, the model's
    IEEE ops and the softmin baseline reproduce bit for bit; U* within the
    FP32 tolerance), then the reference Plant closed loop on both."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    if not (os.path.exists(BIN_PLUGIN) and os.path.exists(PLUGIN_LIB)):
        pytest.skip("plugin drop-in binary not built (needs /root/reference at build time)")
    r = subprocess.run([BIN_PLUGIN, PLUGIN_LIB, "0.4"], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr
    ref, gpu = [json.loads(ln) for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert gpu["rho"] == ref["rho"] and gpu["argmax_w"] == ref["argmax_w"]
    assert abs(gpu["eta"] - ref["eta"]) <= 1e-9 * max(1.0, ref["eta"])
    assert np.allclose(gpu["u"], ref["u"], rtol=1e-4, atol=1e-5)
    assert gpu["solves"] == ref["solves"]
    xr, xg = np.array(ref["x"]), np.array(gpu["x"])
    assert xr.shape == xg.shape and np.allclose(xg, xr, rtol=1e-4, atol=1e-5)
