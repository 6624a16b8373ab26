"""CPU: the C-ABI library loads without a GPU, exports every function
include/smpc_b200.h declares, and fails loudly (status, message) when no CUDA
device is present instead of falling back to the CPU."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "smpc_b200.h")


def declared():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(smpc_[a-z0-9_]+)\s*\(", text)))


@pytest.fixture(scope="module")
def lib():
    from paper_2409_07563_b200 import _lib
    if not os.path.exists(_lib.LIB_PATH):
        import __graft_entry__
        __graft_entry__.build()
    return _lib.load()


def test_header_symbols_exported(lib):
    names = declared()
    assert len(names) >= 20
    for n in names:
        assert hasattr(lib, n), n


def test_python_binding_covers_header():
    from paper_2409_07563_b200 import _lib
    assert sorted(_lib.EXPORTED) == declared()


def test_version_and_libm_probe(lib):
    assert b"sm_100a" in lib.smpc_version()
    # the host probe agrees with the exhaustive checker's notion of the default dispatch
    assert lib.smpc_host_libm_uses_fma() in (0, 1)


def test_create_without_gpu_fails_loudly(lib):
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_2409_07563_b200 import scenario as S
    p = S.cartpole_scenario(num_samples=16, horizon=4).to_problem()
    ctx = ctypes.c_void_p()
    rc = lib.smpc_create(ctypes.byref(p), ctypes.byref(ctx))
    assert rc == 4 and not ctx.value
    assert lib.smpc_last_error(None)
    from paper_2409_07563_b200.controllers import SmpcError, make_controller
    with pytest.raises(SmpcError):
        make_controller(S.cartpole_scenario(num_samples=16, horizon=4))


def test_config_errors_need_no_gpu(lib):
    """Validation runs before any device work and reports the reference's text."""
    from paper_2409_07563_b200 import scenario as S
    from paper_2409_07563_b200.controllers import SmpcConfigError, SmpcError, make_controller
    with pytest.raises(SmpcError, match="^mppi: lambda must be > 0$"):
        make_controller(S.Scenario(num_samples=16, horizon=5, dynamics="cartpole", cost="road",
                                   control_std=(1.0,), lambda_=0.0))
    with pytest.raises(SmpcConfigError, match="expects 4 output channels but model 'unicycle' produces 3"):
        make_controller(S.Scenario(num_samples=16, horizon=5, dynamics="unicycle", cost="circle_track"))
    with pytest.raises(SmpcError, match="^sampler: std_dev entries must be > 0$"):
        make_controller(S.Scenario(num_samples=16, horizon=5, dynamics="cartpole", cost="road", control_std=(0.0,)))
    with pytest.raises(SmpcError, match=r"^dmd: step sizes must be in \(0, 1\]$"):
        make_controller(S.Scenario(num_samples=16, horizon=5, dynamics="cartpole", cost="road", control_std=(1.0,),
                                   controller="dmd", step_size=1.5))
    with pytest.raises(SmpcError, match=r"^mppi: iterations must be in \[1, 256\]$"):
        make_controller(S.Scenario(num_samples=16, horizon=5, dynamics="cartpole", cost="road", control_std=(1.0,),
                                   iterations=300))


def test_noise_strategy_rule_mirrors_auto_select():
    """RolloutEngine::auto_select's decision (engine.cpp:281-320; tested with
    an injected clock in test_engine.cpp:334-390): over the scratch budget ->
    the no-scratch strategy; otherwise fused only if strictly faster, ties ->
    split. Pure function, no GPU needed."""
    from paper_2409_07563_b200 import _lib
    L = _lib.load()
    SPLIT, FUSED = _lib.NOISE_SPLIT, _lib.NOISE_FUSED
    assert L.smpc_noise_strategy_rule(1e9, 1e6, 1.0, 5.0) == FUSED   # budget exceeded: no timing matters
    assert L.smpc_noise_strategy_rule(1e3, 1e6, 2.0, 1.0) == FUSED   # fused strictly faster
    assert L.smpc_noise_strategy_rule(1e3, 1e6, 1.0, 2.0) == SPLIT
    assert L.smpc_noise_strategy_rule(1e3, 1e6, 1.5, 1.5) == SPLIT   # tie -> split
    assert L.smpc_noise_strategy_rule(1e6, 1e6, 1.0, 2.0) == SPLIT   # at the budget is within it
