"""Multi-GPU over NCCL (one process per GPU): the sample shards of one problem
on 2 GPUs exchange their per-iteration records with ncclAllGather inside the
captured solve graph (smpc_comm_init). Both exchange modes must give every
rank a bitwise-identical mean whose rho/argmin equal the single-GPU solve
exactly and whose U* is within the north-star tolerance. Skipped on a box
with fewer than 2 GPUs (the round-end GPU tiers have one; the in-process
ShardGroup tests cover the same kernels and gather layouts there)."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TOL = 1e-4


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank_main(rank, world, port, mode, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    import ctypes

    import torch
    import torch.distributed as dist
    from paper_2409_07563_b200 import _lib
    from paper_2409_07563_b200 import scenario as S
    from paper_2409_07563_b200.controllers import make_controller
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", rank))
    sc = S.di_swarm_scenario(num_samples=100003, horizon=60, seed=11)
    sc.device = rank
    ctl = make_controller(sc, shard=S.shard_range(sc.num_samples, rank, world))
    ctl.comm_set_mode(mode)
    uid = bytes(128)
    if rank == 0:
        buf = ctypes.create_string_buffer(128)
        _lib.check(_lib.load().smpc_comm_unique_id(buf))
        uid = buf.raw
    obj = [uid]
    dist.broadcast_object_list(obj, src=0)
    ctl.comm_init(obj[0], rank, world)
    out = []
    for _ in range(3):
        s = ctl.compute_control(sc.x0())
        out.append((s.weights.baseline, s.weights.argmin, s.weights.normalizer, s.controls.tobytes()))
    q.put((rank, out))
    dist.destroy_process_group()


@pytest.mark.parametrize("mode", ["single", "exact"])
def test_two_gpu_nccl_solve_matches_single_gpu(mode):
    import torch
    if not torch.cuda.is_available() or torch.cuda.device_count() < 2:
        pytest.skip("needs >= 2 GPUs")
    import torch.multiprocessing as mp
    from paper_2409_07563_b200 import scenario as S
    from paper_2409_07563_b200.controllers import make_controller
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank_main, args=(r, 2, port, mode, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert res[0] == res[1]  # every rank bitwise identical
    sc = S.di_swarm_scenario(num_samples=100003, horizon=60, seed=11)
    one = make_controller(sc)
    for rho, arg, eta, ub in res[0]:
        s = one.compute_control(sc.x0())
        u = np.frombuffer(ub, np.float32).reshape(s.controls.shape)
        assert rho == s.weights.baseline and arg == s.weights.argmin
        assert abs(eta - s.weights.normalizer) <= TOL * max(1.0, abs(eta))
        assert np.all(np.abs(u - s.controls) <= TOL * np.maximum(1.0, np.abs(s.controls)))
        one.set_mean(u)  # same warm start as the sharded solve
