"""CPU, world_size 2 over gloo: the multi-GPU sample-sharding protocol.

Each rank owns the global samples [r*M/W, (r+1)*M/W) (WorkerPool chunk rule,
worker_pool.hpp:28-29), draws their noise from the same Philox counters
(sampling.cpp:74-75: the counter carries the global m), rolls them out and
exchanges exactly what the device path all-gathers per iteration, in the
device's arithmetic order (the division by eta happens once per entry at
commit, kernels.cuh commit_update):

"exact" mode (three collectives, SMPC_COMM_EXACT):
  1. (rho_g, argmin_g)          -> global rho / lowest-index argmin
  2. eta_g = sum_local exp(-(J-rho)/lambda)
  3. S_g = sum_local e_m eps_m  (T x n_u doubles, unnormalised)
"single" mode (one collective, SMPC_COMM_SINGLE): every rank weighs its
samples against its LOCAL baseline rho_g and all-gathers one record
  (rho_g, argmin_g, eta_g, S_g) with eta_g = sum_local exp(-(J-rho_g)/lambda),
  S_g = sum_local exp(-(J-rho_g)/lambda) eps_m;
the combine rescales rank g by exp(-(rho_g - rho)/lambda) before summing.
Both combine in fixed rank order (kernels.cuh global_min / global_eta /
combine_kernel), so every rank ends with a bitwise-identical mean
U* = mu + gamma * S / eta. The result must equal the single-process reference
iteration: rho and argmin exactly, eta and U* within 1e-12 / 1e-4. The CPU
oracle stands in for the per-rank device kernels here.
"""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2409_07563_b200 import scenario as S


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank_main(rank, world, port, sc_args, mode, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import torch
    from oracle.bindings import Oracle
    sc = S.cartpole_scenario(**sc_args)
    n_x, n_u, n_y = sc.dims
    T, M = sc.horizon, sc.num_samples
    o = Oracle("port")
    b, e = S.shard_range(M, rank, world)
    mean = np.zeros((T, n_u), np.float32)
    eps, _ = o.generate_samples(sc, mean, 0, m_begin=b, m_end=e)
    costs = o.rollout(sc, sc.x0()[None], mean[None], eps)[0] if e > b else np.zeros(0)
    loc_rho = costs.min() if e > b else np.inf
    loc_arg = b + int(np.argmin(costs)) if e > b else 2 ** 62

    def rank_min(recs):  # rank order == ascending global index: ties keep the lowest
        rho, arg = np.inf, 2 ** 62
        for r in recs:
            if r[0] < rho or (r[0] == rho and r[1] < arg):
                rho, arg = r[0], int(r[1])
        return rho, arg

    TU = T * n_u
    if mode == "exact":
        g1 = [torch.zeros(2, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(g1, torch.tensor([loc_rho, float(loc_arg)], dtype=torch.float64))
        rho, arg = rank_min([t.numpy() for t in g1])
        ev = np.exp(-(costs - rho) / sc.lambda_)
        g2 = [torch.zeros(1, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(g2, torch.tensor([ev.sum()]))
        eta = 0.0
        for t in g2:
            eta += t.item()
        acc = np.zeros(TU)
        for i in range(e - b):  # ascending m, unnormalised
            acc += ev[i] * eps[i].reshape(-1).astype(np.float64)
        g3 = [torch.zeros(TU, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(g3, torch.tensor(acc))
        tot = np.zeros(TU)
        for t in g3:
            tot += t.numpy()
    else:
        ev = np.exp(-(costs - loc_rho) / sc.lambda_) if e > b else np.zeros(0)
        acc = np.zeros(TU)
        for i in range(e - b):
            acc += ev[i] * eps[i].reshape(-1).astype(np.float64)
        rec = np.concatenate([[loc_rho, float(loc_arg), ev.sum()], acc])
        g = [torch.zeros(3 + TU, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(g, torch.tensor(rec))  # the only collective of the iteration
        recs = [t.numpy() for t in g]
        rho, arg = rank_min(recs)
        eta, tot = 0.0, np.zeros(TU)
        for r in recs:
            if r[0] == np.inf:  # an empty shard contributes nothing
                continue
            scale = np.exp(-(r[0] - rho) / sc.lambda_)
            eta += scale * r[2]
            tot += scale * r[3:]
    u = (mean.reshape(-1).astype(np.float64) + tot / eta).astype(np.float32)
    out_q.put((rank, rho, arg, eta, u.tobytes()))
    dist.destroy_process_group()


@pytest.mark.parametrize("mode", ["exact", "single"])
@pytest.mark.parametrize("M", [1000, 257])
def test_two_rank_iteration_matches_single_process(oracle_built, M, mode):
    world = 2
    sc_args = dict(num_samples=M, horizon=40, seed=3)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank_main, args=(r, world, port, sc_args, mode, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=120) for _ in range(world)])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # all ranks bitwise identical
    assert res[0][1:] == res[1][1:]
    _, rho, arg, eta, ub = res[0]
    u = np.frombuffer(ub, np.float32)
    sc = S.cartpole_scenario(**sc_args)
    ref = oracle_built.OracleController(sc, "port").compute_control(sc.x0())
    assert rho == ref["baseline"] and arg == ref["argmin"]
    assert abs(eta - ref["normalizer"]) <= 1e-12 * ref["normalizer"]
    assert np.all(np.abs(u - ref["controls"].ravel()) <= 1e-4 * np.maximum(1, np.abs(u)))


def test_shard_ranges_follow_worker_pool_rule():
    """test_worker_pool.cpp:29-44: n=10, W=4 -> {0,2},{2,5},{5,7},{7,10}."""
    assert [S.shard_range(10, r, 4) for r in range(4)] == [(0, 2), (2, 5), (5, 7), (7, 10)]
    for n in (1, 7, 1 << 20):
        for w in (1, 2, 3, 8):
            rs = [S.shard_range(n, r, w) for r in range(w)]
            assert rs[0][0] == 0 and rs[-1][1] == n
            assert all(rs[i][1] == rs[i + 1][0] for i in range(w - 1))
