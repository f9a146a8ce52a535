"""Independent-sim sharding -- host-side logic on CPU: the sim partition,
and a world-size-2 gloo run in which each rank steps its own sim range (the oracle stands in
for the device step) and the product's gather_rows reassembles every sim in order, equal to
one process stepping all sims. The GPU counterpart is tests/test_gpu_multi.py."""

import os
import socket

import numpy as np
import pytest

from helpers import oracle_sim
from oracle import rdsim as ors
from paper_2102_11026_b200.shard import shard_range


def test_shard_range_partition():
    for total in (0, 1, 7, 100, 4096):
        for world in (1, 2, 3, 4, 8):
            rngs = [shard_range(total, r, world) for r in range(world)]
            assert rngs[0][0] == 0 and rngs[-1][1] == total
            assert all(a[1] == b[0] for a, b in zip(rngs, rngs[1:]))
            sizes = [h - l for l, h in rngs]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard_range(10, 2, 2)


def _sims(P, total):
    n = P.cfg.n_p + P.cfg.n_q
    rng = np.random.default_rng(4)
    return rng.uniform(-0.05, 0.05, (total, n)), rng.uniform(-0.1, 0.1, (total, n)), rng.uniform(0.5, 1.5, total)


def _step_range(P, S, lo, hi, rb, rdb, scale):
    cfg = ors.OSimConfig(dt=P.cfg.dt, fixed_iters=2)
    out = []
    for i in range(lo, hi):
        r, _, _, _ = ors.step(S, rb[i].copy(), rdb[i].copy(), scale[i] * P.f_ext, cfg)
        out.append(r)
    return np.array(out).reshape(hi - lo, -1)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, total, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2102_11026_b200.problem import build_problem
        from paper_2102_11026_b200.shard import gather_rows
        P = build_problem("tiny")
        S = oracle_sim(P)
        rb, rdb, scale = _sims(P, total)
        lo, hi = shard_range(total, rank, world)
        local = _step_range(P, S, lo, hi, rb, rdb, scale)
        q.put((rank, lo, hi, gather_rows(lo, local, world)))
    finally:
        dist.destroy_process_group()


def test_gloo_two_ranks_independent_sims():
    import torch.multiprocessing as mp
    from paper_2102_11026_b200.problem import build_problem
    total = 5
    P = build_problem("tiny")
    S = oracle_sim(P)
    rb, rdb, scale = _sims(P, total)
    want = _step_range(P, S, 0, total, rb, rdb, scale)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, total, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert [(lo, hi) for _, lo, hi, _ in res] == [(0, 2), (2, 5)]
    for _, _, _, allr in res:
        assert np.array_equal(allr, want)  # same arithmetic per sim: bitwise
