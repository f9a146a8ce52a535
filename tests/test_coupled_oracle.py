"""Substructured-scene oracle (oracle/coupled.py) and the host-side sharding logic of
paper_2102_11026_b200/substructure.py on CPU, including a world-size-2 gloo run."""

import os
import socket

import numpy as np
import pytest

from helpers import coupled_setup
from oracle import coupled as oc, rdsim as ors


@pytest.fixture(scope="module")
def tiny_scene():
    from paper_2102_11026_b200.problem import build_problem
    from paper_2102_11026_b200 import synth
    P = build_problem("tiny")
    R, f_world, m_core, k_core, f_core, scene = coupled_setup(P, 3)
    state = synth.coupled_state(3, P.cfg.n_p, P.cfg.n_q)
    return P, scene, state


def test_frames_are_rotations():
    from paper_2102_11026_b200 import synth
    R = synth.string_frames(320)
    assert np.allclose(np.einsum("kij,kil->kjl", R, R), np.eye(3), atol=1e-12)
    assert np.allclose(np.linalg.det(R), 1.0)
    d = R[:, :, 0]
    assert np.abs(d.mean(axis=0)).max() < 0.01  # spread over the sphere


def test_coupled_jacobian_matches_finite_differences(tiny_scene):
    """The arrowhead Newton matrix (string blocks = rdsim.system_jacobian with the coupling load,
    C_s, E_s, Z) against central differences of the coupled residual (exact-sum integration)."""
    P, scene, (rb, rdb, cb, cdb) = tiny_scene
    k, n = rb.shape
    cfg = ors.OSimConfig(dt=P.cfg.dt, integration="exact_sum")
    st = (rb, rdb, cb, cdb)
    rs, c = rb + 0.01, cb + 1e-3
    A = oc.jacobian(scene, rs, c, st, cfg)
    x0 = np.concatenate([rs.reshape(-1), c])

    def F(x):
        p, q = oc.residual(scene, x[:k * n].reshape(k, n), x[k * n:], st, cfg)
        return np.concatenate([p.reshape(-1), q])
    Afd = np.zeros_like(A)
    for j in range(x0.size):
        e = np.zeros_like(x0)
        hh = 1e-6 * max(1.0, abs(x0[j]))
        e[j] = hh
        Afd[:, j] = (F(x0 + e) - F(x0 - e)) / (2 * hh)
    assert np.abs(A - Afd).max() / np.abs(Afd).max() < 1e-7


def test_uncoupled_limit(tiny_scene):
    """With the core pinned (infinite mass, no motion) each string is exactly the single-body
    rdsim residual under its rotated load."""
    P, scene, (rb, rdb, cb, cdb) = tiny_scene
    cfg = ors.OSimConfig(dt=P.cfg.dt)
    z = np.zeros(3)
    phis, _ = oc.residual(scene, rb + 0.01, z, (rb, rdb, z, z), cfg)
    for s in range(scene.k):
        f_loc = oc.to_local(scene.R[s], scene.f_world[s])
        want = ors.residual(scene.sim, rb[s] + 0.01, (rb[s], rdb[s]), f_loc, cfg)
        assert np.abs(phis[s] - want).max() <= 1e-13 * np.abs(want).max()


def test_sharded_single_rank_equals_dense(tiny_scene):
    """Schur-complement restatement (one rank) == the dense arrowhead LU solve."""
    P, scene, (rb, rdb, cb, cdb) = tiny_scene
    cfg = ors.OSimConfig(dt=P.cfg.dt, fixed_iters=3)
    r1, _, c1, _, _, n1 = oc.step(scene, rb, rdb, cb, cdb, cfg)
    r2, _, c2, _, n2 = oc.step_sharded(scene, rb, rdb, cb, cdb, cfg, 0, 1, lambda v: v)
    assert np.abs(r2 - r1).max() <= 1e-10 * np.abs(r1).max()
    assert np.abs(c2 - c1).max() <= 1e-10 * np.abs(c1).max()
    assert abs(n2 - n1) <= 1e-9 * n1


def test_adaptive_converges(tiny_scene):
    P, scene, (rb, rdb, cb, cdb) = tiny_scene
    cfg = ors.OSimConfig(dt=P.cfg.dt, newton_tol=1e-9)
    r, rd, c, cd, it, nrm = oc.step(scene, rb, rdb, cb, cdb, cfg)
    assert nrm <= 1e-9 and 1 <= it <= cfg.max_iters


def test_shard_partition():
    from paper_2102_11026_b200.substructure import shard
    for k in (1, 7, 320):
        for world in (1, 2, 3, 8):
            if world > k:
                continue
            rngs = [shard(k, r, world) for r in range(world)]
            assert rngs[0][0] == 0 and rngs[-1][1] == k
            assert all(a[1] == b[0] for a, b in zip(rngs, rngs[1:]))
            assert max(h - l for l, h in rngs) - min(h - l for l, h in rngs) <= 1
            assert [oc.shard(k, r, world) for r in range(world)] == rngs


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _gloo_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2102_11026_b200.problem import build_problem
        from paper_2102_11026_b200 import synth
        from paper_2102_11026_b200.substructure import allreduce_sum, dist_info, shard
        P = build_problem("tiny")
        _, _, _, _, _, scene = coupled_setup(P, 3)
        rb, rdb, cb, cdb = synth.coupled_state(3, P.cfg.n_p, P.cfg.n_q)
        cfg = ors.OSimConfig(dt=P.cfg.dt, fixed_iters=2)

        def ar(v):
            t = torch.from_numpy(v.copy())
            allreduce_sum(t)  # the product's host collective (gloo here, NCCL on the GPU box)
            return t.numpy()
        r, rd, c, cd, nrm = oc.step_sharded(scene, rb, rdb, cb, cdb, cfg, rank, world, ar)
        q.put((rank, dist_info(), shard(3, rank, world), r, c, nrm))
    finally:
        dist.destroy_process_group()


def test_gloo_two_ranks_match_dense(tiny_scene):
    """world_size 2 over gloo: strings sharded, one allreduce per Newton iteration; every rank's
    strings and the replicated core equal the dense single-process solve."""
    import torch.multiprocessing as mp
    P, scene, (rb, rdb, cb, cdb) = tiny_scene
    cfg = ors.OSimConfig(dt=P.cfg.dt, fixed_iters=2)
    r1, _, c1, _, _, n1 = oc.step(scene, rb, rdb, cb, cdb, cfg)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gloo_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, info, (lo, hi), r, c, nrm in res:
        assert info == (rank, 2)
        assert np.abs(r - r1[lo:hi]).max() <= 1e-10 * np.abs(r1).max()
        assert np.abs(c - c1).max() <= 1e-10 * np.abs(c1).max()
        assert abs(nrm - n1) <= 1e-9 * n1
