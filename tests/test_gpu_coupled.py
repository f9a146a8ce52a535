"""GPU parity of the substructured scene (paper_2102_11026_b200/substructure.py through the
nlrom_coupled_* C ABI) against the dense CPU oracle (oracle/coupled.py), SURVEY.md §8e."""

import numpy as np
import pytest

from helpers import coupled_setup
from oracle import coupled as oc, rdsim as ors

pytestmark = pytest.mark.gpu


def _scene(P, k, rank=None, world=None):
    from paper_2102_11026_b200.substructure import Core, Scene
    R, f_world, m_core, k_core, f_core, oscene = coupled_setup(P, k)
    sc = Scene(P.rm, P.model, P.cm, R, f_world, Core(m_core, k_core, f_core), rank=rank, world=world)
    return sc, oscene


@pytest.mark.parametrize("name,k", [("tiny", 3), ("cfg1", 4)])
@pytest.mark.parametrize("integ", ["cubature", "exact_sum"])
def test_coupled_fixed_iterations(cuda_ok, name, k, integ):
    from paper_2102_11026_b200.problem import build_problem
    from paper_2102_11026_b200 import rdsim, synth
    P = build_problem(name)
    sc, osc = _scene(P, k)
    rb, rdb, cb, cdb = synth.coupled_state(k, P.cfg.n_p, P.cfg.n_q)
    cfg = rdsim.SimConfig(dt=P.cfg.dt, fixed_iters=2, integration=integ)
    r, rd, c, cd, it, nrm = sc.step(rb, rdb, cb, cdb, cfg)
    ro, rdo, co, cdo, _, no = oc.step(osc, rb, rdb, cb, cdb, ors.OSimConfig(dt=P.cfg.dt, fixed_iters=2,
                                                                             integration=integ))
    assert np.abs(r - ro).max() <= 1e-10 * np.abs(ro).max()
    assert np.abs(rd - rdo).max() <= 1e-9 * np.abs(rdo).max()
    assert np.abs(c - co).max() <= 1e-10 * np.abs(co).max()
    assert np.abs(cd - cdo).max() <= 1e-9 * np.abs(cdo).max()
    assert abs(nrm - no) <= 1e-8 * no + 1e-14


def test_coupled_adaptive(cuda_ok):
    from paper_2102_11026_b200.problem import build_problem
    from paper_2102_11026_b200 import rdsim, synth
    P = build_problem("tiny")
    sc, osc = _scene(P, 3)
    rb, rdb, cb, cdb = synth.coupled_state(3, P.cfg.n_p, P.cfg.n_q)
    cfg = rdsim.SimConfig(dt=P.cfg.dt, newton_tol=1e-9)
    r, rd, c, cd, it, nrm = sc.step(rb, rdb, cb, cdb, cfg)
    ro, rdo, co, cdo, ito, no = oc.step(osc, rb, rdb, cb, cdb, ors.OSimConfig(dt=P.cfg.dt, newton_tol=1e-9))
    assert it == ito and nrm <= 1e-9
    assert np.abs(r - ro).max() <= 1e-9 * np.abs(ro).max()
    assert np.abs(c - co).max() <= 1e-9 * np.abs(co).max()


def test_coupled_emulated_shards(cuda_ok):
    """Two shards (ranks 0 and 1 of 2) driven in lockstep in one process, partials summed as the
    allreduce would: equal to the one-rank run within reduction-order roundoff."""
    import torch
    from paper_2102_11026_b200.problem import build_problem
    from paper_2102_11026_b200 import rdsim, synth
    P = build_problem("cfg1")
    k = 5
    one, _ = _scene(P, k)
    shards = [_scene(P, k, rank=r, world=2)[0] for r in range(2)]
    rb, rdb, cb, cdb = synth.coupled_state(k, P.cfg.n_p, P.cfg.n_q)
    cfg = rdsim.SimConfig(dt=P.cfg.dt, fixed_iters=2)
    r1, _, c1, _, _, n1 = one.step(rb, rdb, cb, cdb, cfg)
    for s in shards:
        s.begin(rb, rdb, cb, cdb, cfg)
    for it in range(cfg.fixed_iters + 1):
        jac = it < cfg.fixed_iters
        for s in shards:
            s.eval(jac)
        torch.cuda.synchronize()
        tot = shards[0].partial + shards[1].partial
        norms = [s.update(1 if jac else 0, 1.0, total=tot.clone(), want_norm=not jac) for s in shards]
    torch.cuda.synchronize()
    for s in shards:
        r, _, c, _ = s.read(cfg.dt)
        assert np.abs(r - r1[s.lo:s.hi]).max() <= 1e-12 * np.abs(r1).max()
        assert np.abs(c - c1).max() <= 1e-12 * np.abs(c1).max()
    assert abs(norms[0] - n1) <= 1e-10 * n1


def test_coupled_batched_strings(cuda_ok, monkeypatch):
    """Many strings per rank take the big-tile batched decoder path (forced here on cfg4's string)."""
    from paper_2102_11026_b200.problem import build_problem
    from paper_2102_11026_b200 import rdsim, synth
    monkeypatch.setenv("NLROM_PATH", "batched")
    P = build_problem("cfg4")
    k = 3
    sc, osc = _scene(P, k)
    rb, rdb, cb, cdb = synth.coupled_state(k, P.cfg.n_p, P.cfg.n_q)
    cfg = rdsim.SimConfig(dt=P.cfg.dt, fixed_iters=1)
    r, rd, c, cd, it, nrm = sc.step(rb, rdb, cb, cdb, cfg)
    ro, _, co, _, _, no = oc.step(osc, rb, rdb, cb, cdb, ors.OSimConfig(dt=P.cfg.dt, fixed_iters=1))
    assert np.abs(r - ro).max() <= 1e-10 * np.abs(ro).max()
    assert np.abs(c - co).max() <= 1e-10 * np.abs(co).max()
