"""SPEC acceptance criteria that run on the device path: #7 fictitious-force relevance
(Fig. 8 mechanism) and #9 weight non-negativity over 10^4 evaluations."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_weight_net_nonnegative_1e4(cuda_ok):
    """10^4 random weight-net evaluations (the product's device net, square output) give no
    negative weight (§5.2 "enforce the non-negative constraint")."""
    from paper_2102_11026_b200.densenet import forward
    from paper_2102_11026_b200.problem import build_problem
    P = build_problem("cfg1")
    rng = np.random.default_rng(9)
    u = rng.standard_normal((P.model.N, 10_000)) * 10.0 ** rng.uniform(-4, 0, 10_000)
    w = forward(P.cm.wnet, u)
    assert w.shape == (P.model.n_tets, 10_000)
    assert np.isfinite(w).all() and int((w < 0).sum()) == 0


def test_fictitious_force_relevance(cuda_ok):
    """A curved decoder and a high-velocity start: every accepted step of the full dynamics has
    ||phi|| <= newton_tol, while the drop_fict trajectory, evaluated with the full residual,
    exceeds the tolerance by >= 10x within 50 steps."""
    from paper_2102_11026_b200.problem import build_problem
    from paper_2102_11026_b200 import rdsim
    from paper_2102_11026_b200.daereduce import ReducedState
    P = build_problem("cfg1", out_scale=2e-2)          # a more curved random decoder
    n = P.cfg.n_p + P.cfg.n_q
    rd0 = np.zeros(n)
    rd0[P.cfg.n_p:] = 3.0                                # high latent velocity
    full = rdsim.SimConfig(dt=P.cfg.dt, newton_tol=1e-8)
    drop = rdsim.SimConfig(dt=P.cfg.dt, newton_tol=1e-8, drop_fict=True)
    st = ReducedState(np.zeros(n), rd0, full.dt)
    for _ in range(50):
        st, (it, nrm) = rdsim.step(P.rm, P.model, st, P.f_ext, full, return_info=True)
        assert nrm <= full.newton_tol
    st = ReducedState(np.zeros(n), rd0, drop.dt)
    worst = 0.0
    for _ in range(50):
        new = rdsim.step(P.rm, P.model, st, P.f_ext, drop)
        phi_full = rdsim.residual(P.rm, P.model, st, P.f_ext, full, r=new.r)
        worst = max(worst, float(np.linalg.norm(phi_full)))
        st = new
    assert worst >= 10 * full.newton_tol, worst
