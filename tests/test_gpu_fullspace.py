"""GPU full-space implicit Euler (csrc/fullspace.cu) and pose generation against the oracle
(oracle/fullspace.py: scipy direct solves). Iterative (PCG) vs direct linear solves: the
converged Newton states agree to the Newton tolerance, written in each test."""

import numpy as np
import pytest

from conftest import rel
from oracle import elastic as oe, fullspace as ofs

pytestmark = pytest.mark.gpu


def _models(name, **kw):
    from paper_2102_11026_b200.problem import build_problem
    from helpers import oracle_sim
    P = build_problem(name, **kw)
    return P, oracle_sim(P).model


@pytest.mark.parametrize("name", ["tiny", "cfg1"])
def test_energy_and_force(cuda_ok, name):
    from paper_2102_11026_b200.fullspace import session_for
    P, om = _models(name)
    u = 1e-2 * np.random.default_rng(5).standard_normal(P.model.N)
    e, f = session_for(P.model).energy_force(u)
    assert abs(e - oe.stvk_energy(om, u)) <= 1e-12 * abs(e)
    assert rel(f, oe.internal_force(om, u)) <= 1e-12


def test_rest_and_divergence(cuda_ok):
    from paper_2102_11026_b200 import _lib
    from paper_2102_11026_b200.elastic import fullspace_step
    from paper_2102_11026_b200.fullspace import FullspaceConfig
    P, _ = _models("tiny")
    z = np.zeros(P.model.N)
    u, v, info = fullspace_step(P.model, z, z, z, 1 / 60, return_info=True)
    assert info.iters == 0 and not u.any() and not v.any()
    with pytest.raises(_lib.NewtonDivergence):
        fullspace_step(P.model, z, z, P.f_ext, 1 / 60, cfg=FullspaceConfig(max_iters=0))
    with pytest.raises(ValueError):
        fullspace_step(P.model, z, z, z, 0.0)


@pytest.mark.parametrize("name,beta", [("tiny", 0.0), ("cfg1", 0.0), ("tiny", 0.01)])
def test_trajectory_vs_oracle(cuda_ok, name, beta):
    """Gravity from rest, 5 steps: u' and v' within 1e-8 (norm-relative) of the direct-solve
    oracle; Newton converges in the same number of iterations."""
    from paper_2102_11026_b200.fullspace import FullspaceConfig, FullspaceSession
    P, om = _models(name)
    s = FullspaceSession(P.model, beta=beta)
    cfg = FullspaceConfig(newton_tol=1e-10)
    u = v = np.zeros(P.model.N)
    uo = vo = np.zeros(P.model.N)
    for k in range(5):
        u, v, info = s.step(u, v, P.f_ext, P.cfg.dt, cfg)
        uo, vo, ito, _ = ofs.fullspace_step(om, uo, vo, P.f_ext, P.cfg.dt, beta=beta, newton_tol=1e-10)
        assert rel(u, uo) <= 1e-8 and rel(v, vo) <= 1e-8, k
        assert info.iters == ito and info.res_norm <= 1e-10 * max(1.0, np.linalg.norm(P.f_ext))
        assert abs(info.energy - oe.stvk_energy(om, u)) <= 1e-9 * max(info.energy, 1e-30)


def test_cfg2_mesh_step(cuda_ok):
    """cfg2 mesh (N = 6720): one step from rest under gravity vs the oracle."""
    from paper_2102_11026_b200.fullspace import FullspaceConfig, session_for
    P, om = _models("cfg2", n_fc=2, width=16)
    z = np.zeros(P.model.N)
    u, v, info = session_for(P.model).step(z, z, P.f_ext, P.cfg.dt, FullspaceConfig(newton_tol=1e-10))
    uo, vo, ito, _ = ofs.fullspace_step(om, z, z, P.f_ext, P.cfg.dt, newton_tol=1e-10)
    assert rel(u, uo) <= 1e-8 and rel(v, vo) <= 1e-8 and info.iters == ito


def test_generate_poses_vs_oracle(cuda_ok):
    """posegen.generate_poses (GPU integrator) == oracle pose generator on the same script;
    deterministic under seed (bit-identical on a rerun)."""
    from paper_2102_11026_b200 import posegen
    from paper_2102_11026_b200.fullspace import FullspaceConfig
    P, om = _models("tiny")
    sc = posegen.ForceScript(seed=3, episodes=3, radius=0.12, magnitude=(0.5, 2.0), steps=3, dt=P.cfg.dt)
    cfg = FullspaceConfig(newton_tol=1e-10)
    ps = posegen.generate_poses(P.model, sc, cfg)
    assert ps.poses.shape == (P.model.N, 3 * 3 + 1) and not ps.poses[:, -1].any()
    X, E = ofs.generate_poses(om, 3, 3, 3, P.cfg.dt, 0.12, (0.5, 2.0))
    assert rel(ps.poses, X) <= 1e-8 and rel(ps.energies, E) <= 1e-8
    ps2 = posegen.generate_poses(P.model, sc, cfg)
    assert np.array_equal(ps.poses, ps2.poses) and np.array_equal(ps.energies, ps2.energies)
    assert np.isclose(ps.weights.mean(), 1.0) and np.argmax(ps.weights) == ps.energies.size - 1
    U = posegen.pca_basis(ps, 3, 6)
    assert np.abs(U.T @ U - np.eye(3)).max() <= 1e-10
