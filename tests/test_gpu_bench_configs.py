"""The benchmarked configurations themselves, checked at the size they are timed (VERDICT r1:
"the benchmarked configuration is never parity-checked"):

* cfg2 exactly (n_q = 30, L = 10, w = 256, |C| = 500): 10 timesteps x 3 fixed Newton iterations
  through rdsim.step (the e2e path) vs the oracle, and the timed one-iteration graph
  (nlrom_iterate, the graph bench.py replays) vs oracle Newton iterations;
* cfg5 at the full 4096 sims with the default kernel selection (big-tile batched decoder,
  warp-specialised hidden layers, split-K seed GEMM, shared-real vhp backward, cubature with
  several element chunks per CTA): 8 sampled sims vs the single-sim oracle.
Tolerance: norm-relative <= 1e-10 (fp64 path)."""

import numpy as np
import pytest
import scipy.linalg

from conftest import rel
from helpers import oracle_sim, ocfg
from oracle import rdsim as ors

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def cfg2(cuda_ok):
    from paper_2102_11026_b200.problem import build_problem
    P = build_problem("cfg2")
    return P, oracle_sim(P)


def test_cfg2_ten_steps_three_iterations(cfg2):
    from paper_2102_11026_b200 import rdsim
    P, S = cfg2
    # gravity from rest (a random state makes un-damped fixed-iteration Newton diverge, which
    # amplifies roundoff chaotically: not a parity test)
    cfg = rdsim.SimConfig(dt=P.cfg.dt, fixed_iters=3)
    st = P.rest_state()
    ro, rdo = st.r.copy(), st.rdot.copy()
    worst = 0.0
    for _ in range(10):
        st = rdsim.step(P.rm, P.model, st, P.f_ext, cfg)
        ro, rdo, _, _ = ors.step(S, ro, rdo, P.f_ext, ocfg(cfg))
        worst = max(worst, rel(st.r, ro), rel(st.rdot, rdo))
    assert worst <= 1e-10, worst


def test_cfg2_step_norm_optional(cfg2):
    """rdsim.step evaluates the final residual of a fixed-iteration step only when it returns it
    (return_info): the state is bitwise the same either way, and the returned norm is the
    oracle's ||phi|| at the final iterate."""
    from paper_2102_11026_b200 import rdsim
    P, S = cfg2
    cfg = rdsim.SimConfig(dt=P.cfg.dt, fixed_iters=3)
    st = P.rest_state()
    a = rdsim.step(P.rm, P.model, st, P.f_ext, cfg)
    b, (iters, nrm) = rdsim.step(P.rm, P.model, st, P.f_ext, cfg, return_info=True)
    assert iters == 3
    assert np.array_equal(a.r, b.r) and np.array_equal(a.rdot, b.rdot)
    ro, _, _, nrm_o = ors.step(S, st.r.copy(), st.rdot.copy(), P.f_ext, ocfg(cfg))
    assert rel(b.r, ro) <= 1e-10
    assert abs(nrm - nrm_o) <= 1e-8 * max(nrm_o, 1e-300) + 1e-12


def test_cfg2_timed_graph(cfg2):
    from paper_2102_11026_b200 import rdsim
    from paper_2102_11026_b200.session import session_for
    P, S = cfg2
    _, rb, rdb = P.random_state()
    s = session_for(P.rm, P.model, P.cm)
    s.step(rb, rdb, P.f_ext, rdsim.SimConfig(dt=P.cfg.dt, fixed_iters=1))
    r0, _, _ = s.get_iterate()
    oc = ors.OSimConfig(dt=P.cfg.dt)
    ro = r0.copy()
    for _ in range(3):
        s.iterate(1)
        rg, phig, nrm = s.get_iterate()
        phio = ors.residual(S, ro, (rb, rdb), P.f_ext, oc)
        ro = ro + scipy.linalg.lu_solve(scipy.linalg.lu_factor(ors.system_jacobian(S, ro, (rb, rdb), P.f_ext, oc)),
                                        -phio)
        assert rel(phig, phio) <= 1e-10
        assert rel(rg, ro) <= 1e-10
        assert abs(nrm[0] - np.linalg.norm(phio)) <= 1e-10 * np.linalg.norm(phio)


@pytest.mark.parametrize("total", [4096, 1000])
def test_cfg5_full_scale_sampled_sims(cuda_ok, total):
    """4096 sims: the benchmarked configuration; 1000 sims: ragged tcgen05 column tiles (the output
    layer's 42000 and the backward's 21000 columns are not multiples of their 64 / 63-column tiles)."""
    from paper_2102_11026_b200.problem import build_problem
    from paper_2102_11026_b200 import rdsim
    from paper_2102_11026_b200.shard import SimShard
    P = build_problem("cfg5")
    n = P.cfg.n_p + P.cfg.n_q
    rng = np.random.default_rng(4)
    rb = rng.uniform(-0.05, 0.05, (total, n))
    rdb = rng.uniform(-0.1, 0.1, (total, n))
    scale = rng.uniform(0.5, 1.5, total)
    fe = scale[:, None] * P.f_ext[None, :]
    sh = SimShard(P.rm, P.model, P.cm, total, rank=0, world=1)
    assert sh.session.tc_info() == (8, 1, 8)   # hidden, output and backward GEMMs on tcgen05
    cfg = rdsim.SimConfig(dt=P.cfg.dt, fixed_iters=2)
    r, rd, _ = sh.step(rb, rdb, fe, cfg)
    S = oracle_sim(P)
    for i in np.random.default_rng(7).choice(total, 8, replace=False):
        ro, rdo, _, _ = ors.step(S, rb[i].copy(), rdb[i].copy(), fe[i], ocfg(cfg))
        assert rel(r[i], ro) <= 1e-10, i
        assert rel(rd[i], rdo) <= 1e-8, i


# ------------------------------------------------------------------ adaptive Newton on the device
def test_cfg2_adaptive_steps_device_loop(cfg2):
    """rdsim.step in adaptive mode runs the Newton / line-search loops as conditional graph nodes
    (newton_kernels.cuh): iteration counts and states equal the oracle's host loop at cfg2."""
    from paper_2102_11026_b200 import rdsim
    P, S = cfg2
    cfg = rdsim.SimConfig(dt=P.cfg.dt, newton_tol=1e-9)
    st = P.rest_state()
    ro, rdo = st.r.copy(), st.rdot.copy()
    for _ in range(6):
        st, (it, nrm) = rdsim.step(P.rm, P.model, st, P.f_ext, cfg, return_info=True)
        ro, rdo, ito, nro = ors.step(S, ro, rdo, P.f_ext, ocfg(cfg))
        assert it == ito and nrm <= cfg.newton_tol
        assert rel(st.r, ro) <= 1e-10


def test_adaptive_line_search_and_limits(cuda_ok):
    """Hard states (scaled random r_bar, rdot_bar): at 0.45 Newton converges in 6 iterations, at
    0.5 the backtracking line search engages every iteration (oracle halvings 4, 2, 5 after a full
    first step) and 4 iterations do not converge -- the device loop raises NewtonDivergence with
    the oracle's last norm. max_iters = 2 at a 1e-300 tolerance raises after 2 iterations."""
    from paper_2102_11026_b200.problem import build_problem
    from paper_2102_11026_b200 import rdsim
    from paper_2102_11026_b200.daereduce import ReducedState
    from paper_2102_11026_b200._lib import NewtonDivergence
    from oracle.rdsim import NewtonDivergence as ONewtonDivergence
    P = build_problem("cfg2", n_fc=4)
    S = oracle_sim(P)
    _, rb, rdb = P.random_state()
    cfg = rdsim.SimConfig(dt=P.cfg.dt, newton_tol=1e-8, max_iters=30, line_search=True)
    ro, rdo, ito, nro = ors.step(S, 0.45 * rb, 0.45 * rdb, P.f_ext, ocfg(cfg))
    st, (it, nrm) = rdsim.step(P.rm, P.model, ReducedState(0.45 * rb, 0.45 * rdb, cfg.dt), P.f_ext, cfg,
                               return_info=True)
    assert it == ito and rel(st.r, ro) <= 1e-9
    cfg4 = rdsim.SimConfig(dt=P.cfg.dt, newton_tol=1e-8, max_iters=4, line_search=True)
    halvings = []
    with pytest.raises(ONewtonDivergence) as eo:
        ors.step(S, 0.5 * rb, 0.5 * rdb, P.f_ext, ocfg(cfg4), trace=halvings)
    assert sum(halvings) > 0, halvings
    with pytest.raises(NewtonDivergence) as eg:
        rdsim.step(P.rm, P.model, ReducedState(0.5 * rb, 0.5 * rdb, cfg.dt), P.f_ext, cfg4)
    assert abs(eg.value.last_norm - eo.value.last_norm) <= 1e-8 * eo.value.last_norm
    tight = rdsim.SimConfig(dt=P.cfg.dt, newton_tol=1e-300, max_iters=2)
    with pytest.raises(NewtonDivergence) as ei:
        rdsim.step(P.rm, P.model, ReducedState(rb, rdb, cfg.dt), P.f_ext, tight)
    assert "2 iterations" in str(ei.value)
