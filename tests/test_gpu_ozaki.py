"""The batched decoder's hidden jet layers on the 5th-generation tensor cores (tcgen05.mma
kind::i8 Ozaki-scheme fp64, csrc/ozaki_tc.cuh) against the oracle, at a width-256 decoder
(cfg5's 10-layer w256 DAE) with enough sims (160: 15k jet columns, >= 3 waves of 128 x 64 tiles)
that the dispatch puts every hidden layer on tcgen05, and against the fp64-DMMA hidden layers
(NLROM_PATH=dmma_hidden). Norm-relative tolerances as the DMMA path: the Ozaki products carry
~1e-16 of sum |w||x| (55-bit digits), fp64-class. The digit chain (hidden layers handing digit
tiles to each other, csrc/ozaki_chain.cuh) is bitwise equal to the fp64 hand-off."""

import os
import subprocess
import sys

import numpy as np
import pytest

from conftest import rel
from helpers import oracle_sim, ocfg
from oracle import rdsim as ors

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

_SCRIPT = r"""
import sys, numpy as np
sys.path.insert(0, sys.argv[1])
from paper_2102_11026_b200.problem import build_problem
from paper_2102_11026_b200 import rdsim
from paper_2102_11026_b200.session import Session
P = build_problem("cfg5")
ns = int(sys.argv[3])
n = P.cfg.n_p + P.cfg.n_q
s = Session(P.rm, P.model, P.cm, n_sims=ns)
st = [P.random_state(seed=70 + i) for i in range(ns)]
r, rb, rdb = (np.concatenate([x[j] for x in st]) for j in range(3))
fe = np.tile(P.f_ext, ns)
cfg = rdsim.SimConfig(dt=P.cfg.dt)
phi = s.residual(r, rb, rdb, fe, cfg)
S = s.system_jacobian(r, rb, rdb, fe, cfg)
z = np.zeros(ns * n)
r2, rd2, _, _ = s.step(z, z, fe, rdsim.SimConfig(dt=P.cfg.dt, fixed_iters=2))
np.savez(sys.argv[2], phi=phi, S=S, r=r2, rd=rd2, tc=np.array(s.tc_info()))
"""


NS = 160


def _run(tmp_path, path, ns=NS):
    out = str(tmp_path / f"o_{path.replace(',', '_')}.npz")
    env = dict(os.environ, NLROM_PATH=path)
    subprocess.run([sys.executable, "-c", _SCRIPT, ROOT, out, str(ns)], env=env, check=True, timeout=900)
    return np.load(out)


def test_ozaki_hidden_layers_vs_oracle_and_dmma(cuda_ok, tmp_path):
    from paper_2102_11026_b200.problem import build_problem
    from paper_2102_11026_b200 import rdsim
    oz = _run(tmp_path, "")
    dm = _run(tmp_path, "dmma_hidden")
    assert tuple(oz["tc"])[0] == 8 and tuple(dm["tc"])[0] == 0   # hidden GEMMs on tcgen05 / on DMMA
    P = build_problem("cfg5")
    S = oracle_sim(P)
    ns, n = NS, P.cfg.n_p + P.cfg.n_q
    oc = ocfg(rdsim.SimConfig(dt=P.cfg.dt))
    for i in (0, 77, ns - 1):
        r, rb, rdb = P.random_state(seed=70 + i)
        phio = ors.residual(S, r, (rb, rdb), P.f_ext, oc)
        Jo = ors.system_jacobian(S, r, (rb, rdb), P.f_ext, oc)
        assert rel(oz["phi"].reshape(ns, n)[i], phio) < 1e-11, i
        assert rel(oz["S"][i], Jo) < 1e-11, i
    ro, rdo, _, _ = ors.step(S, np.zeros(n), np.zeros(n), P.f_ext,
                             ocfg(rdsim.SimConfig(dt=P.cfg.dt, fixed_iters=2)))
    for i in (0, ns - 1):
        assert np.abs(oz["r"].reshape(ns, n)[i] - ro).max() <= 1e-10 * np.abs(ro).max(), i
    # the two tensor paths agree to fp64 roundoff
    assert rel(oz["S"], dm["S"]) < 1e-12
    assert rel(oz["phi"], dm["phi"]) < 1e-11


@pytest.mark.parametrize("ns", [NS, 161])
def test_digit_chain_bitwise(cuda_ok, tmp_path, ns):
    """Hidden layers handing digit tiles + exponents to each other (default) vs handing fp64
    activations that the consumer converts (NLROM_PATH=oz_fp64_chain): same digits, same
    exponents, so every output is bitwise equal (161 sims: a half-empty last 64-column tile)."""
    dg = _run(tmp_path, "", ns)
    fp = _run(tmp_path, "oz_fp64_chain", ns)
    assert tuple(dg["tc"])[0] == 8
    for k in ("phi", "S", "r", "rd"):
        assert np.array_equal(dg[k], fp[k]), k
    if ns % 2:   # the last sim's columns straddle the half-empty last tile: vs the oracle too
        from paper_2102_11026_b200.problem import build_problem
        from paper_2102_11026_b200 import rdsim
        P = build_problem("cfg5")
        S = oracle_sim(P)
        n = P.cfg.n_p + P.cfg.n_q
        i = ns - 1
        r, rb, rdb = P.random_state(seed=70 + i)
        oc = ocfg(rdsim.SimConfig(dt=P.cfg.dt))
        assert rel(dg["phi"].reshape(ns, n)[i], ors.residual(S, r, (rb, rdb), P.f_ext, oc)) < 1e-11
        assert rel(dg["S"][i], ors.system_jacobian(S, r, (rb, rdb), P.f_ext, oc)) < 1e-11
