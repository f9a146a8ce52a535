"""SPEC known-answer tests and CSFD brute-force oracles for the oracle above mcx
(densenet / diffops / elastic / rdsim). These pin the restatement where no reference
code exists (SPEC.md §examples + acceptance criteria 2, 4, 5, 6, 10)."""

import os

import numpy as np
import pytest

from oracle import diffops as od, elastic as oe, reduced as orr, rdsim as ors, nets as on
from oracle import mcx_np as mc
from paper_2102_11026_b200 import synth
from conftest import rel

GOLD = np.load(os.path.join(os.path.dirname(__file__), "golden", "decoder_golden.npz"))


def scalar_net(kind):
    return [{"kind": "fc", "W": np.eye(1), "b": np.zeros(1)}, {"kind": kind}]


def test_fig5_complex_step_bp():
    # w = (x y)^2 at (2,3), x = 2 + h i: forward w = 36 + 36 h i; BP dw/dx = 36 + 18 h i
    h = 1e-10
    x, y = np.array([2.0, h]), np.array([3.0, 0.0])
    z = mc.mul(x, y)
    w = mc.mul(z, z)
    assert w[0] == pytest.approx(36.0) and w[1] / h == pytest.approx(36.0)
    dwdz = 2.0 * z
    dwdx = mc.mul(dwdz, y)
    assert dwdx[0] == pytest.approx(36.0, rel=1e-12) and dwdx[1] / h == pytest.approx(18.0, rel=1e-12)


def test_scalar_kats():
    sq, cu = scalar_net("square"), scalar_net("cube")
    assert od.hvv(sq, np.array([0.7]), np.array([3.0]))[0] == pytest.approx(18.0, rel=1e-12)
    assert od.svv(cu, np.array([0.4]), np.array([2.0]))[0, 0] == pytest.approx(24.0, rel=1e-12)
    assert np.abs(od.svv(sq, np.array([0.4]), np.array([2.0]))).max() < 1e-12
    # f_fict toy: D = q^2, M = 2, q = 1, q_bar = 0 -> 4
    assert 2.0 * od.hvv(sq, np.array([1.0]), np.array([1.0]))[0] == pytest.approx(4.0, rel=1e-12)
    # dJ toy: D = q^3, q = 1, q_bar = 0, qdot_bar = 0 -> svv + hv(3v) = 6 + 18 = 24
    dj = od.svv(cu, np.array([1.0]), np.array([1.0])) + od.hv(cu, np.array([1.0]), np.array([3.0]))
    assert dj[0, 0] == pytest.approx(24.0, rel=1e-12)


def test_linear_decoder():
    rng = np.random.default_rng(1)
    A = rng.standard_normal((9, 3))
    D = [{"kind": "fc", "W": A, "b": np.zeros(9)}]
    q, v, a = rng.standard_normal(3), rng.standard_normal(3), rng.standard_normal(9)
    assert rel(od.jacobian(D, q), A) < 1e-12
    assert rel(od.jvp(D, q, v), A @ v) < 1e-12
    assert np.abs(od.hvv(D, q, v)).max() == 0 and np.abs(od.hv(D, q, v)).max() == 0
    assert np.abs(od.svv(D, q, v)).max() == 0 and np.abs(od.vhp(D, q, a)).max() == 0
    assert rel(od.vjp(D, q, a), A.T @ a) < 1e-12
    assert np.abs(od.jvp(D, q, np.zeros(3))).max() == 0


def _random_decoder(seed=3, n_q=4, N=30, n_p=5, w=12):
    rng = np.random.default_rng(seed)
    Ws, bs = synth.decoder_weights(n_q, w, 4, N, seed=seed, out_scale=1.0)
    U = synth.pca_like_basis(N, n_p, seed=seed + 1)
    return synth.decoder_layers(Ws, bs, U), U, rng


def test_filter_invariants():
    D, U, rng = _random_decoder()
    for _ in range(20):
        q = rng.uniform(-1, 1, 4)
        u = od.value(D, q)
        assert np.linalg.norm(U.T @ u) <= 1e-8 * (np.linalg.norm(u) + 1)
        J = od.jacobian(D, q)
        assert np.abs(U.T @ J).max() < 1e-8
    x = rng.standard_normal(30)
    f = on.forward([{"kind": "filter", "U": U}], x[None, :, None])[0, :, 0]
    ff = on.forward([{"kind": "filter", "U": U}], f[None, :, None])[0, :, 0]
    assert np.abs(ff - f).max() < 1e-12 and np.linalg.norm(U.T @ f) < 1e-10 * np.linalg.norm(x)


def test_contractions_vs_bruteforce_tensors():
    # Acceptance 4: hv/hvv/svv/vhp vs dense tensors from per-entry CSFD
    D, U, rng = _random_decoder(n_q=4, N=24)
    q, v, a = rng.uniform(-.5, .5, 4), rng.uniform(-.3, .3, 4), rng.standard_normal(24)
    n, eps = 4, 1e-10
    E = np.eye(n)
    H = np.zeros((24, n, n))
    S = np.zeros((24, n, n, n))
    for i in range(n):
        for j in range(n):
            X = od._seed(q, 2, [(1, eps * E[:, i:i + 1]), (2, eps * E[:, j:j + 1])])
            H[:, i, j] = on.forward(D, X)[3][:, 0] / eps**2
            for k in range(n):
                X = od._seed(q, 3, [(1, eps * E[:, i:i + 1]), (2, eps * E[:, j:j + 1]), (4, eps * E[:, k:k + 1])])
                S[:, i, j, k] = on.forward(D, X)[7][:, 0] / eps**3
    assert rel(od.hvv(D, q, v), np.einsum("nij,i,j->n", H, v, v)) < 1e-8
    assert rel(od.hv(D, q, v), np.einsum("nij,j->ni", H, v)) < 1e-8
    assert rel(od.svv(D, q, v), np.einsum("nijk,j,k->ni", S, v, v)) < 1e-8
    V = od.vhp(D, q, a)
    assert rel(V, np.einsum("n,nij->ij", a, H)) < 1e-8
    assert np.linalg.norm(V - V.T) <= 1e-8 * np.linalg.norm(V)


def test_eps_stability():
    D, U, rng = _random_decoder()
    q, v = rng.uniform(-.5, .5, 4), rng.uniform(-.3, .3, 4)
    for fn in (lambda e: od.hv(D, q, v, e), lambda e: od.svv(D, q, v, e), lambda e: od.hvv(D, q, v, e)):
        vals = [fn(e) for e in (1e-6, 1e-8, 1e-10, 1e-12)]
        for x in vals[1:]:
            assert rel(x, vals[0]) <= 1e-6


def test_decoder_matches_reference_golden():
    """Oracle bundle vs the same bundle computed with the reference mcx kernels."""
    g = GOLD
    Ws = [g[f"W{l}"] for l in range(4)]
    bs = [g[f"b{l}"] for l in range(4)]
    D = synth.decoder_layers(Ws, bs, g["U"])
    q, v, a = g["q"], g["v"], g["a"]
    assert rel(od.value(D, q), g["value"]) < 1e-14
    assert rel(od.jacobian(D, q), g["jac"]) < 1e-13
    assert rel(od.hvv(D, q, v), g["hvv"]) < 1e-12
    assert rel(od.hv(D, q, v), g["hv"]) < 1e-12
    assert rel(od.svv(D, q, v), g["svv"]) < 1e-12
    assert rel(od.vjp(D, q, a), g["vjp"]) < 1e-13
    assert rel(od.vhp(D, q, a), g["vhp"]) < 1e-12


def _sim(name="tiny", **over):
    cfg = synth.CONFIGS[name]
    if over:
        cfg = synth.SynthConfig(**{**vars(cfg), **over})
    P = synth.build(cfg)
    model = oe.OModel(P["verts"], P["tets"], P["fixed"], cfg.young, cfg.poisson, cfg.density, cfg.alpha)
    D = synth.decoder_layers(P["dec_W"], P["dec_b"], P["U"])
    rm = orr.OReduced(P["U"], D, cfg.n_p, cfg.n_q)
    return ors.OSim(rm, model, P["cub"], synth.wnet_layers(P["wnet_W"], P["wnet_b"])), cfg, P


def test_elastic_consistency():
    sim, cfg, _ = _sim()
    m = sim.model
    assert m.vertex_mass.sum() == pytest.approx(cfg.density * m.vol.sum(), rel=1e-12)
    u = 1e-3 * np.random.default_rng(5).standard_normal(m.N)
    f = oe.internal_force(m, u)
    g = np.array([np.imag(oe.stvk_energy(m, u + 1j * 1e-20 * np.eye(m.N)[i])) / 1e-20 for i in range(m.N)])
    assert rel(f, g) < 1e-10
    K = oe.stiffness_dense(m, u)
    fc = np.array([np.imag(oe.internal_force(m, u + 1j * 1e-20 * np.eye(m.N)[i])) / 1e-20 for i in range(m.N)]).T
    assert rel(K, fc) < 1e-9 and np.abs(K - K.T).max() <= 1e-9 * np.abs(K).max()
    assert oe.stvk_energy(m, np.zeros(m.N)) == 0 and np.abs(oe.internal_force(m, np.zeros(m.N))).max() == 0


def test_system_jacobian_vs_jacobian_oracle():
    # Acceptance 5: relative Frobenius <= 1e-6 over 20 random states
    sim, cfg, _ = _sim()
    fext = synth.gravity(sim.model.mass)
    for seed in range(20):
        q, qb, qdb, p, pb, pdb = synth.random_state(cfg.n_p, cfg.n_q, seed=100 + seed)
        r, rb, rdb = np.r_[p, q], np.r_[pb, qb], np.r_[pdb, qdb]
        for integ in ("exact_sum", "cubature"):
            c = ors.OSimConfig(dt=cfg.dt, integration=integ, drop_fict=bool(seed % 2))
            S = ors.system_jacobian(sim, r, (rb, rdb), fext, c)
            O = ors.jacobian_oracle(sim, r, (rb, rdb), fext, c)
            assert np.linalg.norm(S - O) <= 1e-6 * np.linalg.norm(O)


def test_quiescence_and_linear_equivalence():
    sim, cfg, _ = _sim()
    n = cfg.n_p + cfg.n_q
    z = np.zeros(n)
    c = ors.OSimConfig(dt=cfg.dt, integration="exact_sum")
    assert np.abs(ors.residual(sim, z, (z, z), np.zeros(sim.model.N), c)).max() < 1e-12
    r, rd, it, nrm = ors.step(sim, z, z, np.zeros(sim.model.N), c)
    assert np.abs(r).max() < 1e-10
    # Acceptance 6: linear decoder -> f_fict = 0 and the classic linear-reduction trajectory
    rng = np.random.default_rng(9)
    N = sim.model.N
    A = rng.standard_normal((N, cfg.n_q)) * 1e-3
    A -= sim.rm.U @ (sim.rm.U.T @ A)
    lin = orr.OReduced(sim.rm.U, [{"kind": "fc", "W": A, "b": np.zeros(N)}], cfg.n_p, cfg.n_q)
    lsim = ors.OSim(lin, sim.model, sim.cub_elems, sim.wnet)
    B = np.concatenate([sim.rm.U, A], axis=1)
    Mr = B.T @ (sim.model.mass[:, None] * B)
    fext = synth.gravity(sim.model.mass)
    h, al = cfg.dt, sim.alpha
    r1 = np.zeros(n); rd1 = np.zeros(n); r2 = r1.copy(); rd2 = rd1.copy()
    for _ in range(100):
        r1, rd1, _, _ = ors.step(lsim, r1, rd1, fext, ors.OSimConfig(dt=h, integration="exact_sum", newton_tol=1e-12))
        # classic linear reduction (Eq. 3 discretised): Newton on Mr((1+a h)(r - r0) - h rd0) + h^2 B^T (f(Br) - fext)
        r0, rdo = r2.copy(), rd2.copy()
        x = r0 + h * rdo
        for _ in range(20):
            g = Mr @ ((1 + al * h) * (x - r0) - h * rdo) + h * h * B.T @ (oe.internal_force(sim.model, B @ x) - fext)
            if np.linalg.norm(g) < 1e-12:
                break
            Kr = B.T @ oe.stiffness_dense(sim.model, B @ x) @ B
            x = x - np.linalg.solve((1 + al * h) * Mr + h * h * Kr, g)
        r2, rd2 = x, (x - r0) / h
    assert np.abs(r1 - r2).max() <= 1e-8
    assert np.abs(ors.fictitious_force(lsim, rng.standard_normal(cfg.n_q), np.zeros(cfg.n_q))).max() == 0
