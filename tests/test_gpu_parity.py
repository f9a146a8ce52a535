"""GPU parity: every hot-path op through the C ABI against the CPU oracle on the same
seeded inputs. fp64 path: norm-relative <= 1e-12 unless stated."""

import numpy as np
import pytest

from conftest import rel
from helpers import oracle_sim, ocfg
from oracle import diffops as od, nets as on, reduced as orr, rdsim as ors, elastic as oe
from oracle import mcx_np as omc

pytestmark = pytest.mark.gpu

TOL = 1e-12


@pytest.fixture(scope="module")
def cfg1(cuda_ok):
    from paper_2102_11026_b200.problem import build_problem
    P = build_problem("cfg1")
    return P, oracle_sim(P)


@pytest.fixture(scope="module")
def tiny(cuda_ok):
    from paper_2102_11026_b200.problem import build_problem
    P = build_problem("tiny")
    return P, oracle_sim(P)


# ------------------------------------------------------------------ generic nets (densenet)
@pytest.mark.parametrize("order", [0, 1, 2, 3])
def test_net_forward_multicomplex(cfg1, order):
    from paper_2102_11026_b200 import densenet
    from paper_2102_11026_b200.mcx import MCArray
    P, S = cfg1
    rng = np.random.default_rng(order)
    q = rng.uniform(-0.5, 0.5, (1 << order, P.cfg.n_q, 7))
    q[1:] *= 1e-3
    got = densenet.forward(P.rm.decoder, MCArray(q)).parts
    want = on.forward(S.rm.D, q)
    for s in range(1 << order):
        assert rel(got[s], want[s]) < 1e-11, s


def test_net_square_and_wnet(cfg1):
    from paper_2102_11026_b200 import densenet
    P, S = cfg1
    u = np.random.default_rng(2).standard_normal(P.model.N) * 1e-3
    got = densenet.forward(P.cm.wnet, u)
    want = on.forward(S.wnet, u[None, :, None])[0, :, 0]
    assert rel(got, want) < TOL and np.all(got >= 0)


@pytest.mark.parametrize("order", [0, 1])
def test_net_backward(cfg1, order):
    from paper_2102_11026_b200 import densenet
    from paper_2102_11026_b200.mcx import MCArray
    P, S = cfg1
    rng = np.random.default_rng(10 + order)
    B = 3
    x = rng.uniform(-0.5, 0.5, (1 << order, P.cfg.n_q, B))
    if order:
        x[1] *= 1e-10
    up = np.zeros((1 << order, P.model.N, B))
    up[0] = rng.standard_normal((P.model.N, B))
    got, grads = densenet.backward(P.rm.decoder, MCArray(x), MCArray(up), want_params=True)
    want, wg = on.backward(S.rm.D, x, up, want_params=True)
    for s in range(1 << order):
        assert rel(got.parts[s], want[s]) < 1e-11
    for (gW, gb), (wW, wb) in zip(grads, wg):
        gW = gW if order else gW[None]
        assert rel(gW, wW) < 1e-11


# ------------------------------------------------------------------ diffops
OPS = ["value", "jvp", "jacobian", "hvv", "hv", "svv", "vjp", "vhp"]


@pytest.mark.parametrize("mode", ["scaled", "multicomplex"])
@pytest.mark.parametrize("op", OPS)
def test_diffops_reduced_ctx(cfg1, op, mode):
    from paper_2102_11026_b200 import diffops
    P, S = cfg1
    q, qb, qdb, *_ = __import__("paper_2102_11026_b200.synth", fromlist=["x"]).random_state(P.cfg.n_p, P.cfg.n_q)
    v = q - qb
    a = np.random.default_rng(1).standard_normal(P.model.N)
    cfg = diffops.DiffConfig(mode=mode)
    args = {"value": (), "jacobian": (), "jvp": (v,), "hvv": (v,), "hv": (v,), "svv": (v,), "vjp": (a,), "vhp": (a,)}[op]
    got = getattr(diffops, op)(P.rm, q, *args, cfg=cfg)
    want = getattr(od, op)(S.rm.D, q, *args)
    tol = 1e-12 if mode == "scaled" else 1e-9
    assert rel(got, want) < tol


@pytest.mark.parametrize("op", ["jacobian", "hvv", "hv", "svv", "vjp", "vhp"])
def test_diffops_generic_densenet(cfg1, op):
    from paper_2102_11026_b200 import diffops
    P, S = cfg1
    rng = np.random.default_rng(4)
    q = rng.uniform(-0.5, 0.5, P.cfg.n_q)
    v = rng.uniform(-0.05, 0.05, P.cfg.n_q)
    a = rng.standard_normal(P.model.N)
    args = {"jacobian": (), "hvv": (v,), "hv": (v,), "svv": (v,), "vjp": (a,), "vhp": (a,)}[op]
    got = getattr(diffops, op)(P.rm.decoder, q, *args)
    want = getattr(od, op)(S.rm.D, q, *args)
    assert rel(got, want) < 1e-9


# ------------------------------------------------------------------ fused bundle pieces
def test_bundle_pieces(cfg1):
    from paper_2102_11026_b200 import rdsim, daereduce
    P, S = cfg1
    r, rb, rdb = P.random_state()
    q, qb, qdb = r[P.cfg.n_p:], rb[P.cfg.n_p:], rdb[P.cfg.n_p:]
    assert rel(daereduce.full_displacement(P.rm, r), orr.full_displacement(S.rm, r)) < TOL
    assert rel(daereduce.jtilde(P.rm, q), orr.jtilde(S.rm, q)) < TOL
    assert rel(rdsim.fictitious_force(P.rm, q, qb), ors.fictitious_force(S, q, qb)) < 1e-11
    for drop in (False, True):
        got = rdsim.delta_j(P.rm, q, qb, qdb, P.cfg.dt, drop_fict=drop)
        want = ors.delta_j(S, q, qb, qdb, P.cfg.dt, drop)
        assert rel(got, want) < 1e-11


def test_cubature_and_wnet(cfg1):
    from paper_2102_11026_b200 import neucubature, session
    P, S = cfg1
    r, _, _ = P.random_state()
    w_all = neucubature.wnet_forward(P.cm.wnet, P.rm, r)
    w_or = orr.wnet_forward(S.wnet, S.rm, r)
    assert rel(w_all, w_or) < TOL
    s = session.session_for(P.rm, P.model, P.cm)
    assert rel(s.wnet_forward_cub(r), w_or[P.cm.C]) < TOL
    u = orr.full_displacement(S.rm, r)
    Jt = orr.jtilde(S.rm, r[P.cfg.n_p:])
    for integ in ("cubature", "exact_sum"):
        f, K = neucubature.cubature_integrate(P.cm, P.rm, P.model, r, integ)
        if integ == "cubature":
            fo, Ko, _ = orr.cubature_integrate(S.model, S.rm, S.cub_elems, w_or[P.cm.C], u, Jt)
        else:
            fo, Ko, _ = orr.cubature_integrate(S.model, S.rm, np.arange(S.model.n_tets), np.ones(S.model.n_tets), u, Jt)
        assert rel(f, fo) < TOL and rel(K, Ko) < TOL


def test_elastic_gpu(cfg1):
    from paper_2102_11026_b200 import elastic
    P, S = cfg1
    u = 1e-3 * np.random.default_rng(6).standard_normal(P.model.N)
    assert rel(elastic.internal_force(P.model, u), oe.internal_force(S.model, u)) < TOL
    Kg = elastic.stiffness(P.model, u).toarray()
    assert rel(Kg, oe.stiffness_dense(S.model, u)) < TOL
    r, _, _ = P.random_state()
    e = [0, 7, 500]
    got = elastic.element_reduced_force(P.model, P.rm, r, e)
    for i, ei in enumerate(e):
        assert rel(got[i], orr.element_reduced_force(S.model, S.rm, r, ei)) < TOL


@pytest.mark.parametrize("integ", ["cubature", "exact_sum"])
@pytest.mark.parametrize("drop", [False, True])
def test_residual_and_system_jacobian(cfg1, integ, drop):
    from paper_2102_11026_b200 import rdsim
    from paper_2102_11026_b200.daereduce import ReducedState
    P, S = cfg1
    r, rb, rdb = P.random_state()
    cfg = rdsim.SimConfig(dt=P.cfg.dt, integration=integ, drop_fict=drop)
    st = ReducedState(rb, rdb, cfg.dt)
    phi = rdsim.residual(P.rm, P.model, st, P.f_ext, cfg, r=r)
    Sg = rdsim.system_jacobian(P.rm, P.model, st, P.f_ext, cfg, r=r)
    oc = ocfg(cfg)
    assert rel(phi, ors.residual(S, r, (rb, rdb), P.f_ext, oc)) < 1e-11
    assert rel(Sg, ors.system_jacobian(S, r, (rb, rdb), P.f_ext, oc)) < 1e-11


def test_cfg2_bundle_and_jacobian(cuda_ok):
    """Metric config (10-layer, width 256, n_q = 30): one Newton iteration's pieces."""
    from paper_2102_11026_b200.problem import build_problem
    from paper_2102_11026_b200 import rdsim
    from paper_2102_11026_b200.daereduce import ReducedState
    P = build_problem("cfg2")
    S = oracle_sim(P)
    r, rb, rdb = P.random_state()
    cfg = rdsim.SimConfig(dt=P.cfg.dt)
    st = ReducedState(rb, rdb, cfg.dt)
    oc = ocfg(cfg)
    assert rel(rdsim.residual(P.rm, P.model, st, P.f_ext, cfg, r=r), ors.residual(S, r, (rb, rdb), P.f_ext, oc)) < 1e-11
    assert rel(rdsim.system_jacobian(P.rm, P.model, st, P.f_ext, cfg, r=r),
               ors.system_jacobian(S, r, (rb, rdb), P.f_ext, oc)) < 1e-11


# ------------------------------------------------------------------ step and trajectories
def test_step_adaptive(cfg1):
    from paper_2102_11026_b200 import rdsim
    P, S = cfg1
    cfg = rdsim.SimConfig(dt=P.cfg.dt, newton_tol=1e-10)
    st = P.rest_state()
    ro, rdo = st.r.copy(), st.rdot.copy()
    for _ in range(5):
        st, (it, nrm) = rdsim.step(P.rm, P.model, st, P.f_ext, cfg, return_info=True)
        ro, rdo, ito, nro = ors.step(S, ro, rdo, P.f_ext, ocfg(cfg))
        assert it == ito and nrm <= cfg.newton_tol
        assert np.abs(st.r - ro).max() <= 1e-10 * max(np.abs(ro).max(), 1e-12) + 1e-14


@pytest.mark.parametrize("integ", ["cubature", "exact_sum"])
def test_trajectory_100_steps(cfg1, integ):
    """100-step trajectories, fixed-iteration mode (bitwise-comparable control flow)."""
    from paper_2102_11026_b200 import rdsim
    P, S = cfg1
    cfg = rdsim.SimConfig(dt=P.cfg.dt, integration=integ, fixed_iters=2)
    st = P.rest_state()
    ro, rdo = st.r.copy(), st.rdot.copy()
    worst = 0.0
    for _ in range(100):
        st = rdsim.step(P.rm, P.model, st, P.f_ext, cfg)
        ro, rdo, _, _ = ors.step(S, ro, rdo, P.f_ext, ocfg(cfg))
        worst = max(worst, np.abs(st.r - ro).max() / max(np.abs(ro).max(), 1e-30))
    assert worst <= 1e-9, worst


# ------------------------------------------------------------------ independent sims in one context
@pytest.mark.parametrize("batched", [False, True, "cpc", "noshare", "sharedcp"])
def test_multi_sim(cfg1, batched, monkeypatch):
    """n_sims independent simulations through one context == the single-sim oracle per sim.
    batched=True forces the big-tile per-layer GEMM path used for thousands of sims (cfg5);
    "cpc" runs the element-chunk cubature kernel (cub_chunked) with each CTA walking 4 element
    chunks of its sim (shared-memory Gram accumulation, prefetched rows, the 3-CTA/SM kernel);
    the other batched variants use the per-sim B-projected kernel (k_cub_sims) of cfg5."""
    from paper_2102_11026_b200 import rdsim
    from paper_2102_11026_b200.session import Session
    P, S = cfg1
    path = {False: None, True: "batched",
            # + the shared-real vhp backward (default only at >= 4 waves of CTAs), 4 element /
            # mass row chunks per cubature / mass CTA
            "cpc": "batched,cpc=4,shared_real,cpm=4,cub_chunked",
            "sharedcp": "batched,shared_real,bwd_cp",        # shared-real vhp on the cp.async GEMM
            "noshare": "batched,no_shared_real,hid_cp",      # 2 n_q dual columns; cp.async hidden layers
            }[batched]
    if path:
        monkeypatch.setenv("NLROM_PATH", path)
    ns = 3
    sess = Session(P.rm, P.model, P.cm, n_sims=ns)
    states = [P.random_state(seed=40 + i) for i in range(ns)]
    r, rb, rdb = (np.concatenate([s[j] for s in states]) for j in range(3))
    fext = np.tile(P.f_ext, ns)
    n = P.cfg.n_p + P.cfg.n_q
    for integ in ("cubature", "exact_sum"):
        for drop in (False, True):
            cfg = rdsim.SimConfig(dt=P.cfg.dt, integration=integ, drop_fict=drop)
            phi = sess.residual(r, rb, rdb, fext, cfg).reshape(ns, n)
            Sg = sess.system_jacobian(r, rb, rdb, fext, cfg)
            oc = ocfg(cfg)
            for i, (ri, rbi, rdbi) in enumerate(states):
                assert rel(phi[i], ors.residual(S, ri, (rbi, rdbi), P.f_ext, oc)) < 1e-11, (integ, drop, i)
                assert rel(Sg[i], ors.system_jacobian(S, ri, (rbi, rdbi), P.f_ext, oc)) < 1e-11, (integ, drop, i)
    # fixed-iteration steps from rest under per-sim load scales
    cfg = rdsim.SimConfig(dt=P.cfg.dt, fixed_iters=2)
    scales = [1.0, 0.5, 2.0]
    fs = np.concatenate([s * P.f_ext for s in scales])
    st = P.rest_state()
    rb = np.tile(st.r, ns)
    rdb = np.tile(st.rdot, ns)
    for _ in range(3):
        rb, rdb, _, _ = sess.step(rb, rdb, fs, cfg)
    for i, s in enumerate(scales):
        ro, rdo = st.r.copy(), st.rdot.copy()
        for _ in range(3):
            ro, rdo, _, _ = ors.step(S, ro, rdo, s * P.f_ext, ocfg(cfg))
        assert np.abs(rb.reshape(ns, n)[i] - ro).max() <= 1e-10 * np.abs(ro).max(), i


# ------------------------------------------------------------------ cfg3 corners (latent-dim x depth sweep)
@pytest.mark.parametrize("n_q,L,n_p", [(5, 4, 30), (64, 16, 30), (48, 6, 30), (64, 4, 60), (10, 5, 30)])
def test_cfg3_corners(cuda_ok, n_q, L, n_p):
    """cfg2 mesh with n_q in 5..64 and depth 4..16 (fused-chain and LU size limits)."""
    from paper_2102_11026_b200.problem import build_problem
    from paper_2102_11026_b200 import rdsim
    from paper_2102_11026_b200.daereduce import ReducedState
    P = build_problem("cfg2", n_q=n_q, n_fc=L, n_p=n_p)   # n = 124 exercises the widest LU block
    S = oracle_sim(P)
    r, rb, rdb = P.random_state()
    cfg = rdsim.SimConfig(dt=P.cfg.dt)
    st = ReducedState(rb, rdb, cfg.dt)
    oc = ocfg(cfg)
    assert rel(rdsim.residual(P.rm, P.model, st, P.f_ext, cfg, r=r), ors.residual(S, r, (rb, rdb), P.f_ext, oc)) < 1e-11
    assert rel(rdsim.system_jacobian(P.rm, P.model, st, P.f_ext, cfg, r=r),
               ors.system_jacobian(S, r, (rb, rdb), P.f_ext, oc)) < 1e-11
    cfgf = rdsim.SimConfig(dt=P.cfg.dt, fixed_iters=2)
    st0 = P.rest_state()
    got = rdsim.step(P.rm, P.model, st0, P.f_ext, cfgf)
    ro, _, _, _ = ors.step(S, st0.r.copy(), st0.rdot.copy(), P.f_ext, ocfg(cfgf))
    assert np.abs(got.r - ro).max() <= 1e-10 * np.abs(ro).max()


def test_loaded_artifacts_same_device_results(cfg1, tmp_path):
    """A ReducedModel / CubatureModel / mesh written and read back drive the GPU path to the
    bitwise-identical residual and system Jacobian."""
    from paper_2102_11026_b200 import artifacts as io, rdsim
    from paper_2102_11026_b200.daereduce import ReducedState
    from paper_2102_11026_b200.elastic import ElasticModel
    P, S = cfg1
    io.save_reduced_model(P.rm, str(tmp_path / "rm"))
    io.save_cubature_model(P.cm, str(tmp_path / "cm"))
    io.write_mesh(P.model.mesh, str(tmp_path / "mesh.txt"))
    rm2 = io.load_reduced_model(str(tmp_path / "rm"))
    cm2 = io.load_cubature_model(str(tmp_path / "cm"))
    model2 = ElasticModel(io.read_mesh(str(tmp_path / "mesh.txt")), P.model.material, P.data["fixed"])
    rm2.attach(model2, cm2)
    r, rb, rdb = P.random_state()
    cfg = rdsim.SimConfig(dt=P.cfg.dt)
    st = ReducedState(rb, rdb, cfg.dt)
    a = rdsim.residual(P.rm, P.model, st, P.f_ext, cfg, r=r)
    b = rdsim.residual(rm2, model2, st, P.f_ext, cfg, r=r)
    assert np.array_equal(a, b)
    assert np.array_equal(rdsim.system_jacobian(P.rm, P.model, st, P.f_ext, cfg, r=r),
                          rdsim.system_jacobian(rm2, model2, st, P.f_ext, cfg, r=r))


_VARIANT_SCRIPT = r"""
import sys, numpy as np
sys.path.insert(0, sys.argv[1])
from paper_2102_11026_b200.problem import build_problem
from paper_2102_11026_b200 import rdsim
from paper_2102_11026_b200.daereduce import ReducedState
P = build_problem("cfg2", n_fc=4)
r, rb, rdb = P.random_state()
cfg = rdsim.SimConfig(dt=P.cfg.dt)
st = ReducedState(rb, rdb, cfg.dt)
phi = rdsim.residual(P.rm, P.model, st, P.f_ext, cfg, r=r)
S = rdsim.system_jacobian(P.rm, P.model, st, P.f_ext, cfg, r=r)
st0 = P.rest_state()
nxt = rdsim.step(P.rm, P.model, st0, P.f_ext, rdsim.SimConfig(dt=P.cfg.dt, fixed_iters=2))
np.savez(sys.argv[2], phi=phi, S=S, r=nxt.r)
"""


@pytest.mark.parametrize("env", [
    {"NLROM_PATH": "unfused"},
    {"NLROM_PATH": "unfused,tangents=7"},
    {"NLROM_PATH": "batched,tangents=1"},
])
def test_kernel_variants(cuda_ok, env, tmp_path):
    """Alternate code paths (NLROM_PATH, read at context creation, hence a fresh process)
    against the oracle: unfused per-layer GEMMs instead of the cluster chains, other jet group
    sizes, the batched kernels at one sim."""
    import os
    import subprocess
    import sys
    from paper_2102_11026_b200.problem import build_problem
    from paper_2102_11026_b200.rdsim import SimConfig
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = str(tmp_path / "v.npz")
    e = dict(os.environ, **env)
    subprocess.run([sys.executable, "-c", _VARIANT_SCRIPT, root, out], env=e, check=True, timeout=600)
    got = np.load(out)
    P = build_problem("cfg2", n_fc=4)
    S = oracle_sim(P)
    r, rb, rdb = P.random_state()
    oc = ocfg(SimConfig(dt=P.cfg.dt))
    assert rel(got["phi"], ors.residual(S, r, (rb, rdb), P.f_ext, oc)) < 1e-11
    assert rel(got["S"], ors.system_jacobian(S, r, (rb, rdb), P.f_ext, oc)) < 1e-11
    st0 = P.rest_state()
    ro, _, _, _ = ors.step(S, st0.r.copy(), st0.rdot.copy(), P.f_ext,
                           ocfg(SimConfig(dt=P.cfg.dt, fixed_iters=2)))
    assert np.abs(got["r"] - ro).max() <= 1e-10 * np.abs(ro).max()


@pytest.mark.parametrize("n_p", [1, 2])
def test_step_small_linear_block(cuda_ok, n_p):
    """Few linear modes: the first pivots fall in the nonlinear block, whose vhp term the LU adds
    while staging (regression: the first pivot row must carry it)."""
    from paper_2102_11026_b200.problem import build_problem
    from paper_2102_11026_b200 import rdsim
    P = build_problem("tiny", n_p=n_p)
    S = oracle_sim(P)
    cfg = rdsim.SimConfig(dt=P.cfg.dt, fixed_iters=3)
    r, rb, rdb = P.random_state()
    from paper_2102_11026_b200.daereduce import ReducedState
    st = ReducedState(rb, rdb, cfg.dt)
    got = rdsim.step(P.rm, P.model, st, P.f_ext, cfg)
    ro, _, _, _ = ors.step(S, rb.copy(), rdb.copy(), P.f_ext, ocfg(cfg))
    # far from the solution (|dr| ~ 1) with cond(S) ~ 1e5: roundoff of the two LU orders grows
    assert np.abs(got.r - ro).max() <= 1e-8 * np.abs(ro).max()


@pytest.mark.parametrize("problem", ["cfg1", "tiny"])
def test_stale_shared_memory(problem):
    """Kernels must not read shared memory they never wrote: every SM's shared memory is
    filled with NaN before each call (regression: the vhp chain's K-padding rows at w = 40)."""
    from paper_2102_11026_b200 import _lib, rdsim
    from paper_2102_11026_b200.problem import build_problem
    from paper_2102_11026_b200.session import Session
    P = build_problem(problem)
    S = oracle_sim(P)
    L = _lib.lib()
    poison = lambda: _lib.check(L.nlrom_debug_poison_shared_memory(0), lambda: b"poison")
    ns = 3
    sess = Session(P.rm, P.model, P.cm, n_sims=ns)
    n = P.cfg.n_p + P.cfg.n_q
    states = [P.random_state(seed=60 + i) for i in range(ns)]
    r, rb, rdb = (np.concatenate([s[j] for s in states]) for j in range(3))
    fext = np.tile(P.f_ext, ns)
    cfg = rdsim.SimConfig(dt=P.cfg.dt)
    poison()
    Sg = sess.system_jacobian(r, rb, rdb, fext, cfg)
    for i, (ri, rbi, rdbi) in enumerate(states):
        assert rel(Sg[i], ors.system_jacobian(S, ri, (rbi, rdbi), P.f_ext, ocfg(cfg))) < 1e-11, i
    cfg = rdsim.SimConfig(dt=P.cfg.dt, fixed_iters=2)
    for k in range(2):
        poison()
        r1, rd1, _, _ = sess.step(rb, rdb, fext, cfg)
        for i, (ri, rbi, rdbi) in enumerate(states):
            ro, _, _, _ = ors.step(S, rbi, rdbi, P.f_ext, ocfg(cfg))
            assert np.abs(r1.reshape(ns, n)[i] - ro).max() <= 1e-10 * np.abs(ro).max(), (k, i)


# ------------------------------------------------------------------ neural-cubature training set
def test_build_train_set(cfg1):
    """Per-element reduced forces of all elements at training poses (GPU k_cubature, per-element
    projection) vs the oracle restatement."""
    from oracle import cubature_train as oct_
    from paper_2102_11026_b200 import cubature_train as ct
    P, S = cfg1
    rng = np.random.default_rng(11)
    rs = rng.uniform(-0.3, 0.3, (3, P.cfg.n_p + P.cfg.n_q))
    ts = ct.build_train_set(P.rm, P.model, rs)
    f, F, u = oct_.train_arrays(S.model, S.rm, rs)
    assert ts.F.shape == F.shape
    for s in range(3):
        assert rel(ts.F[s], F[s]) < 1e-11 and rel(ts.f[s], f[s]) < 1e-11 and rel(ts.u[s], u[s]) < 1e-12
    C, w = ct.greedy_cubature(P.rm, P.model, ts, 10)
    Co, wo = oct_.greedy(f, F, 10)
    assert list(C) == list(Co) and np.allclose(w, wo, rtol=1e-7, atol=1e-10)
