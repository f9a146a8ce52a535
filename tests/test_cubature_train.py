"""Neural-cubature training row: Lawson-Hanson NNLS vs scipy, the greedy
baseline vs the oracle restatement, the Table 2 error metric, the selection GCN (SPEC.md:596-602
examples), farthest-point initialisation and the alternating trainer. CPU:
training sets come from the oracle's per-element reduced forces; the GPU builder is checked
against them in test_gpu_parity.py::test_build_train_set."""

from types import SimpleNamespace

import numpy as np
import pytest
from scipy.optimize import nnls as scipy_nnls

from helpers import oracle_sim
from oracle import cubature_train as oct_
from paper_2102_11026_b200 import cubature_train as ct


@pytest.fixture(scope="module")
def tiny_ts():
    from paper_2102_11026_b200.problem import build_problem
    P = build_problem("tiny")
    S = oracle_sim(P)
    rng = np.random.default_rng(7)
    n = P.cfg.n_p + P.cfg.n_q
    rs = rng.uniform(-0.3, 0.3, (6, n))
    f, F, u = oct_.train_arrays(S.model, S.rm, rs)
    return P, S, ct.CubatureTrainSet(rs, f, F, u)


@pytest.mark.parametrize("seed", range(12))
def test_nnls_matches_scipy(seed):
    rng = np.random.default_rng(seed)
    m, k = rng.integers(5, 40), rng.integers(1, 25)
    A = rng.standard_normal((m, k))
    if seed % 3 == 0:
        A[:, -1] = A[:, 0]  # rank deficient
    b = rng.standard_normal(m)
    x, rn = ct.nnls(A, b)
    xs, rns = scipy_nnls(A, b)
    assert np.all(x >= 0)
    assert abs(rn - rns) <= 1e-9 * max(1.0, rns)
    if seed % 3:
        assert np.allclose(x, xs, atol=1e-9)


def test_greedy_toy_two_elements():
    """target 1 on a 2-element toy where one element carries all force."""
    F = np.zeros((3, 2, 4))
    F[:, 1] = np.random.default_rng(0).standard_normal((3, 4))
    ts = ct.CubatureTrainSet(np.zeros((3, 4)), F.sum(1), F, np.zeros((3, 6)))
    C, w = ct.greedy_cubature(None, None, ts, 1)
    assert list(C) == [1] and np.allclose(w, [1.0])
    assert ct.cubature_error(ts, C, w) < 1e-14


def test_greedy_matches_oracle_and_is_monotone(tiny_ts):
    P, S, ts = tiny_ts
    errs = []
    for size in (2, 4, 8, 16):
        C, w = ct.greedy_cubature(P.rm, P.model, ts, size)
        Co, wo = oct_.greedy(ts.f, ts.F, size)
        assert list(C) == list(Co)
        assert np.allclose(w, wo, rtol=1e-9, atol=1e-12) and np.all(w >= 0)
        errs.append(ct.cubature_error(ts, C, w))
    assert all(b <= a + 1e-12 for a, b in zip(errs, errs[1:])), errs


def test_cubature_error_identity_and_empty(tiny_ts):
    _, _, ts = tiny_ts
    T = ts.n_elems
    assert ct.cubature_error(ts, np.arange(T), np.ones(T)) < 1e-12
    assert ct.cubature_error(ts, [], []) == 1.0


def _toy_model(perm=None):
    from paper_2102_11026_b200.problem import build_problem
    P = build_problem("tiny")
    verts, tets = np.asarray(P.model.mesh.vertices), np.asarray(P.model.mesh.tets)
    vd = np.asarray(P.model.vert_dof)
    if perm is None:
        return SimpleNamespace(mesh=SimpleNamespace(vertices=verts, tets=tets), vert_dof=vd), P
    inv = np.argsort(perm)  # new id of old vertex v is inv[v]
    return SimpleNamespace(mesh=SimpleNamespace(vertices=verts[perm], tets=inv[tets]), vert_dof=vd[perm]), P


def test_snet_scores_are_a_distribution():
    m, P = _toy_model()
    g = ct.mesh_graph(m)
    u = np.random.default_rng(1).standard_normal(P.model.N) * 0.1
    s = ct.snet_forward(ct.SelectionNet.init(3), g, u)
    assert s.shape == (len(m.mesh.tets),) and np.all(s >= 0) and abs(s.sum() - 1) < 1e-10
    z = ct.snet_forward(ct.SelectionNet.zeros(), g, u)
    assert np.allclose(z, 1.0 / z.size, atol=1e-15)


def test_snet_vertex_permutation_equivariance():
    """permuting vertex ids and the graph consistently leaves element scores unchanged
    (elements keep their order)."""
    m0, P = _toy_model()
    perm = np.random.default_rng(5).permutation(len(m0.mesh.vertices))
    m1, _ = _toy_model(perm)
    u = np.random.default_rng(2).standard_normal(P.model.N) * 0.1
    net = ct.SelectionNet.init(4)
    s0 = ct.snet_forward(net, ct.mesh_graph(m0), u)
    s1 = ct.snet_forward(net, ct.mesh_graph(m1), u)
    assert np.allclose(s0, s1, rtol=1e-12, atol=1e-15)


def test_farthest_point_and_select_topk():
    _, P = _toy_model()
    C = ct.farthest_point_elements(P.model, 5, seed=0)
    assert len(set(C.tolist())) == 5
    from paper_2102_11026_b200.neucubature import select_topk
    s = np.zeros(P.model.n_tets)
    s[[3, 7, 9]] = [0.5, 0.5, 0.2]
    C2 = select_topk([7], s, 2)
    assert list(C2) == [7, 3, 9]  # already-selected never re-added; ties by lower id


def test_train_alternating(tiny_ts):
    P, S, ts = tiny_ts
    cm0 = ct.train_alternating(P.rm, P.model, ts, K=2, rounds=0, wnet=P.cm.wnet, n_init=3, device="cpu")
    assert list(cm0.C) == list(ct.farthest_point_elements(P.model, 3, 0))
    cm, log = ct.train_alternating(P.rm, P.model, ts, K=2, rounds=3, wnet=P.cm.wnet, n_init=3, epochs=15,
                                   lr=1e-2, device="cpu", return_log=True)
    assert log.sizes == [5, 7, 9] and len(set(cm.C.tolist())) == 9
    assert all(np.isfinite(log.loss_w)) and all(np.isfinite(log.loss_s))
    # the trained W is a drop-in weight net: nonnegative weights for every element
    from oracle import nets as on
    from paper_2102_11026_b200 import synth
    Ws = [cm.wnet.weights[i] for i, L in enumerate(cm.wnet.layers) if L.kind == "fully_connected"]
    bs = [cm.wnet.biases[i] for i, L in enumerate(cm.wnet.layers) if L.kind == "fully_connected"]
    w = on.forward(synth.wnet_layers(Ws, bs), ts.u[0][None, :, None])[0, :, 0]
    assert w.shape == (ts.n_elems,) and np.all(w >= 0)
