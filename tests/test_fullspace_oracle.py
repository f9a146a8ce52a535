"""Oracle full-space integrator and pose generator against the
SPEC's examples, plus the host-side posegen pieces of the product (no GPU)."""

import numpy as np
import pytest

from oracle import elastic as oe, fullspace as ofs
from paper_2102_11026_b200 import synth


def _model(nx=4, ny=2, nz=2, alpha=0.1, young=5e5):
    verts, tets, fixed = synth.box_mesh(nx, ny, nz)
    return oe.OModel(verts, tets, fixed, young, 0.45, 1000.0, alpha)


def test_rest_is_fixed_point():
    """f_ext = 0, u = v = 0 -> state unchanged, zero Newton iterations."""
    m = _model()
    u, v, it, gn = ofs.fullspace_step(m, np.zeros(m.N), np.zeros(m.N), np.zeros(m.N), 1 / 60)
    assert it == 0 and gn == 0.0 and not u.any() and not v.any()


def test_energy_decays_with_damping():
    """alpha > 0, f_ext = 0: total (kinetic + elastic) energy decays monotonically."""
    m = _model(alpha=2.0)
    rng = np.random.default_rng(0)
    u = np.zeros(m.N)
    v = 0.05 * rng.standard_normal(m.N)
    e_prev = np.inf
    for _ in range(12):
        u, v, _, _ = ofs.fullspace_step(m, u, v, np.zeros(m.N), 1 / 60)
        e = 0.5 * np.sum(m.mass * v * v) + oe.stvk_energy(m, u)
        assert e < e_prev
        e_prev = e


def test_static_sag_force_balance():
    """Gravity on a clamped bar settles to a static sag: f_int = f_ext."""
    m = _model(alpha=30.0, young=5e6)
    f = synth.gravity(m.mass)
    u, v = np.zeros(m.N), np.zeros(m.N)
    for _ in range(300):
        u, v, _, _ = ofs.fullspace_step(m, u, v, f, 1 / 30, newton_tol=1e-11)
    res = np.linalg.norm(oe.internal_force(m, u) - f) / np.linalg.norm(f)
    assert res <= 1e-8 and u[1::3].min() < 0


def test_newton_matrix_matches_finite_differences():
    """The Newton step uses K = d f_int / du: central differences of f_int agree."""
    m = _model()
    rng = np.random.default_rng(1)
    u = 1e-2 * rng.standard_normal(m.N)
    _, K = ofs.stiffness_sparse(m, u)
    d = rng.standard_normal(m.N)
    h = 1e-6
    fd = (oe.internal_force(m, u + h * d) - oe.internal_force(m, u - h * d)) / (2 * h)
    assert np.abs(K @ d - fd).max() <= 1e-6 * np.abs(fd).max()


def test_surface_and_plan_match_product():
    """Product posegen host logic (surface vertices, episode plan) == oracle restatement."""
    from paper_2102_11026_b200 import posegen
    from paper_2102_11026_b200.elastic import ElasticModel, Material, TetMesh
    verts, tets, fixed = synth.box_mesh(5, 2, 2)
    assert np.array_equal(posegen.surface_vertices(tets), ofs.surface_vertices(tets))
    assert np.array_equal(posegen.surface_vertices(np.array([[0, 1, 2, 3]])), np.arange(4))
    pm = ElasticModel(TetMesh(verts, tets), Material(), fixed)
    om = oe.OModel(verts, tets, fixed, 5e5, 0.45, 1000.0, 0.1)
    sc = posegen.ForceScript(seed=7, episodes=4, radius=0.15, magnitude=(1.0, 5.0), steps=2)
    got = posegen._plan(pm, sc)
    want = ofs.episode_plan(om.verts, om.tets, om.fixed, 7, 4, 0.15, (1.0, 5.0))
    for (gi, gf), (wi, wf) in zip(got, want):
        assert np.array_equal(gi, wi) and np.array_equal(gf, wf)
        assert np.array_equal(posegen._load(pm, gi, gf), ofs.episode_force(om, wi, wf))


def test_energy_weights_examples():
    """SPEC.md:409-412."""
    from paper_2102_11026_b200.posegen import PoseSet, energy_weights
    ps = PoseSet(np.zeros((3, 4)), np.full(4, 2.0))
    assert np.allclose(energy_weights(ps, 1e-6), 1.0)
    e = np.array([1e-9, 1.0, 2.0, 4.0])
    w = energy_weights(PoseSet(np.zeros((3, 4)), e), 1e-3)
    assert np.argmax(w) == 0 and np.isclose(w.mean(), 1.0)
    w2 = energy_weights(PoseSet(np.zeros((3, 4)), 2 * e), 2e-3)
    assert np.allclose(w2, w)
    with pytest.raises(ValueError):
        energy_weights(ps, 0.0)


def test_pca_basis_examples():
    """one-vector poses, orthonormality, monotone reconstruction error."""
    from paper_2102_11026_b200.posegen import PoseSet, pca_basis
    rng = np.random.default_rng(3)
    a = rng.standard_normal(20)
    ps = PoseSet(np.outer(a, [1.0, -2.0, 3.0]), np.array([1.0, 2.0, 3.0]))
    U = pca_basis(ps, 1, 3)
    assert abs(abs(U[:, 0] @ a) / np.linalg.norm(a) - 1.0) <= 1e-12
    with pytest.raises(ValueError):
        pca_basis(ps, 2, 3)  # rank deficient
    X = rng.standard_normal((30, 12))
    ps = PoseSet(X, rng.uniform(0, 1, 12))
    errs = []
    for n_p in range(1, 8):
        U = pca_basis(ps, n_p, 10)
        assert np.abs(U.T @ U - np.eye(n_p)).max() <= 1e-10
        idx = np.argsort(ps.energies, kind="stable")[:10]
        errs.append(np.linalg.norm(X[:, idx] - U @ (U.T @ X[:, idx])))
    assert all(e1 >= e2 - 1e-12 for e1, e2 in zip(errs, errs[1:]))
    Uo, _ = ofs.pca_basis(X, ps.energies, 4, 10)
    assert np.abs(np.abs(Uo.T @ pca_basis(ps, 4, 10)) - np.eye(4)).max() <= 1e-10
