"""Oracle substructured scene: k DAE strings attached to a translating core (TEST INFRASTRUCTURE).

The reference has no coupled scenes; the puffer ball
couples 320 identical strings, each with its own n_p + n_q subspace and shared networks.
SURVEY.md §8e proposes star-topology substructuring; this module is the builder-defined
model the GPU path must reproduce, restated densely (one global LU-pp solve per Newton
iteration, no Schur complement) so it is independent of the sharded product algorithm.

World position of string s's free vertices: x_s = X_s + R_s u_s(r_s) + T c, with R_s a
fixed rotation (string frame -> world), u_s = U p + D(q) the string's local displacement
(base face fixed in the string frame) and c the core translation; T stacks I_3 per vertex.
The elastic energy of a string depends on u_s only, so c enters through inertia alone.
Implicit Euler in the paper's reduced form (Eq. 10, oracle/rdsim.py) with mass-proportional
damping applied to the world motion, h = dt, ah = alpha h:

  Dc   = (1 + ah)(c - c_bar) - h cdot_bar                        (core "inertia argument")
  c_s  = (1 + ah)(r_s - r_bar_s) - h rdot_bar_s
  a_s  = M J~_s c_s + f_fict,s + M T R_s^T Dc + h^2 (f_int,s - R_s^T f_ext,s)
  phi_s = J~_s^T a_s                                            == rdsim.residual with
          f_eff,s = R_s^T f_ext,s - M T R_s^T Dc / h^2          (coupling = effective load)
  phi_c = (m_c + sum_s m_s) Dc + sum_s R_s (K_s c_s + t_s)
          + h^2 (k_c c - f_c - sum_s T^T f_ext,s)
  K_s  = T^T M J~_s (3 x n),  t_s = T^T f_fict,s,  m_s = string mass

Newton matrix (arrowhead), the Eq. 11 approximation d(M J~ c + f_fict)/dr = M[(1+ah)U,
(1+ah)J + dJ] used for the string blocks (rdsim.system_jacobian) and for the core row:

  d phi_s / d r_s = rdsim.system_jacobian(..., f_eff,s)
  d phi_s / d c   = C_s = (1 + ah) K_s^T R_s^T                  (n x 3)
  d phi_c / d r_s = E_s = R_s ((1 + ah) K_s + [0, T^T M dJ_s])   (3 x n)
  d phi_c / d c   = Z   = ((1 + ah)(m_c + sum_s m_s) + h^2 k_c) I_3

step: Newton on x = [r_1 .. r_k, c] with predictor x_bar + h xdot_bar, dense LU-pp,
halving line search on ||[phi_1 .. phi_k, phi_c]||_2 (same control flow as rdsim.step).
``step_sharded`` is the distributed restatement (Schur complement onto the core, one
allreduce of 16 doubles per Newton iteration) used by the CPU gloo tests.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import scipy.linalg

from . import rdsim as ors
from .reduced import split, jtilde
from . import diffops


@dataclass
class OScene:
    sim: ors.OSim              # the shared string model (one training re-used)
    R: np.ndarray              # (k, 3, 3) string frame -> world
    f_world: np.ndarray        # (k, N) external load on the free DOFs, world frame
    m_core: float = 1.0
    k_core: float = 0.0
    f_core: np.ndarray = None  # (3,)

    def __post_init__(self):
        self.R = np.asarray(self.R, dtype=float)
        self.f_world = np.asarray(self.f_world, dtype=float)
        self.f_core = np.zeros(3) if self.f_core is None else np.asarray(self.f_core, dtype=float)

    @property
    def k(self):
        return self.R.shape[0]

    @property
    def m_string(self):
        return float(self.sim.model.mass[0::3].sum())


def axis_sums(v):
    """T^T v for a free-DOF vector / matrix (rows = xyz-interleaved DOFs): (3, ...)."""
    v = np.asarray(v)
    return np.stack([v[d::3].sum(axis=0) for d in range(3)])


def to_local(R, v):
    """R^T applied per vertex to an xyz-interleaved free-DOF vector."""
    return (np.asarray(v).reshape(-1, 3) @ R).reshape(-1)


def core_delta(scene, c, c_bar, cdot_bar, h):
    return (1.0 + scene.sim.alpha * h) * (np.asarray(c) - c_bar) - h * np.asarray(cdot_bar)


def string_terms(scene, s, r, state_s, Dc, cfg, want_jac):
    """Per-string pieces: phi_s, the core-row contribution, and (want_jac) S_s, C_s, E_s."""
    sim, h = scene.sim, cfg.dt
    ah = sim.alpha * h
    m = sim.model.mass
    R = scene.R[s]
    d = R.T @ Dc
    f_eff = to_local(R, scene.f_world[s]) - m * np.tile(d, m.size // 3) / (h * h)
    phi = ors.residual(sim, r, state_s, f_eff, cfg)
    p, q = split(sim.rm, r)
    J = diffops.jacobian(sim.rm.D, q, cfg.eps)
    Jt = jtilde(sim.rm, q, J)
    K = axis_sums(m[:, None] * Jt)                                  # (3, n)
    t = np.zeros(3)
    if not cfg.drop_fict:
        q_bar = state_s[0][sim.rm.n_p:]
        t = axis_sums(ors.fictitious_force(sim, q, q_bar, cfg.eps))
    cs = (1.0 + ah) * (np.asarray(r) - state_s[0]) - h * state_s[1]
    core = scene.m_string * Dc + R @ (K @ cs + t) - h * h * axis_sums(scene.f_world[s])
    if not want_jac:
        return phi, core
    S = ors.system_jacobian(sim, r, state_s, f_eff, cfg)
    q_bar = state_s[0][sim.rm.n_p:]
    qdot_bar = state_s[1][sim.rm.n_p:]
    dJ = ors.delta_j(sim, q, q_bar, qdot_bar, h, cfg.drop_fict, cfg.eps)
    TMdJ = axis_sums(m[:, None] * dJ)                               # (3, n_q)
    C = (1.0 + ah) * K.T @ R.T                                      # (n, 3)
    E = R @ ((1.0 + ah) * K + np.concatenate([np.zeros((3, sim.rm.n_p)), TMdJ], axis=1))
    return phi, core, S, C, E


def core_terms(scene, c, Dc, h):
    """Core-only part of phi_c and the core diagonal block Z."""
    ah = scene.sim.alpha * h
    mt = scene.m_core + scene.k * scene.m_string
    part = scene.m_core * Dc + h * h * (scene.k_core * np.asarray(c) - scene.f_core)
    Z = ((1.0 + ah) * mt + h * h * scene.k_core) * np.eye(3)
    return part, Z


def residual(scene, rs, c, state, cfg):
    """(phi_s (k, n), phi_c (3)); state = (r_bar (k,n), rdot_bar (k,n), c_bar, cdot_bar)."""
    rb, rdb, cb, cdb = state
    h = cfg.dt
    Dc = core_delta(scene, c, cb, cdb, h)
    phis = []
    phic, _ = core_terms(scene, c, Dc, h)
    for s in range(scene.k):
        ph, core = string_terms(scene, s, rs[s], (rb[s], rdb[s]), Dc, cfg, want_jac=False)
        phis.append(ph)
        phic = phic + core
    return np.array(phis), phic


def jacobian(scene, rs, c, state, cfg):
    """Dense (k n + 3)^2 Newton matrix of the arrowhead system."""
    rb, rdb, cb, cdb = state
    h = cfg.dt
    Dc = core_delta(scene, c, cb, cdb, h)
    n = rs.shape[1]
    k = scene.k
    A = np.zeros((k * n + 3, k * n + 3))
    _, Z = core_terms(scene, c, Dc, h)
    A[k * n:, k * n:] = Z
    for s in range(k):
        _, _, S, C, E = string_terms(scene, s, rs[s], (rb[s], rdb[s]), Dc, cfg, want_jac=True)
        A[s * n:(s + 1) * n, s * n:(s + 1) * n] = S
        A[s * n:(s + 1) * n, k * n:] = C
        A[k * n:, s * n:(s + 1) * n] = E
    return A


def _norm(phis, phic):
    return float(np.sqrt(np.sum(phis * phis) + phic @ phic))


def step(scene, r_bar, rdot_bar, c_bar, cdot_bar, cfg):
    """One coupled implicit timestep. Returns (r, rdot, c, cdot, iters, ||phi||)."""
    r_bar = np.asarray(r_bar, dtype=float)
    rdot_bar = np.asarray(rdot_bar, dtype=float)
    c_bar = np.asarray(c_bar, dtype=float)
    cdot_bar = np.asarray(cdot_bar, dtype=float)
    state = (r_bar, rdot_bar, c_bar, cdot_bar)
    h = cfg.dt
    k, n = r_bar.shape
    rs = r_bar + h * rdot_bar
    c = c_bar + h * cdot_bar

    def solve(rs, c, phis, phic):
        A = jacobian(scene, rs, c, state, cfg)
        dx = scipy.linalg.lu_solve(scipy.linalg.lu_factor(A), -np.concatenate([phis.reshape(-1), phic]))
        return dx[:k * n].reshape(k, n), dx[k * n:]

    phis, phic = residual(scene, rs, c, state, cfg)
    if cfg.fixed_iters is not None:
        for _ in range(cfg.fixed_iters):
            dr, dc = solve(rs, c, phis, phic)
            rs, c = rs + dr, c + dc
            phis, phic = residual(scene, rs, c, state, cfg)
        return rs, (rs - r_bar) / h, c, (c - c_bar) / h, cfg.fixed_iters, _norm(phis, phic)
    nrm = _norm(phis, phic)
    it = 0
    while nrm > cfg.newton_tol:
        if it >= cfg.max_iters:
            raise ors.NewtonDivergence(f"Newton did not converge in {cfg.max_iters} iterations; "
                                       f"last residual norm {nrm:.3e}", nrm)
        dr, dc = solve(rs, c, phis, phic)
        t = 1.0
        for _ in range(11):
            r_try, c_try = rs + t * dr, c + t * dc
            phis_t, phic_t = residual(scene, r_try, c_try, state, cfg)
            n_try = _norm(phis_t, phic_t)
            if not cfg.line_search or n_try < nrm:
                break
            t *= 0.5
        rs, c, phis, phic, nrm = r_try, c_try, phis_t, phic_t, n_try
        it += 1
    return rs, (rs - r_bar) / h, c, (c - c_bar) / h, it, nrm


# ----------------------------------------------------------------------------- sharded restatement
def shard(k, rank, world):
    """Contiguous string ranges per rank (the product's partition, paper_2102_11026_b200/substructure.py)."""
    return rank * k // world, (rank + 1) * k // world


def step_sharded(scene, r_bar, rdot_bar, c_bar, cdot_bar, cfg, rank, world, allreduce):
    """Fixed-iteration coupled step with strings [lo, hi) on this rank; ``allreduce(np.ndarray)``
    sums a float64 vector over ranks. Per Newton iteration: X_s = S_s^{-1}[C_s | phi_s] locally,
    one allreduce of [sum E_s X_s (12) | core contributions (3) | sum ||phi_s||^2 (1)], the 3 x 3
    core solve replicated on every rank, then dr_s = -X_s[:, 3] - X_s[:, :3] dc locally."""
    assert cfg.fixed_iters is not None
    lo, hi = shard(scene.k, rank, world)
    h = cfg.dt
    r_bar = np.asarray(r_bar, dtype=float)
    rdot_bar = np.asarray(rdot_bar, dtype=float)
    rs = (r_bar + h * rdot_bar)[lo:hi].copy()
    c = np.asarray(c_bar, dtype=float) + h * np.asarray(cdot_bar, dtype=float)
    nrm = None
    for it in range(cfg.fixed_iters + 1):
        Dc = core_delta(scene, c, c_bar, cdot_bar, h)
        part = np.zeros(16)
        X = []
        for i, s in enumerate(range(lo, hi)):
            st = (r_bar[s], rdot_bar[s])
            if it < cfg.fixed_iters:
                phi, core, S, C, E = string_terms(scene, s, rs[i], st, Dc, cfg, want_jac=True)
                Xs = scipy.linalg.lu_solve(scipy.linalg.lu_factor(S), np.concatenate([C, phi[:, None]], axis=1))
                part[:12] += (E @ Xs).reshape(-1)
                X.append(Xs)
            else:
                phi, core = string_terms(scene, s, rs[i], st, Dc, cfg, want_jac=False)
            part[12:15] += core
            part[15] += phi @ phi
        tot = allreduce(part)
        cpart, Z = core_terms(scene, c, Dc, h)
        phic = cpart + tot[12:15]
        nrm = float(np.sqrt(tot[15] + phic @ phic))
        if it == cfg.fixed_iters:
            break
        A = tot[:12].reshape(3, 4)
        dc = np.linalg.solve(Z - A[:, :3], -phic + A[:, 3])
        for i in range(hi - lo):
            rs[i] = rs[i] - X[i][:, 3] - X[i][:, :3] @ dc
        c = c + dc
    return rs, (rs - r_bar[lo:hi]) / h, c, (c - np.asarray(c_bar)) / h, nrm
