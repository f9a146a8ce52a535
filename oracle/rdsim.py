"""Oracle reduced implicit-Euler Newton integrator (TEST INFRASTRUCTURE).

Restates SPEC.md [MODULE] rdsim and PAPER.md Eqs. 7-12
 with the corrections recorded in SURVEY.md:

  residual (Eq. 10, h = dt):
      phi(r) = J~^T a,
      a = M J~ c + f_fict + h^2 (f_int(u(r)) - f_ext),
      c = (1 + alpha h)(r - r_bar) - h rdot_bar,
      f_fict = M hvv(q, q - q_bar)            (Eq. 8; omitted when drop_fict)
  The mass-proportional Rayleigh term alpha h J~^T M J~ (r - r_bar) is the
  h^2-scaled form of SPEC.md:567's alpha J~^T M J~ (r - r_bar)/dt.

  system Jacobian (Eq. 11 with the +h^2 sign fix F2, SURVEY.md:32):
      dphi/dr = diag(0, vhp(q, a)) + J~^T M [(1+alpha h) U, (1+alpha h) J + dJ]
                + h^2 J~^T K J~
      dJ = svv(q, v) + hv(q, (3 + alpha h) v - h qdot_bar),  v = q - q_bar  (Eq. 12)
      (drop_fict: dJ = hv(q, (1 + alpha h) v - h qdot_bar))
  K~ uses the same cubature set and weights as the force with
  dw/dr ignored (F8).

  step: Newton with LU partial pivoting, backtracking line
  search by halving (<= 10 halvings) on ||phi||_2, predictor r0 = r_bar +
  h rdot_bar, convergence ||phi||_2 <= newton_tol, rdot = (r - r_bar)/h.
  ``fixed_iters`` runs exactly that many full Newton steps (no line search,
  no early exit) for bitwise-comparable control flow.

  jacobian_oracle: column j = Im(phi(r + i eps e_j))/eps,
  residual evaluated over complex128 scalars, cubature weights frozen.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import scipy.linalg

from . import diffops, elastic
from .reduced import split, jtilde, cubature_integrate, wnet_forward


@dataclass
class OSimConfig:
    dt: float = 1.0 / 60.0
    newton_tol: float = 1e-8
    max_iters: int = 20
    drop_fict: bool = False
    integration: str = "cubature"          # or "exact_sum"
    line_search: bool = True
    fixed_iters: int | None = None
    eps: float = diffops.EPS


class OSim:
    """Bundle of everything one simulation needs (reduced model, FE model,
    cubature set + weight net)."""

    def __init__(self, rm, model, cub_elems=None, wnet=None, alpha=None):
        self.rm, self.model = rm, model
        self.cub_elems = None if cub_elems is None else np.asarray(cub_elems, dtype=np.int64)
        self.wnet = wnet
        self.alpha = model.alpha if alpha is None else alpha

    def weights(self, r):
        w_all = wnet_forward(self.wnet, self.rm, r)
        return w_all[self.cub_elems]


def fictitious_force(sim, q, q_bar, eps=diffops.EPS):
    return sim.model.mass * diffops.hvv(sim.rm.D, q, np.asarray(q) - np.asarray(q_bar), eps)


def delta_j(sim, q, q_bar, qdot_bar, dt, drop_fict=False, eps=diffops.EPS):
    ah = sim.alpha * dt
    v = np.asarray(q) - np.asarray(q_bar)
    if drop_fict:
        return diffops.hv(sim.rm.D, q, (1.0 + ah) * v - dt * np.asarray(qdot_bar), eps)
    return (diffops.svv(sim.rm.D, q, v, eps)
            + diffops.hv(sim.rm.D, q, (3.0 + ah) * v - dt * np.asarray(qdot_bar), eps))


def _force_terms(sim, r, cfg, want_K, weights=None):
    rm, model = sim.rm, sim.model
    p, q = split(rm, r)
    J = diffops.jacobian(rm.D, q, cfg.eps)
    Jt = jtilde(rm, q, J)
    u = rm.U @ p + diffops.value(rm.D, q)
    if cfg.integration == "exact_sum":
        elems = np.arange(model.n_tets)
        w = np.ones(elems.size)
    else:
        elems = sim.cub_elems
        w = sim.weights(np.real(r)) if weights is None else weights
    f_red, K_red, f_sc = cubature_integrate(model, rm, elems, w, u, Jt, want_K=want_K)
    return q, J, Jt, f_sc, K_red


def _a_vector(sim, r, state, f_ext, cfg, q, Jt, f_sc):
    h = cfg.dt
    c = (1.0 + sim.alpha * h) * (np.asarray(r) - state[0]) - h * state[1]
    a = sim.model.mass * (Jt @ c) + h * h * (f_sc - f_ext)
    if not cfg.drop_fict:
        q_bar = state[0][sim.rm.n_p:]
        a = a + fictitious_force(sim, q, q_bar, cfg.eps)
    return a


def residual(sim, r, state, f_ext, cfg, weights=None):
    """phi(r). ``state`` = (r_bar, rdot_bar)."""
    q, J, Jt, f_sc, _ = _force_terms(sim, r, cfg, want_K=False, weights=weights)
    a = _a_vector(sim, r, state, f_ext, cfg, q, Jt, f_sc)
    return Jt.T @ a


def system_jacobian(sim, r, state, f_ext, cfg, weights=None):
    """Analytic Eq. 11 + Eq. 12 assembly, F2 sign fix."""
    rm, model = sim.rm, sim.model
    h = cfg.dt
    ah = sim.alpha * h
    q, J, Jt, f_sc, K_red = _force_terms(sim, r, cfg, want_K=True, weights=weights)
    a = _a_vector(sim, r, state, f_ext, cfg, q, Jt, f_sc)
    q_bar = state[0][rm.n_p:]
    qdot_bar = state[1][rm.n_p:]
    dJ = delta_j(sim, q, q_bar, qdot_bar, h, cfg.drop_fict, cfg.eps)
    R = np.concatenate([(1.0 + ah) * rm.U, (1.0 + ah) * J + dJ], axis=1)
    S = Jt.T @ (model.mass[:, None] * R) + h * h * K_red
    S[rm.n_p:, rm.n_p:] += diffops.vhp(rm.D, q, a, cfg.eps)
    return S


def jacobian_oracle(sim, r, state, f_ext, cfg, eps=1e-10):
    """CSFD of residual over complex128 scalars."""
    r = np.asarray(r, dtype=float)
    w = None
    if cfg.integration != "exact_sum":
        w = sim.weights(r)
    n = r.size
    out = np.zeros((n, n))
    for j in range(n):
        rc = r.astype(complex)
        rc[j] += 1j * eps
        out[:, j] = np.imag(residual(sim, rc, state, f_ext, cfg, weights=w)) / eps
    return out


class NewtonDivergence(RuntimeError):
    def __init__(self, msg, last_norm):
        super().__init__(msg)
        self.last_norm = last_norm


def step(sim, r_bar, rdot_bar, f_ext, cfg, trace=None):
    """One implicit timestep. Returns (r, rdot, iters, ||phi||); ``trace``
    (a list) receives the line-search halvings of every Newton iteration."""
    r_bar = np.asarray(r_bar, dtype=float)
    rdot_bar = np.asarray(rdot_bar, dtype=float)
    state = (r_bar, rdot_bar)
    r = r_bar + cfg.dt * rdot_bar
    if cfg.fixed_iters is not None:
        for _ in range(cfg.fixed_iters):
            phi = residual(sim, r, state, f_ext, cfg)
            S = system_jacobian(sim, r, state, f_ext, cfg)
            r = r + scipy.linalg.lu_solve(scipy.linalg.lu_factor(S), -phi)
        phi = residual(sim, r, state, f_ext, cfg)
        return r, (r - r_bar) / cfg.dt, cfg.fixed_iters, float(np.linalg.norm(phi))
    phi = residual(sim, r, state, f_ext, cfg)
    nrm = float(np.linalg.norm(phi))
    it = 0
    while nrm > cfg.newton_tol:
        if it >= cfg.max_iters:
            raise NewtonDivergence(f"Newton did not converge in {cfg.max_iters} iterations; "
                                   f"last residual norm {nrm:.3e}", nrm)
        S = system_jacobian(sim, r, state, f_ext, cfg)
        dr = scipy.linalg.lu_solve(scipy.linalg.lu_factor(S), -phi)
        t = 1.0
        for k in range(11):
            r_try = r + t * dr
            phi_try = residual(sim, r_try, state, f_ext, cfg)
            n_try = float(np.linalg.norm(phi_try))
            if not cfg.line_search or n_try < nrm:
                break
            t *= 0.5
        if trace is not None:
            trace.append(k)
        r, phi, nrm = r_try, phi_try, n_try
        it += 1
    return r, (r - r_bar) / cfg.dt, it, nrm
