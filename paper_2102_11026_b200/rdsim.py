"""nlrom.rdsim — reduced implicit-Euler Newton integrator (Eqs. 7-12).

Every operation runs on the device session of (ReducedModel, ElasticModel,
CubatureModel); see DESIGN.md for the fused per-iteration pipeline:

  phi(r)  = J~^T a,  a = M J~ c + f_fict + dt^2 (f_int - f_ext),
            c = (1 + alpha dt)(r - r_bar) - dt rdot_bar            (Eq. 10 + SPEC.md:567)
  dphi/dr = diag(0, vhp(a)) + J~^T M [(1+alpha dt) U, (1+alpha dt) J + dJ] + dt^2 K~
            (Eq. 11 with the +dt^2 sign fix)
  dJ      = svv(v) + hv((3 + alpha dt) v - dt qdot_bar), v = q - q_bar (Eq. 12)
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from ._lib import NewtonDivergence
from .daereduce import ReducedModel, ReducedState


@dataclass
class SimConfig:
    """SPEC.md:506-509 (+ line_search flag SPEC.md:568, fixed_iters for bitwise-comparable runs)."""
    dt: float = 1.0 / 60.0
    newton_tol: float = 1e-8
    max_iters: int = 20
    drop_fict: bool = False
    integration: str = "cubature"
    line_search: bool = True
    fixed_iters: int | None = None

    def __post_init__(self):
        if not (self.dt > 0 and self.newton_tol > 0):
            raise ValueError("dt > 0 and newton_tol > 0 required (SPEC.md:508)")
        if self.integration not in ("cubature", "exact_sum"):
            raise ValueError("integration must be 'cubature' or 'exact_sum'")


def _sess(rm: ReducedModel, model, cm=None):
    from .session import session_for
    return session_for(rm, model, cm if cm is not None else rm.cm)


def fictitious_force(rm: ReducedModel, q, q_bar, model=None):
    """M hvv(q, q - q_bar) (Eq. 8)."""
    return _sess(rm, model or rm.model).fictitious_force(q, q_bar)


def delta_j(rm: ReducedModel, q, q_bar, qdot_bar, dt, model=None, drop_fict=False):
    """svv(q, v) + hv(q, 3v - dt qdot_bar), v = q - q_bar (Eq. 12).
    Uses the Rayleigh alpha of the attached model ((3 + alpha dt) v)."""
    return _sess(rm, model or rm.model).delta_j(q, q_bar, qdot_bar, dt, drop_fict)


def residual(rm: ReducedModel, model, state: ReducedState, f_ext, cfg: SimConfig, r=None, cm=None):
    """phi at candidate r (default: state.r) for the previous state (r_bar, rdot_bar) = state."""
    r = state.r if r is None else r
    return _sess(rm, model, cm).residual(r, state.r, state.rdot, f_ext, cfg)


def system_jacobian(rm: ReducedModel, model, state: ReducedState, f_ext, cfg: SimConfig, r=None, cm=None):
    """Analytic Eq. 11 + Eq. 12 assembly."""
    r = state.r if r is None else r
    return _sess(rm, model, cm).system_jacobian(r, state.r, state.rdot, f_ext, cfg)


def step(rm: ReducedModel, model, state: ReducedState, f_ext, cfg: SimConfig, cm=None, return_info=False):
    """One implicit timestep: Newton + LU-pp + halving line search
    on the device; returns the new ReducedState (and (iters, ||phi||) if asked)."""
    # the final residual norm of a fixed-iteration step is evaluated only when it is returned
    r, rdot, iters, nrm = _sess(rm, model, cm).step(state.r, state.rdot, f_ext, cfg, want_norm=return_info)
    new = ReducedState._owned(r, rdot, cfg.dt)
    return (new, (iters, nrm)) if return_info else new


__all__ = ["SimConfig", "fictitious_force", "delta_j", "residual", "system_jacobian", "step", "NewtonDivergence"]
