"""nlrom.daereduce — PCA + PCA-orthogonal DAE subspace (Eq. 9-10)."""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .densenet import DenseNet


class ReducedModel:
    """U (N x n_p), decoder D (ends with the filter I - U U^T), dims.

    Queries that need only the decoder and U use a device session; the mass matrix
    comes from the ElasticModel attached with ``attach``."""

    def __init__(self, U, decoder: DenseNet, n_p: int, n_q: int, encoder: DenseNet | None = None):
        self.U = np.ascontiguousarray(U, dtype=float)
        self.decoder, self.encoder = decoder, encoder
        self.n_p, self.n_q = int(n_p), int(n_q)
        if self.U.shape[1] != self.n_p:
            raise ValueError("U must be N x n_p")
        self.model = None
        self.cm = None

    @property
    def n(self):
        return self.n_p + self.n_q

    def attach(self, model, cm=None):
        """Bind the FE model (and cubature model) whose mesh the decoder lives on."""
        self.model, self.cm = model, cm
        return self

    def session(self):
        from .session import session_for
        if self.model is None:
            raise ValueError("attach an ElasticModel first (ReducedModel.attach)")
        return session_for(self, self.model, self.cm)


@dataclass
class ReducedState:
    """r = (p, q), rdot, dt."""
    r: np.ndarray
    rdot: np.ndarray
    dt: float = 1.0 / 60.0

    def __post_init__(self):
        self.r = np.asarray(self.r, dtype=float).copy()
        self.rdot = np.asarray(self.rdot, dtype=float).copy()
        if self.r.shape != self.rdot.shape or not (np.all(np.isfinite(self.r)) and np.all(np.isfinite(self.rdot))):
            raise ValueError("ReducedState must be finite with matching r / rdot (SPEC.md:452)")


def _split(rm, r):
    r = np.asarray(r, dtype=float)
    return r[: rm.n_p], r[rm.n_p:]


def full_displacement(rm: ReducedModel, r) -> np.ndarray:
    """u = U p + D(q) (Eq. 9)."""
    return rm.session().full_displacement(r)


def jtilde(rm: ReducedModel, q) -> np.ndarray:
    """J~ = [U, J(q)] (N x (n_p + n_q), Eq. 10)."""
    return rm.session().jtilde(q)


def reduced_mass(rm: ReducedModel, q, model=None) -> np.ndarray:
    """J~^T M J~ (Eq. 10): the mass block of the exact_sum system
    Jacobian with dt = 0 and zero state offsets."""
    from .rdsim import SimConfig
    from .session import session_for
    s = rm.session() if model is None else session_for(rm, model, rm.cm)
    r = np.concatenate([np.zeros(rm.n_p), np.asarray(q, dtype=float)])
    # The device system Jacobian at r = r_bar, rdot_bar = 0, f_ext = 0, drop_fict and
    # dt -> 0 is exactly the mass block J~^T M [U, J] (dJ, vhp(a), dt^2 K all vanish).
    cfg = SimConfig(dt=1e-30, integration="exact_sum", drop_fict=True)
    return s.system_jacobian(r, r, np.zeros(rm.n), np.zeros(s.N), cfg)


def encode(rm: ReducedModel, u):
    """(p, q) = (U^T u, encoder(u)); needs a trained encoder."""
    from .densenet import forward
    if rm.encoder is None:
        raise ValueError("no encoder: DAE training is offline (SURVEY.md §2)")
    u = np.asarray(u, dtype=float)
    return rm.U.T @ u, forward(rm.encoder, u)


def build_dae(*_a, **_k):
    """DAE construction / training is offline, out of scope."""
    raise NotImplementedError("build_dae is offline training, out of scope for the B200 hot path")
