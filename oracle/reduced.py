"""Oracle reduced model and neural cubature (TEST INFRASTRUCTURE).

Restates SPEC.md [MODULE] daereduce (Eq. 9-10,
PAPER.md:237-247) and the simulation-time part of [MODULE] neucubature
(PAPER.md:397-419):

  u(r)          = U p + D(q)                                  (Eq. 9)
  J~(q)         = [U, J(q)]                                   (Eq. 10)
  wnet(r)       = square(FC(sin)^3 -> FC)(u(r)), one output per element
  cubature(r)   = sum_{e in C} w_e J~_e^T f_e,  sum_e w_e J~_e^T K_e J~_e
                  (same C and w for force and stiffness, SPEC.md:654;
                   dw/dr ignored, SPEC.md:654 / SURVEY F8)
"""

from __future__ import annotations

import numpy as np

from . import diffops
from . import elastic
from .nets import forward


class OReduced:
    def __init__(self, U, decoder_layers, n_p, n_q):
        self.U = np.asarray(U, dtype=float)
        self.D = decoder_layers
        self.n_p, self.n_q = n_p, n_q

    @property
    def n(self):
        return self.n_p + self.n_q


def split(rm, r):
    r = np.asarray(r)
    return r[: rm.n_p], r[rm.n_p:]


def full_displacement(rm, r):
    p, q = split(rm, r)
    return rm.U @ p + diffops.value(rm.D, q)


def jtilde(rm, q, J=None):
    if J is None:
        J = diffops.jacobian(rm.D, q)
    return np.concatenate([rm.U.astype(J.dtype), J], axis=1)


def reduced_mass(rm, model, q):
    Jt = jtilde(rm, q)
    return Jt.T @ (model.mass[:, None] * Jt)


def wnet_forward(wnet_layers, rm, r):
    """Weights for all elements, >= 0 by the final square."""
    u = full_displacement(rm, r)
    X = np.asarray(u)[None, :, None]
    return forward(wnet_layers, X)[0][:, 0]


def element_reduced_force(model, rm, r, e, Jt=None):
    """J~_e^T f_e for one element."""
    p, q = split(rm, r)
    if Jt is None:
        Jt = jtilde(rm, q)
    u = full_displacement(rm, r)
    f, _ = elastic.element_force_stiffness(model, u, [e], want_K=False)
    rows = model.rows[e]
    m = rows >= 0
    return Jt[rows[m]].T @ f[0][m]


def cubature_integrate(model, rm, elems, weights, u, Jt, want_K=True):
    """Weighted sums over the cubature set C.

    Returns (f_red (n,), K_red (n,n) or None, f_scatter (N,)) where f_scatter is
    the cubature-approximate full-space force sum_e w_e scatter(f_e), whose
    J~-projection equals f_red."""
    elems = np.asarray(elems, dtype=np.int64)
    n = Jt.shape[1]
    if elems.size == 0:
        z = np.zeros(n, dtype=Jt.dtype)
        return z, (np.zeros((n, n), dtype=Jt.dtype) if want_K else None), np.zeros(model.N, dtype=Jt.dtype)
    f, K = elastic.element_force_stiffness(model, u, elems, want_K=want_K)
    w = np.asarray(weights)
    rows = model.rows[elems]                               # (E,12)
    Jz = np.concatenate([Jt, np.zeros((1, n), dtype=Jt.dtype)], axis=0)
    Je = Jz[np.where(rows >= 0, rows, model.N)]            # (E,12,n), zero rows for fixed
    f_red = np.einsum("e,ein,ei->n", w, Je, f)
    K_red = None
    if want_K:
        K_red = np.einsum("e,eim,eij,ejn->mn", w, Je, K, Je, optimize=True)
    f_sc = elastic.scatter(model, f, elems, w)
    return f_red, K_red, f_sc
