"""Oracle (TEST INFRASTRUCTURE ONLY; the product never imports this) for the neural-cubature
training row (Eq. 18).

* per-element reduced forces f~_e(r) = J~_e(r)^T f_e(u(r)) for all elements, restated in numpy
  from the oracle StVK element forces (oracle/elastic.py) and the oracle J~ (oracle/reduced.py);
* the greedy residual-matching + NNLS baseline as a plain loop over
  scipy.optimize.nnls (scipy 1.18, Lawson-Hanson; the SPEC's named algorithm).

Parity is pinned by SPEC examples only (no reference code exists above mcx: SURVEY.md §8c).
"""

import numpy as np
from scipy.optimize import nnls as scipy_nnls

from . import elastic, reduced


def element_reduced_forces(model, rm, r):
    """(T, n): J~_e^T f_e for every element at pose r."""
    p, q = reduced.split(rm, r)
    Jt = reduced.jtilde(rm, q)
    u = reduced.full_displacement(rm, r)
    f, _ = elastic.element_force_stiffness(model, u, None, want_K=False)
    rows = model.rows
    n = Jt.shape[1]
    Jz = np.concatenate([Jt, np.zeros((1, n))], axis=0)
    Je = Jz[np.where(rows >= 0, rows, model.N)]  # (T, 12, n)
    return np.einsum("ein,ei->en", Je, f)


def train_arrays(model, rm, rs):
    """(f (S, n), F (S, T, n), u (S, N)) at poses rs."""
    F = np.stack([element_reduced_forces(model, rm, r) for r in rs])
    u = np.stack([reduced.full_displacement(rm, r) for r in rs])
    return F.sum(axis=1), F, u


def greedy(f, F, target):
    """SPEC.md:629-636 with every pose's block scaled by 1 / ||f_s||; returns (C, w)."""
    S, T, n = F.shape
    sc = 1.0 / np.linalg.norm(f, axis=1)
    A = (F * sc[:, None, None]).transpose(1, 0, 2).reshape(T, S * n)
    b = (f * sc[:, None]).reshape(-1)
    norms = np.linalg.norm(A, axis=1)
    C, w, res = [], np.zeros(0), b.copy()
    for _ in range(target):
        best, be = -np.inf, -1
        for e in range(T):
            if e in C or norms[e] == 0:
                continue
            s = A[e] @ res / norms[e]
            if s > best:
                best, be = s, e
        if be < 0:
            break
        C.append(be)
        w, _ = scipy_nnls(A[C].T, b)
        res = b - A[C].T @ w
    return np.array(C), w
