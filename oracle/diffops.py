"""Oracle CSFD contraction operators (TEST INFRASTRUCTURE).

Restates SPEC.md [MODULE] diffops and PAPER.md §4.3-4.4
 with the reference pass structure:

  op        passes  order  seeds (per pass j)                  extracted
  value     1       0      -                                   slot 0
  jvp       1       1      i1 = v                              slot 0b1 / eps
  jacobian  n_q     1      i1 = e_j                            slot 0b1 / eps
  hvv       1       2      i1 = v, i2 = v                      slot 0b11 / eps^2
  hv        n_q     2      i1 = e_j, i2 = v                    slot 0b11 / eps^2
  svv       n_q     3      i1 = e_j, i2 = v, i3 = v            slot 0b111 / eps^3
  vjp       1 bwd   0      seed a                              input cotangent
  vhp       n_q     1+bwd  i1 = e_j, seed a                    Im(input cot)/eps

All n_q passes of one operator are one batch; vhp is a separate
batch.  Every function accepts q with complex128 entries, which
the rdsim jacobian_oracle uses as an extra outer CSFD direction.
"""

from __future__ import annotations

import numpy as np

from . import mcx_np as mc
from .nets import forward, backward

EPS = 1e-10  # DiffConfig.eps default


def _check(x, what):
    if not np.all(np.isfinite(x)):
        raise FloatingPointError(f"{what}: non-finite result")
    return x


def _seed(q, order, seeds):
    """Part stack (2**order, n_q, P) with slot 0 = q and the given seed slots."""
    q = np.asarray(q)
    P = seeds[0][1].shape[1] if seeds else 1
    X = np.zeros((1 << order, q.shape[0], P), dtype=np.result_type(q.dtype, np.float64))
    X[0] = q[:, None]
    for slot, arr in seeds:
        X[slot] = X[slot] + arr
    return X


def value(D, q):
    return _check(forward(D, _seed(q, 0, []))[0][:, 0], "value")


def jvp(D, q, v, eps=EPS):
    X = _seed(q, 1, [(1, eps * np.asarray(v, dtype=float)[:, None])])
    return _check(forward(D, X)[1][:, 0] / eps, "jvp")


def jacobian(D, q, eps=EPS):
    n = len(q)
    X = _seed(q, 1, [(1, eps * np.eye(n))])
    return _check(forward(D, X)[1] / eps, "jacobian")


def hvv(D, q, v, eps=EPS):
    ev = eps * np.asarray(v)[:, None]
    X = _seed(q, 2, [(1, ev), (2, ev)])
    return _check(forward(D, X)[3][:, 0] / eps**2, "hvv")


def hv(D, q, v, eps=EPS):
    n = len(q)
    X = _seed(q, 2, [(1, eps * np.eye(n)), (2, eps * np.repeat(np.asarray(v)[:, None], n, 1))])
    return _check(forward(D, X)[3] / eps**2, "hv")


def svv(D, q, v, eps=EPS):
    n = len(q)
    V = eps * np.repeat(np.asarray(v)[:, None], n, 1)
    X = _seed(q, 3, [(1, eps * np.eye(n)), (2, V), (4, V)])
    return _check(forward(D, X)[7] / eps**3, "svv")


def vjp(D, q, a):
    a = np.asarray(a)
    X = _seed(q, 0, [])
    up = a[None, :, None].astype(np.result_type(a.dtype, X.dtype))
    d, _ = backward(D, X, up)
    return d[0][:, 0]


def vhp(D, q, a, eps=EPS):
    n = len(q)
    a = np.asarray(a)
    X = _seed(q, 1, [(1, eps * np.eye(n))])
    up = np.zeros((2, a.shape[0], n), dtype=np.result_type(a.dtype, X.dtype))
    up[0] = a[:, None]
    d, _ = backward(D, X, up)
    return _check(d[1] / eps, "vhp")


def pass_count(n_q: int) -> int:
    """Network passes of one Newton-iteration bundle."""
    return 4 * n_q + 2
