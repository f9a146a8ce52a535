"""Oracle restatement of the reference multicomplex part kernels (TEST INFRASTRUCTURE).

Follows /root/reference/pkg/src/nlrom/mcx.py:
  * slot layout: parts[s] is the coefficient of prod_{d: bit d-1 of s} i_d
    (mcx.py:1-8); axis 0 of every array is the slot axis.
  * product: split on the top direction, (z1 + z2 i_n)(w1 + w2 i_n) =
    (z1 w1 - z2 w2) + (z1 w2 + z2 w1) i_n                       (mcx.py:39-49)
  * reciprocal via the conjugate on the top direction            (mcx.py:52-60)
  * sin/cos/sinh/cosh by the angle-addition recursion, sin(u + v i_n) =
    sin u cosh v + cos u sinh v i_n, sinh(u + v i_n) = sinh u cos v +
    cosh u sin v i_n                                              (mcx.py:63-100)
  * exp(u + v i_n) = exp u (cos v + sin v i_n)                   (mcx.py:103-110)
  * Cauchy-Riemann block matrix [[a, -b], [b, a]]                (mcx.py:113-121)

All kernels are dtype-generic (float64 or complex128 coefficients).  The
complex128 case is how the oracle realises one EXTRA commuting imaginary
direction (numpy's ``1j``) on top of up to three multicomplex directions; the
rdsim jacobian_oracle uses it for the outer CSFD
perturbation of the residual.
"""

from __future__ import annotations

import numpy as np

MAX_ORDER = 3


def order_of(n_slots: int) -> int:
    k = int(n_slots).bit_length() - 1
    if n_slots != (1 << k) or k > MAX_ORDER:
        raise ValueError(f"{n_slots} slots is not 2**k with k <= {MAX_ORDER}")
    return k


def _halves(p):
    h = p.shape[0] >> 1
    return p[:h], p[h:]


def mul(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """Multicomplex product of equal-order part stacks (mcx.py:39-49)."""
    if a.shape[0] == 1:
        return a * b
    z1, z2 = _halves(a)
    w1, w2 = _halves(b)
    re = mul(z1, w1) - mul(z2, w2)
    im = mul(z1, w2) + mul(z2, w1)
    return np.concatenate((re, im), axis=0)


def inv(a: np.ndarray) -> np.ndarray:
    """1/(z1 + z2 i_n) = (z1 - z2 i_n) / (z1^2 + z2^2)  (mcx.py:52-60)."""
    if a.shape[0] == 1:
        return 1.0 / a
    z1, z2 = _halves(a)
    d = inv(mul(z1, z1) + mul(z2, z2))
    return np.concatenate((mul(z1, d), -mul(z2, d)), axis=0)


def sin_cos(p: np.ndarray):
    """(sin p, cos p) by the angle-addition recursion (mcx.py:63-73)."""
    if p.shape[0] == 1:
        return np.sin(p), np.cos(p)
    u, v = _halves(p)
    su, cu = sin_cos(u)
    shv, chv = sinh_cosh(v)
    s = np.concatenate((mul(su, chv), mul(cu, shv)), axis=0)
    c = np.concatenate((mul(cu, chv), -mul(su, shv)), axis=0)
    return s, c


def sinh_cosh(p: np.ndarray):
    """(sinh p, cosh p) by the angle-addition recursion (mcx.py:76-86)."""
    if p.shape[0] == 1:
        return np.sinh(p), np.cosh(p)
    u, v = _halves(p)
    shu, chu = sinh_cosh(u)
    sv, cv = sin_cos(v)
    sh = np.concatenate((mul(shu, cv), mul(chu, sv)), axis=0)
    ch = np.concatenate((mul(chu, cv), mul(shu, sv)), axis=0)
    return sh, ch


def sin(p):
    return sin_cos(p)[0]


def cos(p):
    return sin_cos(p)[1]


def sinh(p):
    return sinh_cosh(p)[0]


def cosh(p):
    return sinh_cosh(p)[1]


def exp(p: np.ndarray) -> np.ndarray:
    """exp(u + v i_n) = exp(u)(cos v + sin v i_n)  (mcx.py:103-110)."""
    if p.shape[0] == 1:
        return np.exp(p)
    u, v = _halves(p)
    eu = exp(u)
    sv, cv = sin_cos(v)
    return np.concatenate((mul(eu, cv), mul(eu, sv)), axis=0)


def cr_matrix(p: np.ndarray) -> np.ndarray:
    """Block-recursive Cauchy-Riemann matrix of a 1-d part stack (mcx.py:113-121)."""
    if p.shape[0] == 1:
        return np.asarray(p, dtype=float).reshape(1, 1)
    a, b = _halves(p)
    A, B = cr_matrix(a), cr_matrix(b)
    return np.block([[A, -B], [B, A]])


def dirs_index(dirs) -> int:
    """Bitmask slot index of a set of imaginary directions (mcx.py:128-134)."""
    s = 0
    for d in dirs:
        d = int(d)
        if not 1 <= d <= MAX_ORDER:
            raise ValueError(f"direction {d} out of range")
        s |= 1 << (d - 1)
    return s


def promote(x: np.ndarray, order: int) -> np.ndarray:
    """Embed a real (or complex128) array at the given order, all imaginaries 0."""
    x = np.asarray(x)
    out = np.zeros((1 << order,) + x.shape, dtype=np.result_type(x.dtype, np.float64))
    out[0] = x
    return out
