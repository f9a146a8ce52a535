"""nlrom.diffops — CSFD contraction operators (§4.3-4.4).

``D`` is either a decoder ``DenseNet`` (generic GPU net path, literal multicomplex
arithmetic with DiffConfig.eps, exactly the reference algorithm) or a
``ReducedModel`` (fused device context: the decoder layers with multi-dual
epilogues on eps-scaled slots, or literal multicomplex when
``DiffConfig.mode == "multicomplex"``). Both keep the reference pass structure
(n_q passes of one operator submitted as one batch).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib
from .densenet import DenseNet, forward, backward
from .mcx import MCArray


@dataclass
class DiffConfig:
    """eps: CSFD step. mode: "scaled" (multi-dual on eps-scaled
    slots; equals multicomplex CSFD to relative O(eps^2)) or "multicomplex"."""
    eps: float = 1e-10
    mode: str = "scaled"

    def __post_init__(self):
        if not self.eps > 0:
            raise ValueError("eps must be > 0 (SPEC.md:206)")
        if self.mode not in ("scaled", "multicomplex"):
            raise ValueError("mode must be 'scaled' or 'multicomplex'")


@dataclass
class DecoderJet:
    """SPEC.md:208-211."""
    value: np.ndarray
    jac: np.ndarray | None = None
    hvv: np.ndarray | None = None
    hv: np.ndarray | None = None
    svv: np.ndarray | None = None


_DEFAULT = DiffConfig()


def _finite(x, what):
    if not np.all(np.isfinite(x)):
        raise FloatingPointError(f"{what}: non-finite result")
    return x


def _ctx(D):
    from .daereduce import ReducedModel
    if isinstance(D, ReducedModel):
        return D.session()
    return None


def _net(D):
    from .daereduce import ReducedModel
    return D.decoder if isinstance(D, ReducedModel) else D


def _mc_forward(D, q, order, seeds, eps):
    """Generic-net literal multicomplex pass batch: seeds = [(slot, (n_q, P) array)]."""
    q = np.asarray(q, dtype=float)
    P = seeds[0][1].shape[1] if seeds else 1
    X = np.zeros((1 << order, q.size, P))
    X[0] = q[:, None]
    for s, a in seeds:
        X[s] += eps * a
    return forward(_net(D), MCArray(X)).parts


def _run(D, op, q, vec, cfg, generic):
    s = _ctx(D)
    if s is not None:
        return s.diffop(op, q, vec, cfg.eps, 0 if cfg.mode == "scaled" else 1)
    return generic()


def value(D, q, cfg: DiffConfig = _DEFAULT):
    return _finite(_run(D, _lib.OP_VALUE, q, None, cfg,
                        lambda: forward(_net(D), np.asarray(q, dtype=float))), "value")


def jvp(D, q, v, cfg: DiffConfig = _DEFAULT):
    """J v = Im_1 / eps of one order-1 pass."""
    def g():
        return _mc_forward(D, q, 1, [(1, np.asarray(v, float)[:, None])], cfg.eps)[1][:, 0] / cfg.eps
    return _finite(_run(D, _lib.OP_JVP, q, v, cfg, g), "jvp")


def jacobian(D, q, cfg: DiffConfig = _DEFAULT):
    """N x n_q Jacobian, n_q canonical order-1 passes in one batch."""
    n = len(q)

    def g():
        return _mc_forward(D, q, 1, [(1, np.eye(n))], cfg.eps)[1] / cfg.eps
    return _finite(_run(D, _lib.OP_JACOBIAN, q, None, cfg, g), "jacobian")


def hvv(D, q, v, cfg: DiffConfig = _DEFAULT):
    """(H v) v = Im_12 / eps^2 of one order-2 pass."""
    def g():
        vv = np.asarray(v, float)[:, None]
        return _mc_forward(D, q, 2, [(1, vv), (2, vv)], cfg.eps)[3][:, 0] / cfg.eps**2
    return _finite(_run(D, _lib.OP_HVV, q, v, cfg, g), "hvv")


def hv(D, q, v, cfg: DiffConfig = _DEFAULT):
    """H v as N x n_q: pass j seeds i1 = e_j, i2 = v."""
    n = len(q)

    def g():
        V = np.repeat(np.asarray(v, float)[:, None], n, 1)
        return _mc_forward(D, q, 2, [(1, np.eye(n)), (2, V)], cfg.eps)[3] / cfg.eps**2
    return _finite(_run(D, _lib.OP_HV, q, v, cfg, g), "hv")


def svv(D, q, v, cfg: DiffConfig = _DEFAULT):
    """(S v) v as N x n_q: pass j seeds i1 = e_j, i2 = i3 = v."""
    n = len(q)

    def g():
        V = np.repeat(np.asarray(v, float)[:, None], n, 1)
        return _mc_forward(D, q, 3, [(1, np.eye(n)), (2, V), (4, V)], cfg.eps)[7] / cfg.eps**3
    return _finite(_run(D, _lib.OP_SVV, q, v, cfg, g), "svv")


def vjp(D, q, a, cfg: DiffConfig = _DEFAULT):
    """J^T a by one real backward pass."""
    def g():
        return backward(_net(D), np.asarray(q, float), np.asarray(a, float))
    return _finite(_run(D, _lib.OP_VJP, q, a, cfg, g), "vjp")


def vhp(D, q, a, cfg: DiffConfig = _DEFAULT):
    """H^T a (n_q x n_q) by complex-step BP: pass j forwards q + eps e_j i1, backward
    of g = a . D(q); column j = Im(input cotangent)/eps."""
    n = len(q)

    def g():
        X = np.zeros((2, n, n))
        X[0] = np.asarray(q, float)[:, None]
        X[1] = cfg.eps * np.eye(n)
        up = np.zeros((2, len(a), n))
        up[0] = np.asarray(a, float)[:, None]
        return backward(_net(D), MCArray(X), MCArray(up)).parts[1] / cfg.eps
    return _finite(_run(D, _lib.OP_VHP, q, a, cfg, g), "vhp")


def jet(D, q, v, cfg: DiffConfig = _DEFAULT) -> DecoderJet:
    return DecoderJet(value(D, q, cfg), jacobian(D, q, cfg), hvv(D, q, v, cfg), hv(D, q, v, cfg), svv(D, q, v, cfg))


def pass_count(n_q: int) -> int:
    """Network passes of one Newton-iteration bundle in the reference structure."""
    return 4 * n_q + 2
