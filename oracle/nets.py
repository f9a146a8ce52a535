"""Oracle dense networks over real / multicomplex scalars (TEST INFRASTRUCTURE).

Restates SPEC.md [MODULE] densenet:
  * layers: fully connected (W (out,in) row-major, b (out,)), fixed filter
    (I - U U^T), sin activation (SPEC.md:116,
    PAPER.md:233), square activation;
  * forward over multicomplex inputs acts part-wise with real W (the
    Cauchy-Riemann block rule, mcx.py:297-300), bias added to the
    real slot only (mcx.py:333-338);
  * backward is standard reverse mode executed in the same
    (multi)complex arithmetic as the forward, so a complex-perturbed forward
    followed by a real-seeded backward is the complex-step BP of Fig. 5
    (PAPER.md:353-366).

A net here is a plain list of layer dicts::

    {"kind": "fc", "W": (out,in), "b": (out,)}
    {"kind": "filter", "U": (N, n_p)}
    {"kind": "sin"} | {"kind": "square"}

Arrays of values are part stacks ``(2**k, dim, batch)`` (MCArray layout,
mcx.py:294-300) of float64 or complex128.
"""

from __future__ import annotations

import numpy as np

from . import mcx_np as mc


def init_uniform(rng: np.random.Generator, out_dim: int, in_dim: int):
    """U(-sqrt(6/fan_in), +sqrt(6/fan_in)) weights and biases."""
    lim = np.sqrt(6.0 / in_dim)
    W = rng.uniform(-lim, lim, (out_dim, in_dim))
    b = rng.uniform(-lim, lim, out_dim)
    return W, b


def _filter(U, X):
    # X: (S, N, B); x - U (U^T x) per slot (factored form of delta_ij - sum_k U_ik U_jk)
    return X - np.matmul(U, np.matmul(U.T, X))


def forward(layers, X, cache=None):
    """Layer-by-layer evaluation over a part stack. ``cache`` (list) receives
    each layer's input for the backward pass."""
    X = np.asarray(X)
    if X.ndim != 3:
        raise ValueError("part stack must be (2**k, dim, batch)")
    for L in layers:
        if cache is not None:
            cache.append(X)
        k = L["kind"]
        if k == "fc":
            W, b = L["W"], L["b"]
            if X.shape[1] != W.shape[1]:
                raise ValueError("dimension mismatch")
            X = np.matmul(W, X)
            X[0] = X[0] + b[:, None]
        elif k == "filter":
            X = _filter(L["U"], X)
        elif k == "sin":
            X = mc.sin(X)
        elif k == "square":
            X = mc.mul(X, X)
        elif k == "cube":          # oracle-only, for the SPEC known-answer D(q) = q^3
            X = mc.mul(mc.mul(X, X), X)
        else:
            raise ValueError(f"unsupported layer kind {k}")
    return X


def backward(layers, X, upstream, want_params=False):
    """Reverse mode in the arithmetic of X (real or order-1 complex, possibly with
    complex128 coefficients). Returns (input cotangent, [param cotangents])."""
    cache = []
    forward(layers, X, cache)
    d = np.asarray(upstream)
    grads = []
    for L, x in zip(reversed(layers), reversed(cache)):
        k = L["kind"]
        if k == "fc":
            if want_params:
                # dW[s] = sum_b (d x^T) in multicomplex arithmetic; db = sum_b d
                dW = mc.mul(d[:, :, None, :], x[:, None, :, :]).sum(axis=-1)
                grads.append((dW, d.sum(axis=-1)))
            d = np.matmul(L["W"].T, d)
        elif k == "filter":
            d = _filter(L["U"], d)
        elif k == "sin":
            d = mc.mul(d, mc.cos(x))
        elif k == "square":
            d = mc.mul(d, 2.0 * x)
        elif k == "cube":
            d = mc.mul(d, 3.0 * mc.mul(x, x))
    grads.reverse()
    return d, grads
