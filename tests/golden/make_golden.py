"""Generate golden vectors from the REFERENCE implementation (run in the build container).

    python tests/golden/make_golden.py        # needs /root/reference (read-only)

Imports the reference ``nlrom/mcx.py`` by file path (it is a namespace package
without ``__init__``, SURVEY.md probe §9.5) and records
  * mcx_golden.npz: reference part kernels (parts_mul/inv/sin/cos/sinh/cosh/exp,
    cr_matrix) on seeded random inputs of every order, scalar and batched;
  * decoder_golden.npz: the CSFD decoder bundle (value, jacobian, hvv, hv, svv,
    vjp, vhp) of a small random sin decoder evaluated with the reference part
    kernels and the SPEC pass structure, eps = 1e-10.
The fixtures are committed; nothing at test time reads /root/reference.
"""

from __future__ import annotations

import importlib.util
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_MCX = "/root/reference/pkg/src/nlrom/mcx.py"


def load_reference_mcx():
    spec = importlib.util.spec_from_file_location("_ref_nlrom_mcx", REF_MCX)
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def mcx_golden(mcx):
    rng = np.random.default_rng(20260101)
    out = {}
    for k in range(4):
        n = 1 << k
        a = rng.uniform(-1.0, 1.0, (n, 7, 3))
        b = rng.uniform(-1.0, 1.0, (n, 7, 3))
        pos = rng.uniform(0.5, 1.5, (n, 7, 3))
        out[f"a{k}"], out[f"b{k}"], out[f"pos{k}"] = a, b, pos
        out[f"mul{k}"] = mcx.parts_mul(a, b)
        out[f"inv{k}"] = mcx.parts_inv(pos)
        out[f"sin{k}"] = mcx.parts_sin(a)
        out[f"cos{k}"] = mcx.parts_cos(a)
        out[f"sinh{k}"] = mcx.parts_sinh(a)
        out[f"cosh{k}"] = mcx.parts_cosh(a)
        out[f"exp{k}"] = mcx.parts_exp(a)
        out[f"cr{k}"] = mcx.parts_cr_matrix(a[:, 0, 0])
        # eps-scaled (CSFD-like) inputs: slot s ~ 1e-10^popcount(s)
        sc = np.array([1e-10 ** bin(s).count("1") for s in range(n)])[:, None, None]
        out[f"epsa{k}"] = a * sc
        out[f"epssin{k}"] = mcx.parts_sin(a * sc)
    return out


def decoder_golden(mcx):
    """Small random decoder n_q=3 -> 6 -> 6 -> 6 -> N=20 (sin) + filter, reference kernels."""
    rng = np.random.default_rng(77)
    n_q, N, n_p, w = 3, 20, 4, 6
    dims = [n_q, w, w, w, N]
    Ws, bs = [], []
    for l in range(4):
        lim = np.sqrt(6.0 / dims[l])
        Ws.append(rng.uniform(-lim, lim, (dims[l + 1], dims[l])))
        bs.append(rng.uniform(-lim, lim, dims[l + 1]))
    U, _ = np.linalg.qr(rng.standard_normal((N, n_p)))
    q = rng.uniform(-0.5, 0.5, n_q)
    v = rng.uniform(-0.1, 0.1, n_q)
    a = rng.uniform(-1.0, 1.0, N)
    eps = 1e-10

    def fwd(X, cache=None):
        for l in range(4):
            X = np.einsum("oi,sib->sob", Ws[l], X)
            X[0] += bs[l][:, None]
            if l < 3:
                if cache is not None:
                    cache.append(X)
                X = mcx.parts_sin(X)
        return X - np.einsum("nk,skb->snb", U, np.einsum("nk,snb->skb", U, X))

    def seed(order, slots):
        P = slots[0][1].shape[1]
        X = np.zeros((1 << order, n_q, P))
        X[0] = q[:, None]
        for s, arr in slots:
            X[s] += arr
        return X

    I = np.eye(n_q)
    V = np.repeat(v[:, None], n_q, 1)
    value = fwd(seed(0, [(0, np.zeros((n_q, 1)))]))[0][:, 0]
    jac = fwd(seed(1, [(1, eps * I)]))[1] / eps
    hvv = fwd(seed(2, [(1, eps * v[:, None]), (2, eps * v[:, None])]))[3][:, 0] / eps**2
    hv = fwd(seed(2, [(1, eps * I), (2, eps * V)]))[3] / eps**2
    svv = fwd(seed(3, [(1, eps * I), (2, eps * V), (4, eps * V)]))[7] / eps**3

    def bwd(X, up):
        cache = []
        fwd(X, cache)
        d = up - np.einsum("nk,skb->snb", U, np.einsum("nk,snb->skb", U, up))
        for l in range(3, -1, -1):
            d = np.einsum("oi,sob->sib", Ws[l], d)
            if l > 0:
                d = mcx.parts_mul(d, mcx.parts_cos(cache[l - 1]))
        return d

    vjp = bwd(seed(0, [(0, np.zeros((n_q, 1)))]), a[None, :, None])[0][:, 0]
    up = np.zeros((2, N, n_q))
    up[0] = a[:, None]
    vhp = bwd(seed(1, [(1, eps * I)]), up)[1] / eps
    out = dict(q=q, v=v, a=a, U=U, value=value, jac=jac, hvv=hvv, hv=hv, svv=svv, vjp=vjp, vhp=vhp)
    for l in range(4):
        out[f"W{l}"], out[f"b{l}"] = Ws[l], bs[l]
    return out


def main():
    if not os.path.exists(REF_MCX):
        print("reference not mounted; nothing to do", file=sys.stderr)
        return 1
    mcx = load_reference_mcx()
    np.savez(os.path.join(HERE, "mcx_golden.npz"), **mcx_golden(mcx))
    np.savez(os.path.join(HERE, "decoder_golden.npz"), **decoder_golden(mcx))
    print("wrote mcx_golden.npz, decoder_golden.npz")
    return 0


if __name__ == "__main__":
    sys.exit(main())
