"""Pin the oracle multicomplex kernels: reference golden vectors (tests/golden/mcx_golden.npz,
made by tests/golden/make_golden.py from /root/reference/pkg/src/nlrom/mcx.py) and the
checks of the reference test file pkg/tests/test_mcx.py re-derived independently."""

import os
from math import sin, cos, sinh, cosh

import numpy as np
import pytest

from oracle import mcx_np as mc

GOLD = np.load(os.path.join(os.path.dirname(__file__), "golden", "mcx_golden.npz"))


@pytest.mark.parametrize("k", range(4))
def test_oracle_matches_reference_golden(k):
    a, b, pos = GOLD[f"a{k}"], GOLD[f"b{k}"], GOLD[f"pos{k}"]
    checks = [("mul", mc.mul(a, b)), ("inv", mc.inv(pos)), ("sin", mc.sin(a)), ("cos", mc.cos(a)),
              ("sinh", mc.sinh(a)), ("cosh", mc.cosh(a)), ("exp", mc.exp(a)),
              ("epssin", mc.sin(GOLD[f"epsa{k}"]))]
    for name, got in checks:
        want = GOLD[f"{name}{k}"]
        assert np.abs(got - want).max() <= 1e-15 * max(np.abs(want).max(), 1e-300), name
    assert np.array_equal(mc.cr_matrix(a[:, 0, 0]), GOLD[f"cr{k}"])


def _order2_closed_form(a, b, c, d):
    # Appendix A a'..d' (test_mcx.py:9-15 re-derived from sin(u)cosh(v), cos(u)sinh(v))
    return np.array([
        sin(a) * cosh(b) * cosh(c) * cos(d) - cos(a) * sinh(b) * sinh(c) * sin(d),
        sin(a) * cosh(b) * sinh(c) * sin(d) + cos(a) * sinh(b) * cosh(c) * cos(d),
        cos(a) * cosh(b) * sinh(c) * cos(d) + sin(a) * sinh(b) * cosh(c) * sin(d),
        cos(a) * cosh(b) * cosh(c) * sin(d) - sin(a) * sinh(b) * sinh(c) * cos(d)])


def test_order2_closed_form():
    rng = np.random.default_rng(5)
    for _ in range(1000):
        v = rng.uniform(-1, 1, 4)
        want = _order2_closed_form(*v)
        assert np.abs(mc.sin(v) - want).max() <= 1e-13 * np.maximum(np.abs(want), 1e-3).max()


def _taylor_sin(z, terms=30):
    acc = np.zeros_like(z)
    p = z.copy()
    z2 = mc.mul(z, z)
    fact, sign, k = 1.0, 1.0, 1
    for _ in range(terms):
        acc = acc + p * (sign / fact)
        p = mc.mul(p, z2)
        fact *= (k + 1) * (k + 2)
        k += 2
        sign = -sign
    return acc


def test_sin_vs_ring_taylor():
    rng = np.random.default_rng(7)
    for _ in range(50):
        k = rng.integers(0, 4)
        z = rng.uniform(-0.8, 0.8, 1 << k)
        want = _taylor_sin(z)
        assert np.abs(mc.sin(z) - want).max() <= 1e-13 * max(np.abs(want).max(), 1.0)


def test_exp_vs_complex128_and_ring_axioms():
    rng = np.random.default_rng(8)
    for _ in range(50):
        a, b = rng.uniform(-1, 1, 2)
        w = np.exp(a + 1j * b)
        got = mc.exp(np.array([a, b]))
        assert got[0] == pytest.approx(w.real, rel=1e-14) and got[1] == pytest.approx(w.imag, rel=1e-14)
    rng = np.random.default_rng(11)
    for _ in range(200):
        k = rng.integers(0, 4)
        a, b, c = (rng.uniform(-1, 1, 1 << k) for _ in range(3))
        lhs = mc.mul(a + b, c)
        assert np.abs(lhs - (mc.mul(a, c) + mc.mul(b, c))).max() <= 1e-14 * max(np.abs(lhs).max(), 1)
        assert np.allclose(mc.mul(a, b), mc.mul(b, a), rtol=1e-14, atol=0)


def test_cr_homomorphism_and_division():
    rng = np.random.default_rng(10)
    for k in (1, 2, 3):
        for _ in range(50):
            a, b = rng.uniform(-1, 1, 1 << k), rng.uniform(-1, 1, 1 << k)
            rhs = mc.cr_matrix(mc.mul(a, b))
            assert np.abs(mc.cr_matrix(a) @ mc.cr_matrix(b) - rhs).max() <= 1e-13 * max(np.abs(rhs).max(), 1)
    rng = np.random.default_rng(3)
    for k in range(4):
        z = rng.uniform(0.5, 1.5, 1 << k)
        assert np.allclose(mc.mul(z, mc.inv(z)), np.eye(1, 1 << k, 0)[0], atol=1e-13)


def test_order3_real_coefficient_vs_16_terms():
    # test_mcx.py:18-49 table, re-derived: real coefficient of sin at order 3
    T = [(+1, sin, cosh, cosh, cos, cosh, cos, cos, cosh), (+1, sin, cosh, cosh, cos, sinh, sin, sin, sinh),
         (+1, sin, cosh, sinh, sin, cosh, cos, sin, sinh), (-1, sin, cosh, sinh, sin, sinh, sin, cos, cosh),
         (+1, cos, sinh, cosh, cos, cosh, cos, sin, sinh), (-1, cos, sinh, cosh, cos, sinh, sin, cos, cosh),
         (-1, cos, sinh, sinh, sin, cosh, cos, cos, cosh), (-1, cos, sinh, sinh, sin, sinh, sin, sin, sinh),
         (-1, cos, cosh, sinh, cos, sinh, cos, sin, cosh), (+1, cos, cosh, sinh, cos, cosh, sin, cos, sinh),
         (+1, cos, cosh, cosh, sin, sinh, cos, cos, sinh), (+1, cos, cosh, cosh, sin, cosh, sin, sin, cosh),
         (-1, sin, sinh, sinh, cos, sinh, cos, cos, sinh), (-1, sin, sinh, sinh, cos, cosh, sin, sin, cosh),
         (-1, sin, sinh, cosh, sin, sinh, cos, sin, cosh), (+1, sin, sinh, cosh, sin, cosh, sin, cos, sinh)]
    rng = np.random.default_rng(6)
    for _ in range(1000):
        v = rng.uniform(-1, 1, 8)
        want = sum(t[0] * np.prod([f(x) for f, x in zip(t[1:], v)]) for t in T)
        assert abs(mc.sin(v)[0] - want) <= 1e-12 * max(abs(want), 1e-3)
