"""SPEC acceptance criterion 1: CSFD correctness. For 20 random compositions of
{sin, exp, x, +} on <= 5 variables, first / second / third derivatives from multicomplex steps
(the drop-in nlrom.mcx; slot i1, i1 i2, i1 i2 i3 divided by eps^k) match the analytic values
(sympy) to relative error <= 1e-10, for every eps in 1e-6 .. 1e-12 (stable across eps)."""

import time

import numpy as np
import pytest

sympy = pytest.importorskip("sympy")

from nlrom import mcx
from nlrom.mcx import MultiComplex


def _random_expr(rng, syms, depth):
    if depth == 0 or rng.random() < 0.2:
        if rng.random() < 0.8:
            return syms[rng.integers(len(syms))]
        return sympy.Float(round(float(rng.uniform(-1.5, 1.5)), 3))
    op = rng.integers(4)
    if op == 0:
        return sympy.sin(_random_expr(rng, syms, depth - 1))
    if op == 1:   # keep exp arguments moderate
        return sympy.exp(sympy.Rational(1, 2) * _random_expr(rng, syms, depth - 1))
    a, b = _random_expr(rng, syms, depth - 1), _random_expr(rng, syms, depth - 1)
    return a * b if op == 2 else a + b


def _eval_mc(expr, env):
    """Evaluate a sympy tree with MultiComplex arithmetic (sin / exp / * / + only)."""
    if expr.is_Symbol:
        return env[expr.name]
    if expr.is_Number:
        return float(expr)
    args = [_eval_mc(a, env) for a in expr.args]
    if isinstance(expr, sympy.sin):
        return mcx.mc_sin(args[0])
    if isinstance(expr, sympy.exp):
        return mcx.mc_exp(args[0])
    if isinstance(expr, sympy.Pow):   # sympy folds x*x into x**2: integer powers by repeated products
        base, n = args[0], int(expr.args[1])
        assert n >= 1 and n == expr.args[1]
        out = base
        for _ in range(n - 1):
            out = out * base
        return out
    assert isinstance(expr, (sympy.Add, sympy.Mul)), type(expr)
    out = args[0]
    for a in args[1:]:
        out = out + a if isinstance(expr, sympy.Add) else out * a
    return out


def _lift(x, order, dirs):
    """x + eps e_dirs: the perturbation of one variable on the listed imaginary directions."""
    parts = np.zeros(1 << order)
    parts[0] = x
    for d in dirs:
        parts[1 << (d - 1)] = 1.0
    return parts


def test_random_compositions_derivatives_stable_across_eps():
    rng = np.random.default_rng(1)
    t0 = time.time()
    checked = 0
    for case in range(20):
        nv = int(rng.integers(1, 6))
        syms = sympy.symbols(" ".join(f"x{i}" for i in range(nv)))
        syms = syms if isinstance(syms, tuple) else (syms,)
        expr = _random_expr(rng, syms, 4)
        while not expr.free_symbols:
            expr = _random_expr(rng, syms, 4)
        x = rng.uniform(-1.0, 1.0, nv)
        subs = {s: x[i] for i, s in enumerate(syms)}
        a, b, c = (int(rng.integers(nv)) for _ in range(3))
        want = [float(sympy.diff(expr, syms[a]).evalf(subs=subs)),
                float(sympy.diff(expr, syms[a], syms[b]).evalf(subs=subs)),
                float(sympy.diff(expr, syms[a], syms[b], syms[c]).evalf(subs=subs))]
        for eps in (1e-6, 1e-8, 1e-10, 1e-12):
            got = []
            for order, dirs_of in ((1, {a: [1]}), (2, {a: [1], b: [2]}), (3, {a: [1], b: [2], c: [3]})):
                env = {}
                for i, s in enumerate(syms):
                    dirs = []
                    if order >= 1 and i == a:
                        dirs.append(1)
                    if order >= 2 and i == b:
                        dirs.append(2)
                    if order >= 3 and i == c:
                        dirs.append(3)
                    p = _lift(x[i], order, dirs)
                    p[1:] *= eps
                    env[s.name] = MultiComplex(p)
                z = _eval_mc(expr, env)
                z = z if isinstance(z, MultiComplex) else MultiComplex.promote(float(z), order)
                got.append(z.im(set(range(1, order + 1))) / eps ** order)
            for k in range(3):
                scale = max(abs(want[k]), 1e-3)
                assert abs(got[k] - want[k]) <= 1e-10 * scale, (case, eps, k, str(expr), got[k], want[k])
            checked += 1
    assert checked == 80
    assert time.time() - t0 < 60
