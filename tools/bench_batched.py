#!/usr/bin/env python
"""Throughput of n_sims independent simulations in one context (cfg5-style).

    python tools/bench_batched.py [--cfg cfg5] [--sims 512 4096] [--iters 20]

Prints one JSON line per sim count: device ms per Newton iteration (all sims, one graph
replay), sim-iterations/s, the per-stage split, and the §8d decoder roofline
F_dec = (18 n_q + 6)(2 sum_l in_l out_l + 4 N n_p) per sim against the measured fp64 DMMA peak.
"""

from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def f_dec(P):
    c = P.cfg
    widths = [c.n_q] + [c.width] * (c.n_fc - 1) + [P.model.N]
    mac = sum(a * b for a, b in zip(widths[:-1], widths[1:]))
    return (18 * c.n_q + 6) * (2.0 * mac + 4.0 * P.model.N * c.n_p)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cfg", default="cfg5")
    ap.add_argument("--sims", type=int, nargs="+", default=[512, 4096])
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--flush", type=int, default=1)
    args = ap.parse_args()
    from paper_2102_11026_b200.problem import build_problem
    from paper_2102_11026_b200 import rdsim
    from paper_2102_11026_b200.session import Session
    P = build_problem(args.cfg)
    fp64 = json.load(open(os.path.join(ROOT, "profiles", "fp64_peak.json")))["dmma_tflops"]
    n = P.cfg.n_p + P.cfg.n_q
    for ns in args.sims:
        s = Session(P.rm, P.model, P.cm, n_sims=ns)
        states = [P.random_state(seed=4 + i) for i in range(ns)]
        rb = np.concatenate([st[1] for st in states]) * 0.1
        rdb = np.concatenate([st[2] for st in states]) * 0.1
        fext = np.tile(P.f_ext, ns)
        cfg = rdsim.SimConfig(dt=P.cfg.dt, fixed_iters=1)
        s.step(rb, rdb, fext, cfg)
        s.bench_iterations(3, flush_l2=bool(args.flush))
        tot, _ = s.bench_iterations(args.iters, flush_l2=bool(args.flush))
        ms = tot / args.iters
        stages = s.bench_kernels(max(3, args.iters // 4), flush_l2=bool(args.flush))
        dec_ms = stages[0] + stages[1] + stages[2]
        F = f_dec(P) * ns
        print(json.dumps({
            "cfg": args.cfg, "n_sims": ns, "ms_per_iteration": ms, "sim_iters_per_s": ns * 1e3 / ms,
            "stages_ms": {"jet_fwd": stages[0], "output": stages[1], "vhp_bwd": stages[2], "lu": stages[3]},
            "decoder_ms": dec_ms, "F_dec_tflop": F / 1e12,
            "decoder_tflops_alg": F / (dec_ms * 1e-3) / 1e12, "frac_of_dmma_peak": F / (dec_ms * 1e-3) / 1e12 / fp64,
            "step_tflops_alg": F / (ms * 1e-3) / 1e12, "launches": s.launches_per_iteration(),
        }), flush=True)
        del s


if __name__ == "__main__":
    main()
