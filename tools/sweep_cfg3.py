#!/usr/bin/env python
"""cfg3 sweep: cfg2 mesh, n_q in 5..64 x depth 4..16, single sim.
Prints one JSON line per point: ms per Newton iteration (graph replay, L2 flushed), per-stage
split, and the decoder roofline (F_dec / decoder time vs the measured fp64 DMMA peak)."""

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--nq", type=int, nargs="+", default=[5, 10, 20, 30, 48, 64])
    ap.add_argument("--depth", type=int, nargs="+", default=[4, 8, 12, 16])
    ap.add_argument("--iters", type=int, default=100)
    ap.add_argument("--sims", type=int, default=1, help="independent sims per context (throughput mode)")
    args = ap.parse_args()
    from paper_2102_11026_b200.problem import build_problem
    from paper_2102_11026_b200 import rdsim
    from paper_2102_11026_b200.session import Session
    _, tc = bench.peaks()
    for L in args.depth:
        for nq in args.nq:
            P = build_problem("cfg2", n_q=nq, n_fc=L)
            ns = args.sims
            s = Session(P.rm, P.model, P.cm, n_sims=ns)
            st_ = [P.random_state(seed=4 + i) for i in range(ns)]
            import numpy as np
            rb = np.concatenate([x[1] for x in st_]) * (0.1 if ns > 1 else 1.0)
            rdb = np.concatenate([x[2] for x in st_]) * (0.1 if ns > 1 else 1.0)
            s.step(rb, rdb, np.tile(P.f_ext, ns), rdsim.SimConfig(dt=P.cfg.dt, fixed_iters=1))
            s.bench_iterations(5)
            tot, _ = s.bench_iterations(args.iters)
            st = s.bench_kernels(max(10, args.iters // 4))
            roof = bench.decoder_roofline(P, st, ns, tc, s.tc_info())
            print(json.dumps({"n_q": nq, "depth": L, "n_sims": ns, "ms_per_iteration": tot / args.iters,
                              "sim_iterations_per_s": ns * 1e3 / (tot / args.iters),
                              "hz_3_iters": 1000.0 / (3 * tot / args.iters),
                              "decoder_ms": roof["kernel_ms"], "lu_ms": st[3],
                              "F_dec_gflop": roof["algorithmic"]["flops_per_launch"] / 1e9,
                              "decoder_tflops_alg": roof["algorithmic"]["tflops_equivalent"],
                              "executed_frac": roof["frac"], "pipes": roof.get("pipes"),
                              "stages_ms": roof["stages_ms"], "launches": s.launches_per_iteration()}),
                  flush=True)
            del s


if __name__ == "__main__":
    main()
