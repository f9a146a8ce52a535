#!/usr/bin/env python
"""Cubature kernel throughput at many sims (cfg5 / cfg4 style): device ms of one k_cubature
launch over all sims and SURVEY.md 8d's algorithmic bytes / ms against the HBM peak.

    NLROM_PATH=cpc=1 python tools/bench_cubature.py [--cfg cfg5] [--sims 4096]
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cfg", default="cfg5")
    ap.add_argument("--sims", type=int, nargs="+", default=[4096])
    ap.add_argument("--iters", type=int, default=10)
    args = ap.parse_args()
    from paper_2102_11026_b200.problem import build_problem
    from paper_2102_11026_b200 import rdsim
    from paper_2102_11026_b200.session import Session
    P = build_problem(args.cfg)
    hbm = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))).get("hbm_gbs", 6553.0) \
        if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6553.0
    n = P.cfg.n_p + P.cfg.n_q
    for ns in args.sims:
        rng = np.random.default_rng(4)
        s = Session(P.rm, P.model, P.cm, n_sims=ns)
        s.step(rng.uniform(-0.05, 0.05, ns * n), rng.uniform(-0.1, 0.1, ns * n), np.tile(P.f_ext, ns),
               rdsim.SimConfig(dt=P.cfg.dt, fixed_iters=1))
        s.bench_cubature(2)
        ms, by = s.bench_cubature(args.iters)
        tot, _ = s.bench_iterations(args.iters)
        print(json.dumps({"cfg": args.cfg, "n_sims": ns, "cpc_env": os.environ.get("NLROM_PATH"),
                          "cubature_ms": ms, "bytes": by, "gbs": by / ms / 1e6, "frac": by / ms / 1e6 / hbm,
                          "iteration_ms": tot / args.iters}))
        del s


if __name__ == "__main__":
    main()
