"""Full-space implicit Euler timing (elastic.fullspace_step on the GPU) at the cfg2 mesh
(N = 6720) and the cfg4 string mesh: gravity from rest, wall clock per step (host arrays in
and out), Newton and PCG iteration counts; the scipy oracle timed on one step beside it."""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def run(name, steps=6, **kw):
    from paper_2102_11026_b200.problem import build_problem
    from paper_2102_11026_b200.fullspace import FullspaceConfig, FullspaceSession
    from helpers import oracle_sim
    from oracle import fullspace as ofs
    P = build_problem(name, **kw)
    s = FullspaceSession(P.model)
    cfg = FullspaceConfig()
    u = v = np.zeros(P.model.N)
    u, v, _ = s.step(u, v, P.f_ext, P.cfg.dt, cfg)  # warm-up
    ts, its, cgs = [], [], []
    for _ in range(steps):
        t0 = time.perf_counter()
        u, v, info = s.step(u, v, P.f_ext, P.cfg.dt, cfg)
        ts.append(time.perf_counter() - t0)
        its.append(info.iters)
        cgs.append(info.cg_iters)
    om = oracle_sim(P).model
    t0 = time.perf_counter()
    ofs.fullspace_step(om, u, v, P.f_ext, P.cfg.dt)
    t_cpu = time.perf_counter() - t0
    ms = 1e3 * float(np.median(ts))
    return {"mesh": name, "N": P.model.N, "tets": P.model.n_tets, "ms_per_step": ms,
            "newton_iters": its, "cg_iters": cgs,
            "us_per_cg_iter": 1e3 * sum(1e3 * t for t in ts) / max(1, sum(cgs)),
            "oracle_ms_per_step": 1e3 * t_cpu}


if __name__ == "__main__":
    out = [run("cfg2", n_fc=2, width=16), run("cfg1")]
    for o in out:
        print(json.dumps(o))
