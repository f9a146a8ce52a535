#!/usr/bin/env python
"""In-graph critical-path attribution of one Newton iteration: marginal device time of each
launch, from prefix graphs (nlrom_bench_prefix). Usage: python tools/prefix_profile.py [cfg2]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
    from paper_2102_11026_b200.problem import build_problem
    from paper_2102_11026_b200 import rdsim
    from paper_2102_11026_b200.session import Session
    P = build_problem(name)
    s = Session(P.rm, P.model, P.cm)
    r, rb, rdb = P.random_state()
    s.step(rb, rdb, P.f_ext, rdsim.SimConfig(dt=P.cfg.dt, fixed_iters=1))
    rows, cum = s.bench_prefix(n_iters=100)
    tot, _ = s.bench_iterations(100)
    print(f"{name}: full graph {tot / 100 * 1e3:.1f} us per Newton iteration; prefix total {cum[-1] * 1e3:.1f} us")
    for i, (nm, d) in enumerate(rows):
        short = nm.split("(")[0].replace("void ", "").replace("nlrom::", "")
        print(f"{i + 1:3d} {d * 1e3:8.2f} us  cum {cum[i] * 1e3:8.2f}  {short[:100]}")


if __name__ == "__main__":
    main()
