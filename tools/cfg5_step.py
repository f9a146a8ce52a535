"""One cfg5 (4096 independent sims) Newton iteration graph, for ncu captures of the batched
kernels: python tools/cfg5_step.py [n_sims] [iters]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2102_11026_b200.problem import build_problem
from paper_2102_11026_b200 import rdsim
from paper_2102_11026_b200.session import Session

ns = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 1
P = build_problem("cfg5")
n = P.cfg.n_p + P.cfg.n_q
rng = np.random.default_rng(4)
s = Session(P.rm, P.model, P.cm, n_sims=ns)
s.step(rng.uniform(-0.05, 0.05, ns * n), rng.uniform(-0.1, 0.1, ns * n), np.tile(P.f_ext, ns),
       rdsim.SimConfig(dt=P.cfg.dt, fixed_iters=1))
s.iterate(iters)
print("cfg5_step done", flush=True)
