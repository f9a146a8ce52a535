"""cfg4 (320-string puffer ball) Newton iterations for ncu launch lists of the coupled path:
python tools/cfg4_step.py [strings] [iters]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2102_11026_b200.problem import build_problem
from paper_2102_11026_b200 import rdsim, synth
from paper_2102_11026_b200.substructure import Core, Scene

k = int(sys.argv[1]) if len(sys.argv) > 1 else 320
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 2
P = build_problem("cfg4")
R = synth.string_frames(k)
f_world = np.tile(P.f_ext, (k, 1))
m_core = 2.0 * float(P.model.mass[0::3].sum())
sc = Scene(P.rm, P.model, P.cm, R, f_world, Core(m_core, 50.0, np.array([0.0, -9.81 * m_core, 0.0])))
rb, rdb, cb, cdb = synth.coupled_state(k, P.cfg.n_p, P.cfg.n_q)
cfg = rdsim.SimConfig(dt=P.cfg.dt, fixed_iters=1)
sc.step(rb, rdb, cb, cdb, cfg)
sc.begin(rb, rdb, cb, cdb, cfg)
for _ in range(iters):
    sc.eval(True)
    sc.reduce()
    sc.update(1, 1.0)
print("cfg4_step done", flush=True)
