"""One line of tools/skip_sweep.sh: cfg2 device ms per Newton iteration (graph replays, L2 flushed)
with NLROM_DEBUG_SKIP as set in the environment (experiment library only)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2102_11026_b200.problem import build_problem  # noqa: E402
from paper_2102_11026_b200 import rdsim  # noqa: E402
from paper_2102_11026_b200.session import Session  # noqa: E402

P = build_problem("cfg2")
s = Session(P.rm, P.model, P.cm)
st = P.rest_state()
s.step(st.r, st.rdot, P.f_ext, rdsim.SimConfig(dt=P.cfg.dt, fixed_iters=1))
s.bench_replays(20)
ms = s.bench_replays(200)
print(f"skip=[{os.environ.get('NLROM_DEBUG_SKIP', '')}] ms={np.mean(ms):.4f}", flush=True)
