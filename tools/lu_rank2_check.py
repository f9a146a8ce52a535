"""Bitwise comparison of an opt-in LU variant with the default row-block LU over 3
fixed-iteration steps on several configs (fresh process per variant). Variant = the env switch
in argv[1]: NLROM_LU_RANK2 (csrc/lu_rank2.cuh, the default) or NLROM_LU_LA (k_lu_la)."""
import os, sys, subprocess, numpy as np
root = "/root/repo" if os.path.exists("/root/repo") else os.environ["GRAFT_REPO_ROOT"]
code = r'''
import sys, numpy as np
sys.path.insert(0, sys.argv[1])
from paper_2102_11026_b200.problem import build_problem
from paper_2102_11026_b200 import rdsim
out = {}
for name, kw in [("cfg2", {}), ("cfg1", {}), ("cfg2", {"n_q": 31}), ("cfg2", {"n_q": 64, "n_fc": 4})]:
    P = build_problem(name, **kw)
    st = P.rest_state()
    cfg = rdsim.SimConfig(dt=P.cfg.dt, fixed_iters=3)
    for i in range(3):
        st = rdsim.step(P.rm, P.model, st, P.f_ext, cfg)
    out[name + str(kw)] = st.r
np.savez(sys.argv[2], **{k.replace(" ", ""): v for k, v in out.items()})
'''
VAR = sys.argv[1] if len(sys.argv) > 1 else "NLROM_LU_RANK2"
res = {}
for env in ("0", "1"):
    e = dict(os.environ)
    if env == "1": e[VAR] = "1"
    f = f"/tmp/lu_{env}.npz"
    subprocess.run([sys.executable, "-c", code, root, f], env=e, check=True)
    res[env] = np.load(f)
for k in res["0"].files:
    a, b = res["0"][k], res["1"][k]
    print(k, "bitwise" if np.array_equal(a, b) else f"max rel diff {np.abs(a-b).max()/np.abs(a).max():.3e}")
