"""Real multi-process multi-GPU runs (torchrun, one process per GPU, NCCL): the product's
SimShard (independent sims, no collective) and Scene (coupled strings, one allreduce per Newton
iteration) at world size 2 against the single-process oracle. Skips unless >= 2 GPUs are
visible (the round's GPU runs use one GPU; the host-side logic is covered on CPU by
tests/test_shard.py and tests/test_coupled_oracle.py)."""

import os
import socket
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

_SCRIPT = r"""
import os, sys
import numpy as np
import torch, torch.distributed as dist
sys.path[:0] = [sys.argv[1], os.path.join(sys.argv[1], "tests")]
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(int(os.environ["LOCAL_RANK"]))
os.environ["NLROM_DEVICE"] = os.environ["LOCAL_RANK"]
dist.init_process_group("nccl")
from helpers import oracle_sim, coupled_setup
from oracle import rdsim as ors, coupled as oc
from paper_2102_11026_b200.problem import build_problem
from paper_2102_11026_b200 import rdsim, synth
from paper_2102_11026_b200.shard import SimShard
from paper_2102_11026_b200.substructure import Core, Scene
P = build_problem("cfg1")
n = P.cfg.n_p + P.cfg.n_q
total = 5
rng = np.random.default_rng(4)
rb, rdb = rng.uniform(-0.05, 0.05, (total, n)), rng.uniform(-0.1, 0.1, (total, n))
cfg = rdsim.SimConfig(dt=P.cfg.dt, fixed_iters=2)
sh = SimShard(P.rm, P.model, P.cm, total)
r, _, _ = sh.step(rb, rdb, P.f_ext, cfg)
allr = sh.gather(r)
S = oracle_sim(P)
worst = 0.0
for i in range(total):
    ro, _, _, _ = ors.step(S, rb[i].copy(), rdb[i].copy(), P.f_ext, ors.OSimConfig(dt=P.cfg.dt, fixed_iters=2))
    worst = max(worst, np.abs(allr[i] - ro).max() / np.abs(ro).max())
assert worst <= 1e-10, worst
k = 4
R, f_world, m_core, k_core, f_core, osc = coupled_setup(P, k)
sc = Scene(P.rm, P.model, P.cm, R, f_world, Core(m_core, k_core, f_core))
sb, sdb, cb, cdb = synth.coupled_state(k, P.cfg.n_p, P.cfg.n_q)
r, rd, c, cd, it, nrm = sc.step(sb, sdb, cb, cdb, cfg)
ro, rdo, co, cdo, _, no = oc.step(osc, sb, sdb, cb, cdb, ors.OSimConfig(dt=P.cfg.dt, fixed_iters=2))
assert np.abs(r - ro[sc.lo:sc.hi]).max() <= 1e-10 * np.abs(ro).max()
assert np.abs(c - co).max() <= 1e-10 * np.abs(co).max()
dist.destroy_process_group()
print("RANK_OK", rank, flush=True)
"""


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_two_gpu_ranks(tmp_path):
    import torch
    if torch.cuda.device_count() < 2:
        pytest.skip("needs >= 2 visible GPUs")
    script = tmp_path / "multi.py"
    script.write_text(_SCRIPT)
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
                        "--master-addr", "127.0.0.1", "--master-port", str(_port()), str(script), ROOT],
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-3000:]
    assert r.stdout.count("RANK_OK") == 2
