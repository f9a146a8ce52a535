"""bench.py launch logic on CPU (no GPU): `--gpus 2` without torchrun launches two ranks
itself; the reference arm runs on rank 0 only, pins the BLAS pool to the host cores despite
torchrun's OMP_NUM_THREADS=1, and prints n_gpus 2 with the same `config` object the GPU arm
prints (bench.config_dict)."""

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_two_ranks():
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--gpus", "2",
                        "--steps", "1", "--warmup", "0"], capture_output=True, text=True, timeout=900, env=env,
                       cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    sys.path.insert(0, ROOT)
    import bench
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["warmup"] == 3
    assert d["config"] == json.loads(json.dumps(bench.config_dict(2)))
    assert d["cpu_baseline"]["cores"] == bench.host_cores()
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["value"] > 0
    assert d["higher_is_better"] is False
