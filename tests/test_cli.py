"""nlrom CLI: argument / config handling and the OBJ surface export on CPU;
the whole gen-data -> train-dae -> train-cubature -> simulate -> validate -> bench pipeline on
the GPU (tiny box mesh)."""

import json
import os

import numpy as np
import pytest

from paper_2102_11026_b200 import cli, synth


def test_help_and_input_errors(tmp_path, capsys):
    assert cli.main(["--help"]) == 0
    assert cli.main(["no-such-command"]) == 2
    assert cli.main(["simulate", "--config", str(tmp_path / "missing.json")]) == cli.EXIT_INPUT
    bad = tmp_path / "bad.json"
    bad.write_text("{not json")
    assert cli.main(["train-dae", "--config", str(bad)]) == cli.EXIT_INPUT
    cfgp = tmp_path / "cfg.json"
    cfgp.write_text(json.dumps({"mesh": {"box": [2, 0, 1]}}))
    assert cli.main(["gen-data", "--config", str(cfgp), "--out", str(tmp_path / "o")]) == cli.EXIT_INPUT


def test_config_overrides(tmp_path):
    cfgp = tmp_path / "cfg.json"
    cfgp.write_text(json.dumps({"out": "a", "seed": 3, "sim": {"steps": 5}}))
    args = cli.parser().parse_args(["simulate", "--config", str(cfgp), "--seed", "7", "--out", "b", "--drop-fict",
                                    "--exact"])
    cfg = cli.load_config(args)
    assert cfg["seed"] == 7 and cfg["out"] == "b"
    assert cfg["sim"] == {"steps": 5, "drop_fict": True, "integration": "exact_sum"}
    sc = cli.sim_config(cfg)
    assert sc.drop_fict and sc.integration == "exact_sum"


def test_surface_faces_and_obj(tmp_path):
    nx, ny, nz = 3, 2, 2
    verts, tets, _ = synth.box_mesh(nx, ny, nz, h=0.1)
    F = cli.surface_faces(tets)
    assert F.shape[0] == 4 * (nx * ny + ny * nz + nx * nz)       # 2 triangles per boundary square
    assert np.unique(np.sort(F, axis=1), axis=0).shape[0] == F.shape[0]
    # outward orientation: the signed volume of the closed surface is the box volume
    p = verts[F]
    vol = np.einsum("ij,ij->i", p[:, 0], np.cross(p[:, 1], p[:, 2])).sum() / 6.0
    assert vol == pytest.approx(nx * ny * nz * 1e-3, rel=1e-12)
    path = tmp_path / "f.obj"
    cli.write_obj(path, verts, F)
    lines = path.read_text().splitlines()
    assert sum(l.startswith("v ") for l in lines) == verts.shape[0]
    assert sum(l.startswith("f ") for l in lines) == F.shape[0]


@pytest.mark.gpu
def test_pipeline_end_to_end(cuda_ok, tmp_path, capsys):
    cfg = {"out": str(tmp_path / "run"), "seed": 1, "mesh": {"box": [6, 2, 2], "h": 0.1},
           "script": {"episodes": 4, "steps": 8, "magnitude": [20.0, 80.0]},
           "arch": {"n_p": 4, "n_q": 2, "depth": 4, "width": 16},
           "train": {"epochs": 60, "batch_size": 16, "learning_rate": 3e-3, "schedule": {}},
           "cubature": {"size": 12, "method": "greedy"},
           "sim": {"steps": 12, "frame_every": 4, "newton_tol": 1e-7, "gravity": -2.0, "integration": "exact_sum"}}
    cp = tmp_path / "run.json"
    cp.write_text(json.dumps(cfg))
    for cmd in ("gen-data", "train-dae", "train-cubature", "simulate"):
        assert cli.main([cmd, "--config", str(cp)]) == 0, cmd
    out = capsys.readouterr().out
    assert '"command": "train-dae"' in out and '"command": "simulate"' in out
    lines = [json.loads(l) for l in open(tmp_path / "run" / "sim.jsonl")]
    assert len(lines) == 12 and all(l["residual_norm"] <= 1e-7 for l in lines)
    assert len(os.listdir(tmp_path / "run" / "frames")) == 3
    assert cli.main(["validate", "--config", str(cp)]) == 0
    assert cli.main(["bench", "--config", str(cp)]) == 0
    assert '"ms_per_newton_iteration"' in capsys.readouterr().out
    # the drop_fict switch and the trained cubature set run too
    assert cli.main(["simulate", "--config", str(cp), "--drop-fict", "--out", str(tmp_path / "run")]) == 0
    cfg["sim"].update(steps=3, gravity=-0.5, newton_tol=1e-6)
    cp.write_text(json.dumps(cfg))
    assert cli.main(["simulate", "--config", str(cp), "--cubature"]) == 0
