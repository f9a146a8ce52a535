"""Artifact I/O: bit-exact round trips
of densenet checkpoints, PoseSets, ReducedModel / CubatureModel directories and meshes."""

import numpy as np
import pytest

from paper_2102_11026_b200 import artifacts as io
from paper_2102_11026_b200.densenet import DenseNet, LayerSpec


@pytest.fixture(scope="module")
def tiny():
    from paper_2102_11026_b200.problem import build_problem
    return build_problem("tiny")


def _same_net(a: DenseNet, b: DenseNet):
    assert [vars(s) for s in a.layers] == [vars(s) for s in b.layers]
    for d1, d2 in ((a.weights, b.weights), (a.biases, b.biases), (a.bases, b.bases)):
        assert d1.keys() == d2.keys()
        for k in d1:
            assert np.array_equal(np.asarray(d1[k]), d2[k])  # bit-exact


def test_checkpoint_roundtrip_bit_exact(tiny, tmp_path):
    net = tiny.rm.decoder
    rng = np.random.default_rng(0)
    net.weights[0] = net.weights[0] + rng.standard_normal(net.weights[0].shape) * np.pi * 1e-7  # awkward floats
    p = tmp_path / "dec.json"
    io.save_checkpoint(net, str(p), {"epochs": 3, "loss": 0.125})
    back = io.load_checkpoint(str(p))
    _same_net(net, back)
    assert back.metadata == {"epochs": 3, "loss": 0.125}


def test_poseset_roundtrip(tmp_path):
    rng = np.random.default_rng(1)
    X = rng.standard_normal((37, 5))
    e = rng.random(5)
    p = str(tmp_path / "poses.bin")
    io.save_poseset(p, X, e, {"episodes": 2})
    Y, e2, script = io.load_poseset(p)
    assert np.array_equal(X, Y) and np.array_equal(e, e2) and script == {"episodes": 2}
    raw = open(p, "rb").read()
    assert np.frombuffer(raw[:16], dtype="<i8").tolist() == [37, 5]
    assert np.array_equal(np.frombuffer(raw[16:16 + 8 * 37], dtype="<f8"), X[:, 0])  # column-major


def test_poseset_rejects_truncated(tmp_path):
    p = str(tmp_path / "bad.bin")
    io.save_poseset(p, np.ones((4, 3)))
    with open(p, "rb+") as f:
        f.truncate(40)
    with pytest.raises(ValueError):
        io.load_poseset(p)


def test_reduced_and_cubature_models_roundtrip(tiny, tmp_path):
    io.save_reduced_model(tiny.rm, str(tmp_path / "rm"))
    rm2 = io.load_reduced_model(str(tmp_path / "rm"))
    assert rm2.n_p == tiny.rm.n_p and rm2.n_q == tiny.rm.n_q
    assert np.array_equal(rm2.U, tiny.rm.U)
    _same_net(tiny.rm.decoder, rm2.decoder)
    io.save_cubature_model(tiny.cm, str(tmp_path / "cm"))
    cm2 = io.load_cubature_model(str(tmp_path / "cm"))
    assert np.array_equal(cm2.C, tiny.cm.C)
    _same_net(tiny.cm.wnet, cm2.wnet)


def test_mesh_roundtrip(tiny, tmp_path):
    from paper_2102_11026_b200.elastic import TetMesh
    m = tiny.model.mesh
    mesh = TetMesh(m.vertices * (1 + 1e-9), m.tets, np.array([[0, 1, 2], [1, 2, 3]]))
    p = str(tmp_path / "mesh.txt")
    io.write_mesh(mesh, p)
    back = io.read_mesh(p)
    assert np.array_equal(back.vertices, mesh.vertices) and np.array_equal(back.tets, mesh.tets)
    assert np.array_equal(back.surface, mesh.surface)
    assert open(p).readline().split() == [str(m.vertices.shape[0]), str(m.tets.shape[0])]
