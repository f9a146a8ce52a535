"""Synthetic inputs match SURVEY.md §8d sizes; meshes are valid."""

import numpy as np
import pytest

from paper_2102_11026_b200 import synth


@pytest.mark.parametrize("name,N,T", [("cfg1", 960, 1080), ("cfg2", 6720, 10290), ("cfg4", 1728, 1944)])
def test_sizes(name, N, T):
    cfg = synth.CONFIGS[name]
    verts, tets, fixed = synth.box_mesh(*cfg.mesh, h=cfg.h)
    assert 3 * int((~fixed).sum()) == N and tets.shape[0] == T
    X = verts[tets]
    det = np.linalg.det(np.transpose(X[:, 1:] - X[:, :1], (0, 2, 1)))
    assert np.all(det > 0)
    assert np.isclose(det.sum() / 6.0, np.prod(np.array(cfg.mesh) * cfg.h))


def test_decoder_rest_pose_and_determinism():
    Ws, bs = synth.decoder_weights(5, 40, 5, 960)
    h = np.zeros(5)
    for l in range(4):
        h = np.sin(Ws[l] @ h + bs[l])
    assert np.abs(Ws[-1] @ h + bs[-1]).max() < 1e-15
    Ws2, _ = synth.decoder_weights(5, 40, 5, 960)
    assert all(np.array_equal(a, b) for a, b in zip(Ws, Ws2))
    U = synth.pca_like_basis(960, 10)
    assert np.abs(U.T @ U - np.eye(10)).max() < 1e-12
