"""DAE training (SPEC.md:159-167 adam_train, 456-464 build_dae) and the
acceptance criteria that need it: #10 orthogonal-subspace constraint on a trained decoder and
#11 depth benefit (GPU: torch fp64 on cuda)."""

import numpy as np
import pytest

from paper_2102_11026_b200.densenet import DenseNet, LayerSpec, TrainConfig, adam_train, init_weights, lr_at
from paper_2102_11026_b200.posegen import PoseSet


def _linear_net(seed=0):
    L = [LayerSpec("fully_connected", 3, 2)]
    W, b = init_weights(L, seed)
    return DenseNet(L, W, b, seed=seed)


def test_lr_schedule_example():
    cfg = TrainConfig(learning_rate=1e-3, schedule={300: 0.8, 3000: 0.8})
    assert lr_at(cfg, 0) == 1e-3 and lr_at(cfg, 299) == 1e-3
    assert lr_at(cfg, 300) == pytest.approx(8e-4)
    assert lr_at(cfg, 3000) == pytest.approx(6.4e-4)


def test_adam_linear_exact_data():
    rng = np.random.default_rng(0)
    X = rng.standard_normal((64, 3))
    Y = X @ rng.standard_normal((2, 3)).T + 0.3
    _, curve = adam_train(_linear_net(), (X, Y), "mse",
                          TrainConfig(learning_rate=0.03, epochs=500, batch_size=16, schedule={}), device="cpu")
    assert curve[-1] < 1e-8


def test_adam_zero_weights_and_nan():
    rng = np.random.default_rng(1)
    X, Y = rng.standard_normal((16, 3)), rng.standard_normal((16, 2))
    net = _linear_net()
    out, _ = adam_train(net, (X, Y), "mse",
                        TrainConfig(epochs=5, batch_size=4, sample_weights=np.zeros(16)), device="cpu")
    assert np.array_equal(out.weights[0], net.weights[0]) and np.array_equal(out.biases[0], net.biases[0])
    Y[3, 1] = np.nan
    with pytest.raises(FloatingPointError):
        adam_train(net, (X, Y), "mse", TrainConfig(epochs=2, batch_size=4), device="cpu")


def bend_family(n_pts=40, T=300, seed=0):
    """Synthetic 2-parameter nonlinear pose family: a rod bent with curvature k in one plane and
    a k-modulated out-of-plane sweep t2 (displacements of n_pts points, N = 3 n_pts)."""
    rng = np.random.default_rng(seed)
    s = np.linspace(0, 1, n_pts)
    P = []
    for k, t2 in zip(rng.uniform(-3, 3, T), rng.uniform(-1, 1, T)):
        k = k if abs(k) > 1e-6 else 1e-6
        P.append(np.stack([np.sin(k * s) / k - s, (1 - np.cos(k * s)) / k, t2 * s ** 2 * np.cos(k * s)], 1).ravel())
    return np.array(P).T


def test_build_dae_span_and_orthogonality():
    """Poses in span(U): the decoder learns ~0; the filter keeps U^T D(q) = 0 for
    any q (acceptance #10), checked on 1000 random latent codes."""
    import torch
    from paper_2102_11026_b200.daereduce import DAEArch, build_dae
    from paper_2102_11026_b200.densenet import _torch_forward
    rng = np.random.default_rng(2)
    N = 30
    U = np.linalg.qr(rng.standard_normal((N, 2)))[0]
    X = U @ rng.standard_normal((2, 80))
    rm = build_dae(PoseSet(X, np.ones(80)), U, DAEArch(depth=4, n_q=2, width=12),
                   TrainConfig(learning_rate=3e-3, epochs=150, batch_size=16, schedule={}), seed=0, device="cpu")
    assert rm.loss_curve[-1] < 1e-2 * rm.loss_curve[0]
    q = torch.as_tensor(rng.uniform(-2, 2, (1000, 2)), dtype=torch.float64)
    p = {i: (torch.as_tensor(rm.decoder.weights[i]), torch.as_tensor(rm.decoder.biases[i])) for i in rm.decoder.weights}
    D = _torch_forward(rm.decoder, p, q).numpy()
    ratio = np.linalg.norm(D @ U, axis=1) / (np.linalg.norm(D, axis=1) + 1.0)
    assert ratio.max() <= 1e-8


@pytest.mark.gpu
def test_depth_benefit_acceptance_11(cuda_ok):
    """Acceptance #11 (Fig. 7): on a 2-parameter bend family (N = 120), an
    8-layer DAE reaches a final training loss <= a 4-layer DAE's, and <= 50% of the PCA-only
    residual (mean squared) at equal total dims (n_p + n_q = 3), median over 3 seeds."""
    from paper_2102_11026_b200.daereduce import DAEArch, build_dae
    X = bend_family()
    N, T = X.shape
    Uf = np.linalg.svd(X, full_matrices=False)[0]
    U = Uf[:, :1]
    R3 = X - Uf[:, :3] @ (Uf[:, :3].T @ X)
    pca_mse = float((R3 ** 2).mean())
    cfg = TrainConfig(learning_rate=3e-3, epochs=800, batch_size=32, schedule={400: 0.5})
    final = {}
    for depth in (4, 8):
        final[depth] = float(np.median([
            build_dae(PoseSet(X, np.ones(T)), U, DAEArch(depth=depth, n_q=2, width=24), cfg, seed=s,
                      device="cuda").loss_curve[-1] for s in range(3)]))
    assert final[8] <= final[4], final
    assert final[8] <= 0.5 * pca_mse, (final, pca_mse)
