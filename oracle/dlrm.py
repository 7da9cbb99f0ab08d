"""DLRM dense arch restatement -- TEST INFRASTRUCTURE ONLY (float64 numpy).

The reference has no dense model; the C3 model follows the
paper's DLRM with SPTT and TorchRec's DLRM:
bottom MLP (ReLU) -> pairwise dot interaction of [bottom output | per-feature
SPTT vectors] (strict lower triangle, row-major) -> top MLP (ReLU hidden
layers, linear logit) -> BCE.  Parity unpinned (no reference counterpart):
the GPU model is checked against this restatement within the north-star
tolerance.
"""

from __future__ import annotations

import numpy as np

__all__ = ["mlp_forward", "mlp_backward", "interaction_forward", "interaction_backward", "dlrm_step"]


def mlp_forward(x, layers, relu_last: bool):
    """layers [(W (out, in), b)]; returns (y, saved activations [x_0 .. x_L])."""
    xs = [np.asarray(x, dtype=np.float64)]
    for l, (w, b) in enumerate(layers):
        z = xs[-1] @ w.T + b
        if l < len(layers) - 1 or relu_last:
            z = np.maximum(z, 0.0)
        xs.append(z)
    return xs[-1], xs


def mlp_backward(xs, layers, relu_last: bool, dy):
    """Returns (dx, [(dW, db)])."""
    g = np.asarray(dy, dtype=np.float64)
    grads = [None] * len(layers)
    for l in range(len(layers) - 1, -1, -1):
        w, _ = layers[l]
        if l < len(layers) - 1 or relu_last:
            g = g * (xs[l + 1] > 0)
        grads[l] = (g.T @ xs[l], g.sum(axis=0))
        g = g @ w
    return g, grads


def _pairs(nv: int):
    return [(i, j) for i in range(1, nv) for j in range(i)]


def interaction_forward(dense, sparse, num_sparse: int):
    B, D = dense.shape
    v = np.concatenate([dense[:, None, :], sparse.reshape(B, num_sparse, D)], axis=1)
    pairs = _pairs(num_sparse + 1)
    dots = (np.stack([np.einsum("bd,bd->b", v[:, i], v[:, j]) for i, j in pairs], axis=1) if pairs
            else np.zeros((B, 0)))
    return np.concatenate([dense, dots], axis=1)


def interaction_backward(gout, dense, sparse, num_sparse: int):
    B, D = dense.shape
    v = np.concatenate([dense[:, None, :], sparse.reshape(B, num_sparse, D)], axis=1)
    dv = np.zeros_like(v)
    dv[:, 0] += gout[:, :D]
    for p, (i, j) in enumerate(_pairs(num_sparse + 1)):
        g = gout[:, D + p][:, None]
        dv[:, i] += g * v[:, j]
        dv[:, j] += g * v[:, i]
    return dv[:, 0], dv[:, 1:].reshape(B, num_sparse * D)


def dlrm_step(dense_x, emb, labels, bottom, top, num_sparse: int, scale: float):
    """Forward + backward of one rank's dense arch given its SPTT output
    ``emb`` (B, F*D).  Returns (loss, d_emb, bottom grads, top grads)."""
    h, hs = mlp_forward(dense_x, bottom, True)
    z = interaction_forward(h, emb, num_sparse)
    logit, ts = mlp_forward(z, top, False)
    y = np.asarray(labels, dtype=np.float64).reshape(logit.shape)
    loss = scale * float(np.sum(np.maximum(logit, 0) - logit * y + np.log1p(np.exp(-np.abs(logit)))))
    dlogit = scale * (1.0 / (1.0 + np.exp(-logit)) - y)
    dz, tg = mlp_backward(ts, top, False, dlogit)
    dh, demb = interaction_backward(dz, h, emb, num_sparse)
    _, bg = mlp_backward(hs, bottom, True, dh)
    return loss, demb, bg, tg
