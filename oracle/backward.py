"""Backward restatement for SPTT -- TEST INFRASTRUCTURE ONLY.

The reference is forward-only (pkg/README.md:186-189), so this
module restates the derivatives of the forward definitions it does have:

* tower modules: derivatives of towermod.py:110-158 w.r.t. inputs and weights.
  The weight gradients are pinned against the reference's own forward-mode
  derivative ``tm_weight_jvp`` (towermod.py:169-191) through the adjoint
  identity <g, J d> = <J^T g, d> (tests/test_oracle_golden.py).
* embedding bags: d pool / d row = 1 for every occurrence (sum / none) or
  1/len (mean), aggregated per unique row -- parity unpinned (no reference).
* optimizers: plain SGD and row-wise Adagrad (one accumulator per row, the
  mean of the squared aggregated row gradient) -- parity unpinned.

Everything is float64.
"""

from __future__ import annotations

import numpy as np

__all__ = [
    "tm_backward",
    "embedding_row_grads",
    "apply_sgd",
    "apply_rowwise_adagrad",
    "flat_model_grads",
    "bce_with_logits",
]


def tm_backward(embs: np.ndarray, cfg: dict, w, gout: np.ndarray):
    """Returns (d_embs (B, F, N), d_weights with the same structure as ``w``).

    Restates the chain rule through towermod.py:110-129 (dlrm) and
    towermod.py:132-158 (dcn).
    """
    B, F, N = embs.shape
    gout = np.asarray(gout, dtype=np.float64)
    if cfg["kind"] == "passthrough":
        return gout.reshape(B, F, N), None
    if cfg["kind"] == "dlrm":
        p_cols = w["w_flat"].shape[0]
        g1 = gout[:, :p_cols]                              # (B, pD)
        g2 = gout[:, p_cols:].reshape(B, F, -1)            # (B, F, cD)
        flat = embs.reshape(B, F * N)
        d_flat = g1 @ w["w_flat"]                          # (B, F*N)
        d_embs = d_flat.reshape(B, F, N) + g2 @ w["w_feat"]
        dw = {
            "w_flat": g1.T @ flat,
            "b_flat": g1.sum(axis=0),
            "w_feat": g2.reshape(B * F, -1).T @ embs.reshape(B * F, N),
            "b_feat": g2.reshape(B * F, -1).sum(axis=0),
        }
        return d_embs, dw
    # dcn: xl+1 = x0 * u + xl with u = xl W^T + b
    x0 = embs.reshape(B, F * N)
    xs, us = [x0], []
    for cw, cb in w["cross"]:
        u = xs[-1] @ cw.T + cb
        us.append(u)
        xs.append(x0 * u + xs[-1])
    g = gout @ w["w_proj"]                                  # d xL
    dw = {"w_proj": gout.T @ xs[-1], "b_proj": gout.sum(axis=0), "cross": []}
    dx0 = np.zeros_like(x0)
    cross_grads = []
    for layer in range(len(w["cross"]) - 1, -1, -1):
        cw, _ = w["cross"][layer]
        xl, u = xs[layer], us[layer]
        gu = g * x0
        cross_grads.append((gu.T @ xl, gu.sum(axis=0)))
        dx0 += g * u
        g = gu @ cw + g
    dx0 += g  # xs[0] is x0 itself
    dw["cross"] = cross_grads[::-1]
    return dx0.reshape(B, F, N), dw


def embedding_row_grads(rows: int, lens: np.ndarray, idx: np.ndarray, gbags: np.ndarray,
                        mode: str = "sum"):
    """Aggregate pooled-output gradients (nbags, N) onto table rows.

    Returns (unique_rows ascending, grads (U, N) float64).
    """
    lens = np.asarray(lens, dtype=np.int64)
    idx = np.asarray(idx, dtype=np.int64)
    bag_of = np.repeat(np.arange(lens.shape[0]), lens)
    g = np.asarray(gbags, dtype=np.float64)[bag_of]
    if mode == "mean":
        g = g / lens[bag_of, None]
    uniq, inv = np.unique(idx, return_inverse=True)
    out = np.zeros((uniq.shape[0], gbags.shape[1]), dtype=np.float64)
    np.add.at(out, inv, g)
    return uniq, out


def apply_sgd(table: np.ndarray, rows: np.ndarray, grads: np.ndarray, lr: float) -> np.ndarray:
    out = np.array(table, dtype=np.float64, copy=True)
    out[rows] -= lr * grads
    return out


def apply_rowwise_adagrad(table: np.ndarray, state: np.ndarray, rows: np.ndarray,
                          grads: np.ndarray, lr: float, eps: float):
    """state[r] += mean(g_r^2); w[r] -= lr * g_r / (sqrt(state[r]) + eps)."""
    w = np.array(table, dtype=np.float64, copy=True)
    s = np.array(state, dtype=np.float64, copy=True)
    s[rows] += np.mean(grads * grads, axis=1)
    w[rows] -= lr * grads / (np.sqrt(s[rows])[:, None] + eps)
    return w, s


def flat_model_grads(pooled_by_tower: dict, tm_cfgs: dict, tm_weights: dict, gouts: dict):
    """Backward of the flat (semantics-equal) model for one rank.

    pooled_by_tower {t: (B, F_t, N)}; gouts {t: (B, O_t)}.  Returns
    ({t: d_pooled}, {t: d_weights}).  SPTT is semantics-preserving (SURVEY
    Appendix B), so the distributed backward must reproduce this per rank, with
    tower weight grads summed over all ranks.
    """
    d_pooled, d_w = {}, {}
    for t, x in pooled_by_tower.items():
        cfg = tm_cfgs.get(t) or {"kind": "passthrough"}
        d_pooled[t], d_w[t] = tm_backward(x, cfg, tm_weights.get(t), gouts[t])
    return d_pooled, d_w


def bce_with_logits(z: np.ndarray, y: np.ndarray, scale: float):
    """Loss head of the full model step (no reference counterpart -- parity
    unpinned): loss = scale * sum(max(z,0) - z y + log1p(exp(-|z|))),
    dz = scale * (sigmoid(z) - y)."""
    z = np.asarray(z, dtype=np.float64)
    y = np.asarray(y, dtype=np.float64).reshape(z.shape)
    loss = scale * float(np.sum(np.maximum(z, 0) - z * y + np.log1p(np.exp(-np.abs(z)))))
    return loss, scale * (1.0 / (1.0 + np.exp(-z)) - y)
