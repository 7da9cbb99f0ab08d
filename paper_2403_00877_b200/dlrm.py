"""DLRM with SPTT -- the C3 model.

    dense features (B, d_in) -> bottom MLP (ReLU) ------------------------ h (B, D)
    sparse KJT -> SPTT (pooled lookup, DLRM tower modules, exchange) ----- e (B, F*D)
    [h | e] -> pairwise dot interaction (dmt_dot_interaction_fwd) -> z (B, D + (F+1)F/2)
    z -> top MLP (ReLU hidden layers) -> logit -> binary cross-entropy

The reference has no dense model; widths follow the paper's DLRM
setup: the tower modules emit D-wide per-feature vectors (towermod.py:102-107,
c = 1, p = 0) that interact with the bottom MLP's D-wide output.  Every matmul
is a tcgen05 GEMM (dmt_gemm) with bias + ReLU fused in the forward epilogue and
the ReLU mask fused in the backward dX epilogue; the interaction runs on the
CUDA cores.  The dense arch is data parallel: its fp32 gradients are
all-reduced over the world and applied by SGD on a side stream while the
embedding update runs (SPTT.backward's dense_hook).
"""

from __future__ import annotations

import math
from typing import Optional, Sequence

import numpy as np
import torch

from . import _lib as L
from . import kernels as K
from .errors import DomainError, ShapeError


def _pad16(n: int, es: int) -> int:
    """Row stride (elements) with 16-byte aligned rows (TMA)."""
    q = 16 // es
    return (n + q - 1) // q * q


def mlp_init(widths: Sequence[int], seed: int):
    """U(-1/sqrt(fan_in), +1/sqrt(fan_in)) weights (out, in) and biases per
    layer from default_rng([seed, layer]) -- float64 numpy, the oracle's too."""
    out = []
    for l in range(len(widths) - 1):
        rng = np.random.default_rng([seed, l])
        bound = 1.0 / math.sqrt(widths[l])
        w = rng.uniform(-bound, bound, size=(widths[l + 1], widths[l]))
        b = rng.uniform(-bound, bound, size=(widths[l + 1],))
        out.append((w, b))
    return out


class MLP:
    """Linear layers on dmt_gemm: y_l = relu(x_l W_l^T + b_l) (the last layer
    linear unless ``relu_last``).  fp32 weight / bias gradients."""

    def __init__(self, widths: Sequence[int], relu_last: bool, dtype: torch.dtype, device, seed: int = 0):
        if len(widths) < 2:
            raise DomainError("an MLP needs at least one layer")
        self.widths = list(widths)
        self.relu_last = relu_last
        self.dtype, self.device = dtype, device
        self.nl = len(widths) - 1
        self.w, self.b = [], []
        for wl, bl in mlp_init(widths, seed):
            self.w.append(torch.as_tensor(wl, device=device).to(dtype).contiguous())
            self.b.append(torch.as_tensor(bl, device=device).float().contiguous())
        self.grads: dict = {}
        self._saved = None
        self._buf: dict = {}

    def relu(self, l: int) -> bool:
        return l < self.nl - 1 or self.relu_last

    def _act(self, name: str, rows: int, cols: int, pad: bool = True) -> torch.Tensor:
        """Persistent activation buffer; ``pad``: 16-byte aligned row stride
        (it feeds a GEMM as an operand), else contiguous."""
        key = (name, rows, cols, pad)
        t = self._buf.get(key)
        if t is None:
            es = torch.empty((), dtype=self.dtype).element_size()
            ld = _pad16(cols, es) if pad else cols
            t = torch.zeros((rows, ld), dtype=self.dtype, device=self.device)[:, :cols]
            self._buf[key] = t
        return t

    def forward(self, x: torch.Tensor, save: bool = True) -> torch.Tensor:
        if x.shape[1] != self.widths[0]:
            raise ShapeError(f"MLP input width {x.shape[1]} != {self.widths[0]}")
        rows = x.shape[0]
        xs = [x]
        for l in range(self.nl):
            y = self._act(f"y{l}", rows, self.widths[l + 1], pad=l < self.nl - 1)
            K.gemm(xs[-1], self.w[l], y, bias=self.b[l], epilogue=L.EPI_BIAS_RELU if self.relu(l) else L.EPI_BIAS)
            xs.append(y)
        if save:
            self._saved = xs
        return xs[-1]

    def backward(self, dy: torch.Tensor, need_dx: bool = False) -> Optional[torch.Tensor]:
        """dy = dL/d(output).  Leaves fp32 grads in self.grads (w0, b0, ...);
        returns dL/d(input) when ``need_dx``."""
        xs = self._saved
        if xs is None:
            raise DomainError("MLP.backward() needs forward(save=True)")
        rows = dy.shape[0]
        f32 = torch.float32
        dz = K.relu_bwd(dy.contiguous(), xs[-1].contiguous()) if self.relu(self.nl - 1) else dy
        dx = None
        for l in range(self.nl - 1, -1, -1):
            self.grads[f"w{l}"] = K.gemm(dz, xs[l], torch.empty(self.w[l].shape, dtype=f32, device=self.device),
                                         trans_a=True, trans_b=True)
            self.grads[f"b{l}"] = K.column_sum(dz)
            if l > 0:
                # dz of layer l-1 = (dz_l W_l) masked by layer l-1's ReLU output
                nxt = self._act(f"dz{l - 1}", rows, self.widths[l])
                K.gemm(dz, self.w[l], nxt, trans_b=True, epilogue=L.EPI_RELU_BWD, x0=xs[l])
                dz = nxt
            elif need_dx:
                dx = self._act("dx", rows, self.widths[0])
                K.gemm(dz, self.w[0], dx, trans_b=True)
        return dx

    def sgd_step(self, lr: float) -> None:
        for l in range(self.nl):
            K.sgd_dense(self.w[l], self.grads[f"w{l}"].contiguous(), lr)
            K.sgd_dense(self.b[l], self.grads[f"b{l}"].contiguous(), lr)

    def host_weights(self):
        return [(self.w[l].double().cpu().numpy(), self.b[l].double().cpu().numpy()) for l in range(self.nl)]


class DLRM:
    """DLRM (MLP interaction) around an SPTT embedding module.

    ``sptt``: an SPTT whose output is F vectors of width D per sample (DLRM
    tower modules with per_feature_outputs = 1, flat_outputs = 0 and out_dim
    D, or pass-through towers with embedding dim D).  ``dense_in``: dense
    feature count; ``bottom`` / ``top``: hidden widths (bottom ends in D, top
    in one logit)."""

    def __init__(self, sptt, dense_in: int, bottom: Sequence[int] = (512, 256), top: Sequence[int] = (512, 256),
                 seed: int = 0):
        self.sptt = sptt
        self.device, self.dtype = sptt.device, sptt.engine.dtype
        dims = self._vector_dim()
        self.D, self.F = dims
        self.bottom = MLP([dense_in, *bottom, self.D], True, self.dtype, self.device, seed=seed * 2 + 101)
        self.P = (self.F + 1) * self.F // 2
        self.top = MLP([self.D + self.P, *top, 1], False, self.dtype, self.device, seed=seed * 2 + 102)
        self._z: dict = {}
        self._loss: dict = {}

    def _vector_dim(self):
        sp = self.sptt
        p = sp.plan
        D = None
        if p.feature_towers is None:  # the flat baseline: the raw embeddings interact
            ds = {p.dims[f] for f in p.features}
            if len(ds) != 1 or sp.global_tm is not None:
                raise DomainError("flat DLRM needs one embedding dim and no global tower module")
            D = ds.pop()
            return D, sp.out_width // D
        for t in range(p.T):
            cfg = sp.tm_cfg[t]
            if cfg.kind == "dlrm":
                if cfg.flat_outputs or cfg.per_feature_outputs != 1:
                    raise DomainError("DLRM interaction needs per-feature tower outputs (c = 1, p = 0)")
                d = cfg.out_dim
            elif cfg.kind == "passthrough":
                ds = {p.dims[f] for f in p.tower_features[t]}
                if len(ds) > 1:
                    raise DomainError("pass-through tower mixes embedding dims")
                d = ds.pop() if ds else None
            else:
                raise DomainError(f"DLRM interaction cannot consume {cfg.kind!r} tower outputs")
            if d is not None:
                if D is not None and d != D:
                    raise DomainError("all towers must emit vectors of one width")
                D = d
        width = sp.out_width
        if D is None or width % D:
            raise DomainError("SPTT output is not a whole number of vectors")
        return D, width // D

    def _zbuf(self, r: int, rows: int) -> torch.Tensor:
        z = self._z.get(r)
        if z is None:
            es = torch.empty((), dtype=self.dtype).element_size()
            w = self.D + self.P
            z = torch.zeros((rows, _pad16(w, es)), dtype=self.dtype, device=self.device)[:, :w]
            self._z[r] = z
        return z

    def train_step(self, kjts: dict, dense_x: dict, labels: dict) -> dict:
        """One step: forward, BCE (mean over the global batch), backward, SGD on
        the dense arch (world all-reduce, overlapped with the embedding update)
        and the fused embedding update.  Returns {rank: loss (1,)} (rank r's
        share of the global mean loss)."""
        sp = self.sptt
        emb = sp.forward(kjts, save=True)
        G, B = sp.plan.G, sp.plan.B
        scale = 1.0 / (G * B)
        d_emb, acc, losses, saved = {}, {}, {}, {}
        for r, e in emb.items():
            h = self.bottom.forward(dense_x[r])
            bsave = self.bottom._saved
            z = K.dot_interaction_fwd(h, e, self.F, out=self._zbuf(r, e.shape[0]))
            logit = self.top.forward(z)
            buf = self._loss.get(r)
            if buf is None:
                buf = self._loss[r] = (torch.empty_like(logit), torch.zeros(1, dtype=torch.float32, device=self.device))
            K.bce_with_logits(logit, labels[r], scale, dz=buf[0], loss=buf[1])
            losses[r] = buf[1]
            dz = self.top.backward(buf[0], need_dx=True)
            dh, d_emb[r] = K.dot_interaction_bwd(dz, h, e, self.F)
            self.bottom._saved = bsave
            self.bottom.backward(dh)
            for mlp, tag in ((self.bottom, "bot_"), (self.top, "top_")):
                for k, v in mlp.grads.items():
                    acc[tag + k] = v.clone() if tag + k not in acc else acc[tag + k].add_(v)

        def dense_step():  # world all-reduce of the dense grads + SGD
            sp.fabric.all_reduce_(list(range(G)), acc)
            for mlp, tag in ((self.bottom, "bot_"), (self.top, "top_")):
                mlp.grads = {k[len(tag):]: v for k, v in acc.items() if k.startswith(tag)}
                mlp.sgd_step(sp.dense_lr)

        sp.backward(d_emb, dense_hook=dense_step)
        return losses

    def capture(self, kjts: dict, dense_x: dict, labels: dict, warmup: int = 2, timers=None):
        """CUDA-graph capture of train_step over static input buffers (see
        SPTT.capture); returns (replay, losses)."""
        return self.sptt.capture(kjts, None, warmup=warmup, timers=timers,
                                 step=lambda: self.train_step(kjts, dense_x, labels))

    def mlp_flops(self, rows: int) -> float:
        """Forward + backward (dX, dW) matmul flops of the dense arch."""
        fl = 0.0
        for mlp in (self.bottom, self.top):
            for l in range(mlp.nl):
                fl += 3 * 2.0 * rows * mlp.widths[l] * mlp.widths[l + 1]
        return fl
