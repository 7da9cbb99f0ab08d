"""Tower modules (TM): configs, seeded weights, widths, flops and the device
forward/backward on tcgen05 GEMMs.

Host API mirrors towersim/towermod.py:23-250 (same config fields, seeded
weight draws, width / flop formulas).  ``TowerModule`` is the device
implementation: weights live in HBM in the compute dtype, every matmul is a
`dmt_gemm` launch (bf16 -> kind::f16, fp32 -> 3xTF32) with the bias /
crossnet gate fused in the epilogue, and the backward produces fp32 weight
gradients (summed over the tower's data-parallel ranks by the caller).
"""

from __future__ import annotations

import os

from dataclasses import dataclass
from typing import Optional

import numpy as np
import torch

from . import _lib as L
from . import kernels as K
from .errors import DomainError, ShapeError

PASSTHROUGH = "passthrough"
DLRM = "dlrm"
DCN = "dcn"
KINDS = (PASSTHROUGH, DLRM, DCN)


@dataclass(frozen=True)
class TMConfig:
    """towermod.py:23-51."""

    kind: str = PASSTHROUGH
    out_dim: int = 64
    per_feature_outputs: int = 1
    flat_outputs: int = 0
    cross_layers: int = 3
    seed: int = 0

    def __post_init__(self) -> None:
        if self.kind not in KINDS:
            raise DomainError(f"unknown tower module kind {self.kind!r}")
        if self.kind == DLRM:
            if self.per_feature_outputs < 0 or self.flat_outputs < 0:
                raise DomainError("per_feature_outputs and flat_outputs must be >= 0")
            if self.per_feature_outputs + self.flat_outputs < 1:
                raise DomainError("dlrm flavor needs per_feature_outputs + flat_outputs >= 1")
        if self.kind != PASSTHROUGH and self.out_dim < 1:
            raise DomainError("out_dim must be >= 1")
        if self.kind == DCN and self.cross_layers < 1:
            raise DomainError("cross_layers must be >= 1")


@dataclass(frozen=True)
class DLRMWeights:
    """towermod.py:54-59."""

    w_flat: np.ndarray  # (flat_outputs*out_dim, F*N)
    b_flat: np.ndarray
    w_feat: np.ndarray  # (per_feature_outputs*out_dim, N)
    b_feat: np.ndarray


@dataclass(frozen=True)
class DCNWeights:
    """towermod.py:62-66."""

    cross: tuple  # per layer (W: M x M, b: M)
    w_proj: np.ndarray  # (F*out_dim, M)
    b_proj: np.ndarray


def _uniform(rng, shape, fan_in):
    bound = 1.0 / np.sqrt(max(fan_in, 1))
    return rng.uniform(-bound, bound, size=shape)


def init_tm_weights(cfg: TMConfig, num_features: int, in_dim: int, salt: int = 0):
    """towermod.py:74-99: U(+-1/sqrt(fan_in)) from default_rng([seed, salt, F, N]),
    drawn in the reference's order (so weights are identical)."""
    rng = np.random.default_rng([cfg.seed, salt, num_features, in_dim])
    if cfg.kind == PASSTHROUGH:
        return None
    D = cfg.out_dim
    if cfg.kind == DLRM:
        fi = num_features * in_dim
        return DLRMWeights(
            w_flat=_uniform(rng, (cfg.flat_outputs * D, fi), fi),
            b_flat=_uniform(rng, (cfg.flat_outputs * D,), fi),
            w_feat=_uniform(rng, (cfg.per_feature_outputs * D, in_dim), in_dim),
            b_feat=_uniform(rng, (cfg.per_feature_outputs * D,), in_dim),
        )
    m = num_features * in_dim
    cross = tuple((_uniform(rng, (m, m), m), _uniform(rng, (m,), m)) for _ in range(cfg.cross_layers))
    return DCNWeights(cross=cross, w_proj=_uniform(rng, (num_features * D, m), m),
                      b_proj=_uniform(rng, (num_features * D,), m))


def tm_output_width(cfg: TMConfig, num_features: int, in_dim: int) -> int:
    """towermod.py:102-107: O = D(c|F| + p) (dlrm), |F| D (dcn), |F| N (pass-through)."""
    if cfg.kind == PASSTHROUGH:
        return num_features * in_dim
    if cfg.kind == DLRM:
        return cfg.out_dim * (cfg.per_feature_outputs * num_features + cfg.flat_outputs)
    return num_features * cfg.out_dim


def tm_flops(cfg: TMConfig, num_features: int, in_dim: int, batch: int) -> float:
    """towermod.py:194-206 (the roofline's TM flop count)."""
    if cfg.kind == PASSTHROUGH or num_features == 0:
        return 0.0
    if cfg.kind == DLRM:
        flat = num_features * in_dim
        return 2.0 * batch * (flat * cfg.flat_outputs * cfg.out_dim
                              + num_features * in_dim * cfg.per_feature_outputs * cfg.out_dim)
    m = num_features * in_dim
    return cfg.cross_layers * (2.0 * batch * m * m + 3.0 * batch * m) + 2.0 * batch * m * num_features * cfg.out_dim


def compression_ratio(tower_widths: list[int], tower_feature_counts: list[int], in_dim: int) -> float:
    """towermod.py:209-223: (total features * in_dim) / sum(tower widths)."""
    if len(tower_widths) != len(tower_feature_counts):
        raise DomainError("tower_widths and tower_feature_counts must align")
    total_out, total_f = sum(tower_widths), sum(tower_feature_counts)
    if total_out <= 0 or total_f * in_dim <= 0:
        raise DomainError("widths and feature counts must be positive")
    return (total_f * in_dim) / total_out


def balanced_group_sizes(total: int, groups: int) -> list[int]:
    """towermod.py:226-228."""
    base, extra = divmod(total, groups)
    return [base + (1 if i < extra else 0) for i in range(groups)]


def interaction_pairs(num_features: int, num_towers: int, reduction_ratio: float) -> tuple[float, float]:
    """towermod.py:231-250 (paper-level pair accounting)."""
    if num_towers < 1:
        raise DomainError("num_towers must be >= 1")
    if not 0 < reduction_ratio <= 1:
        raise DomainError("reduction_ratio must be in (0, 1]")
    flat = num_features * (num_features - 1) / 2
    within = sum(s * (s - 1) / 2 for s in balanced_group_sizes(num_features, num_towers))
    r = reduction_ratio * num_features
    return flat, within + r * (r - 1) / 2


# --------------------------------------------------------------------------- #
# device tower module
# --------------------------------------------------------------------------- #
class TowerModule:
    # DCN backward form (all parity-tested):
    #   "side" (default): light dX epilogues (x0, g_{l+1} in; g_l, gu_l out),
    #     dx0 = sum_l g_{l+1} * u_l and the bias-gradient column sums on a side
    #     stream beside the compute-bound dW GEMMs;
    #   "accumulate": fp32 dx0 read-modify-written by every layer's epilogue;
    #   "pairs": no dx0, every g_l kept, pair-sum final epilogue, bias-gradient
    #     column sums fused into the epilogues (L <= 4).
    dcn_bwd_form = os.environ.get("DMT_DCN_BWD", "side")
    # side form: the element-wise tail (dx0 terms + crossnet bias column sums)
    # as one fused pass after the layer-1 dX GEMM (default), or per layer
    # beside each dW GEMM (DMT_DCN_SIDE=split; measured ~0.2 ms serialised
    # behind the persistent GEMMs at C2: those kernels cannot co-reside)
    _side_fused = os.environ.get("DMT_DCN_SIDE", "fused") == "fused"
    _tail_main = os.environ.get("DMT_DCN_TAIL", "side") == "main"
    _dw_concurrent = os.environ.get("DMT_DW_STREAM", "0") == "1"  # measured neutral at C2 (profiles/r2_step_ab.txt)

    """Device TM of one tower: forward / backward / SGD on libdmt GEMMs.

    Input X is (rows, F*N) in the compute dtype, rows = T*B on an SPTT rank
    (step e stacks the T destination blocks, exchange.py:417-437, so one GEMM
    serves all of them).  Output Y (rows, O) is exactly the step-f send buffer.
    """

    def __init__(self, cfg: TMConfig, num_features: int, in_dim: int, weights, dtype=torch.float32,
                 device=None):
        if cfg.kind == PASSTHROUGH:
            raise DomainError("TowerModule needs a dlrm or dcn config")
        self.cfg, self.F, self.N = cfg, num_features, in_dim
        self.dtype = dtype
        self.device = device or torch.device("cuda")
        self.width = tm_output_width(cfg, num_features, in_dim)
        dev = lambda a, dt=None: torch.as_tensor(np.asarray(a), device=self.device).to(dt or dtype).contiguous()
        f32 = torch.float32
        if cfg.kind == DLRM:
            self.w = {"w_flat": dev(weights.w_flat), "b_flat": dev(weights.b_flat, f32),
                      "w_feat": dev(weights.w_feat), "b_feat": dev(weights.b_feat, f32)}
        else:
            self.w = {"w_proj": dev(weights.w_proj), "b_proj": dev(weights.b_proj, f32)}
            for i, (cw, cb) in enumerate(weights.cross):
                self.w[f"w{i}"] = dev(cw)
                self.w[f"b{i}"] = dev(cb, f32)
        self.grads: dict[str, torch.Tensor] = {}
        self._saved = None

    # -- forward ---------------------------------------------------------------
    def forward(self, x: torch.Tensor, save: bool = False, out: Optional[torch.Tensor] = None,
                out_groups: Optional[tuple] = None) -> torch.Tensor:
        """``out_groups`` = (rows_per_group, [device addresses]): a DCN module's
        projection GEMM stores row block j straight at address j (row stride =
        the output width) -- step f fused into the TM (peer receive buffers);
        ``out`` then only supplies the dtype."""
        rows = x.shape[0]
        if x.dim() != 2 or x.shape[1] != self.F * self.N:
            raise ShapeError(f"TM input {tuple(x.shape)} != (rows, {self.F * self.N})")
        y = out if out is not None else torch.empty((rows, self.width), dtype=self.dtype, device=x.device)
        if rows == 0:
            return y
        if self.cfg.kind == DLRM:
            self._dlrm_fwd(x, y)
            if save:
                self._saved = (x,)
            return y
        xs, us = [x], []
        xl = x
        M = self.F * self.N
        if M == 0:
            y.copy_(self.w["b_proj"].to(y.dtype).expand_as(y))
            return y
        for i in range(self.cfg.cross_layers):
            u = torch.empty((rows, M), dtype=self.dtype, device=x.device) if save else None
            nxt = torch.empty((rows, M), dtype=self.dtype, device=x.device)
            K.gemm(xl, self.w[f"w{i}"], nxt, bias=self.w[f"b{i}"], epilogue=L.EPI_CROSS, x0=x, xl=xl, aux=u)
            if save:
                us.append(u)
                xs.append(nxt)
            xl = nxt
        if out_groups is not None:
            rpg, ptrs = out_groups
            K.gemm(xl, self.w["w_proj"], y, bias=self.w["b_proj"], epilogue=L.EPI_BIAS, rows_per_group=rpg,
                   ld_d=self.width, out_groups=ptrs)
        else:
            K.gemm(xl, self.w["w_proj"], y, bias=self.w["b_proj"], epilogue=L.EPI_BIAS)
        if save:
            self._saved = (xs, us)
        return y

    def _dlrm_fwd(self, x, y):
        c, p, D = self.cfg.per_feature_outputs, self.cfg.flat_outputs, self.cfg.out_dim
        rows, O = x.shape[0], self.width
        pD, cD = p * D, c * D
        if pD:
            if self.F * self.N == 0:
                y[:, :pD].copy_(self.w["b_flat"].to(y.dtype).expand(rows, pD))
            else:
                K.gemm(x, self.w["w_flat"], y, bias=self.w["b_flat"], epilogue=L.EPI_BIAS, ld_d=O)
        if cD and self.F:
            xf = x.view(rows * self.F, self.N)
            yv = y.view(-1)[pD:]
            K.gemm(xf, self.w["w_feat"], yv, bias=self.w["b_feat"], epilogue=L.EPI_BIAS,
                   rows_per_group=self.F, ld_group=O, ld_d=cD)

    # -- backward --------------------------------------------------------------
    def backward(self, gy: torch.Tensor, fused_lr: Optional[float] = None,
                 dx_out: Optional[torch.Tensor] = None, dx_scatter: Optional[tuple] = None) -> torch.Tensor:
        """Returns dX (rows, F*N) in the compute dtype; fp32 weight grads are
        stored in ``self.grads`` (this rank's contribution only).

        ``fused_lr``: when no cross-rank gradient reduction is needed (a tower
        of one rank), the DCN weight matrices are updated in place by the dW
        GEMM epilogue (W -= lr * dW, dmt_gemm SCALE_ACC + ACC) and only the
        bias grads are left in ``self.grads``.  ``dx_out``: write dX there (a
        persistent buffer the embedding backward reads directly)."""
        if self._saved is None:
            raise DomainError("backward() needs forward(save=True)")
        self._dx_out = dx_out
        # (width, [(address, row stride)]): the DCN's final dX GEMM stores each
        # column block straight there (step d^-1 fused; accumulate form only)
        self._dx_scatter = dx_scatter if (self.cfg.kind == DCN and self.dcn_bwd_form != "pairs") else None
        if self.cfg.kind == DLRM:
            return self._dlrm_bwd(gy)
        return self._dcn_bwd(gy, fused_lr)

    def _new_dx(self, like: torch.Tensor) -> torch.Tensor:
        out = getattr(self, "_dx_out", None)
        if out is None:
            return torch.empty_like(like)
        if out.shape != like.shape or out.dtype != like.dtype:
            raise ShapeError(f"dx_out {tuple(out.shape)} {out.dtype} does not match dX {tuple(like.shape)} {like.dtype}")
        return out

    def _dlrm_bwd(self, gy):
        (x,) = self._saved
        c, p, D = self.cfg.per_feature_outputs, self.cfg.flat_outputs, self.cfg.out_dim
        rows, O, F, N = x.shape[0], self.width, self.F, self.N
        pD, cD = p * D, c * D
        dx = self._new_dx(x)
        first = True
        f32 = torch.float32
        if pD:
            g1 = gy[:, :pD]
            if F * N:
                K.gemm(g1, self.w["w_flat"], dx, trans_b=True)
                first = False
                self.grads["w_flat"] = K.gemm(g1, x, torch.empty((pD, F * N), dtype=f32, device=x.device),
                                              trans_a=True, trans_b=True)
            else:
                self.grads["w_flat"] = torch.zeros_like(self.w["w_flat"], dtype=f32)
            self.grads["b_flat"] = K.column_sum(g1)
        else:
            self.grads["w_flat"] = torch.zeros_like(self.w["w_flat"], dtype=f32)
            self.grads["b_flat"] = torch.zeros_like(self.w["b_flat"], dtype=f32)
        if cD and F:
            g2 = gy[:, pD:]
            if pD:  # make the per-feature block contiguous: (rows*F, cD)
                g2c = torch.empty((rows, F * cD), dtype=gy.dtype, device=gy.device)
                K.assemble([K.Block(0, F * cD, [(gy, pD, gy.stride(0))])], g2c, rows)
                g2 = g2c
            g2v = g2.contiguous().view(rows * F, cD)
            xv = x.view(rows * F, N)
            dxv = dx.view(rows * F, N)
            K.gemm(g2v, self.w["w_feat"], dxv, epilogue=L.EPI_NONE if first else L.EPI_ACC,
                   beta=0.0 if first else 1.0, trans_b=True)
            first = False
            self.grads["w_feat"] = K.gemm(g2v, xv, torch.empty((cD, N), dtype=f32, device=x.device),
                                          trans_a=True, trans_b=True)
            self.grads["b_feat"] = K.column_sum(g2v)
        else:
            self.grads["w_feat"] = torch.zeros_like(self.w["w_feat"], dtype=f32)
            self.grads["b_feat"] = torch.zeros_like(self.w["b_feat"], dtype=f32)
        if first:
            dx.zero_()
        return dx

    def _dcn_bwd(self, gy, fused_lr: Optional[float] = None):
        """Crossnet backward with the element-wise work fused into GEMM
        epilogues (dmt_gemm DCN_BWD / DCN_FINAL):
            g_L = gy Wp;  gu_l = g_{l+1} * x0;  dx0 += g_{l+1} * u_l
            dW_l = gu_l^T x_l;  g_l = gu_l W_l + g_{l+1};  dX = g_0 + dx0
        (derivative of towermod.py:132-158; x_0 = X, u_l = x_l W_l^T + b_l).
        Each dX-side GEMM runs before the weight it reads is (optionally)
        updated in place."""
        xs, us = self._saved
        x0 = xs[0]
        rows, M = x0.shape
        L_ = self.cfg.cross_layers
        f32 = torch.float32
        dev = x0.device
        self.grads = {}

        def weight_grad(name, a, b):
            if fused_lr is not None:  # W -= lr * a^T b, in the GEMM epilogue
                K.gemm(a, b, self.w[name], trans_a=True, trans_b=True, epilogue=L.EPI_ACC, beta=1.0,
                       alpha=-fused_lr)
            else:
                self.grads[name] = K.gemm(a, b, torch.empty(self.w[name].shape, dtype=f32, device=dev),
                                          trans_a=True, trans_b=True)

        if L_ <= L.GEMM_MAX_PAIRS and self.dcn_bwd_form == "pairs":
            return self._dcn_bwd_pairs(gy, weight_grad)
        if self.dcn_bwd_form == "side":
            return self._dcn_bwd_side(gy, weight_grad)
        g = torch.empty((rows, M), dtype=self.dtype, device=dev)
        gu = [torch.empty((rows, M), dtype=self.dtype, device=dev) for _ in range(2)]
        dx0 = torch.empty((rows, M), dtype=f32, device=dev)
        # separate bias-gradient column sums: folding them into these epilogues
        # measured slower (+45 us per layer vs 34 us for the standalone pass)
        part = None

        def bias_grad(name, t):
            self.grads[name] = K.column_sum_parts(part) if part is not None else K.column_sum(t)

        K.gemm(gy, self.w["w_proj"], g, trans_b=True, epilogue=L.EPI_DCN_BWD, x0=x0, xl=us[L_ - 1],
               aux=gu[(L_ - 1) % 2], aux2=dx0, aux2_accum=False, colsum_part=part)
        weight_grad("w_proj", gy, xs[-1])
        self.grads["b_proj"] = K.column_sum(gy)
        dx = self._new_dx(g)
        for layer in range(L_ - 1, -1, -1):
            cur = gu[layer % 2]
            bias_grad(f"b{layer}", cur)  # before the next GEMM overwrites the partials
            if layer > 0:
                K.gemm(cur, self.w[f"w{layer}"], g, trans_b=True, epilogue=L.EPI_DCN_BWD, c=g, beta=1.0, x0=x0,
                       xl=us[layer - 1], aux=gu[(layer - 1) % 2], aux2=dx0, aux2_accum=True, colsum_part=part)
            else:
                sc = self._dx_scatter
                K.gemm(cur, self.w["w0"], dx, trans_b=True, epilogue=L.EPI_DCN_FINAL, c=g, beta=1.0, aux2=dx0,
                       col_groups=sc[1] if sc else (), col_group_width=sc[0] if sc else 0)
            weight_grad(f"w{layer}", cur, xs[layer])
        return dx

    def _dw_stream(self) -> torch.cuda.Stream:
        st = getattr(self, "_dws", None)
        if st is None or st.device != torch.cuda.current_stream().device:
            st = self._dws = torch.cuda.Stream(device=torch.cuda.current_stream().device, priority=-1)
        return st

    def _aux_stream(self) -> torch.cuda.Stream:
        st = getattr(self, "_aux", None)
        if st is None or st.device != torch.cuda.current_stream().device:
            st = self._aux = torch.cuda.Stream(device=torch.cuda.current_stream().device)
        return st

    def _dcn_bwd_side(self, gy, weight_grad):
        """Crossnet backward with light dX epilogues (8 bytes / element: x0 and
        g_{l+1} in, g_l and gu_l out -- the "pairs" form's per-layer GEMMs),
        while the element-wise rest runs on a side stream beside the next dW
        GEMM (compute-bound, leaving HBM idle):
            dx0 = sum_{l=L..1} g_l * u_{l-1}   (dmt_dcn_dx0_term, fp32)
            db_l = colsum(gu_l),  db_proj = colsum(gy)
        and the final epilogue is DCN_FINAL: dX = gu_0 W_0 + g_1 + dx0 (with the
        step-d^-1 column scatter when given).  Same dx0 summation order as the
        "accumulate" form; g_l enters dx0 as stored (compute dtype)."""
        xs, us = self._saved
        x0 = xs[0]
        rows, M = x0.shape
        L_ = self.cfg.cross_layers
        dev, dt = x0.device, self.dtype
        main, side = torch.cuda.current_stream(), self._aux_stream()
        # dW GEMMs on their own stream: dW_l (3328^2 outputs: 169 pair tiles =
        # 2.28 persistent waves) and the next dX GEMM are independent, so the
        # next GEMM's CTAs fill the SMs the dW's partial last wave leaves idle
        conc = self._dw_concurrent
        dws = self._dw_stream() if conc else None

        def wgrad(name, a, b):
            if not conc:
                weight_grad(name, a, b)
                return
            dws.wait_stream(main)
            with torch.cuda.stream(dws):
                weight_grad(name, a, b)

        G = [None] + [torch.empty((rows, M), dtype=dt, device=dev) for _ in range(L_)]
        gu = [torch.empty((rows, M), dtype=dt, device=dev) for _ in range(L_)]
        dx0 = torch.empty((rows, M), dtype=torch.float32, device=dev)
        bias = {f"b{l}": torch.empty(M, dtype=torch.float32, device=dev) for l in range(L_)}
        bias["b_proj"] = torch.empty(gy.shape[1], dtype=torch.float32, device=dev)

        fused = self._side_fused and dt in (torch.bfloat16, torch.float16) and M % 8 == 0 and 1 <= L_ <= 4

        def side_work(layer):
            # g_{layer+1} and gu_layer exist (written by the dX GEMM just issued)
            if fused:
                # one pass once every g_l / gu_l exists (after the layer-1 dX
                # GEMM): all dx0 terms + all crossnet bias column sums
                if layer != 0:
                    return
                if self._tail_main:
                    # dx0 on the main chain (the final dX GEMM needs it), the
                    # bias column sums on the side stream, joined at the end
                    K.dcn_side_fused([G[l + 1] for l in range(L_)], [us[l] for l in range(L_)], None, dx0, None)
                    side.wait_stream(main)
                    with torch.cuda.stream(side):
                        for l in range(L_):
                            K.column_sum(gu[l], out=bias[f"b{l}"])
                        K.column_sum(gy, out=bias["b_proj"])
                    return
                side.wait_stream(main)
                with torch.cuda.stream(side):
                    K.dcn_side_fused([G[l + 1] for l in range(L_)], [us[l] for l in range(L_)], gu, dx0,
                                     [bias[f"b{l}"] for l in range(L_)])
                    K.column_sum(gy, out=bias["b_proj"])
                return
            side.wait_stream(main)
            with torch.cuda.stream(side):
                K.dcn_dx0_term(G[layer + 1], us[layer], dx0, accumulate=layer != L_ - 1)
                K.column_sum(gu[layer], out=bias[f"b{layer}"])
                if layer == L_ - 1:
                    K.column_sum(gy, out=bias["b_proj"])

        K.gemm(gy, self.w["w_proj"], G[L_], trans_b=True, epilogue=L.EPI_DCN_BWD, x0=x0, aux=gu[L_ - 1])
        side_work(L_ - 1)
        wgrad("w_proj", gy, xs[-1])
        dx = self._new_dx(x0)
        for layer in range(L_ - 1, -1, -1):
            cur = gu[layer]
            if layer > 0:
                K.gemm(cur, self.w[f"w{layer}"], G[layer], trans_b=True, epilogue=L.EPI_DCN_BWD, c=G[layer + 1],
                       beta=1.0, x0=x0, aux=gu[layer - 1])
                side_work(layer - 1)
                wgrad(f"w{layer}", cur, xs[layer])
            else:
                # the side stream's last dx0 term ran beside dW_1; dW_0 stays
                # after this GEMM (a fused SGD updates W_0 in place)
                if not (fused and self._tail_main):
                    main.wait_stream(side)
                sc = self._dx_scatter
                K.gemm(cur, self.w["w0"], dx, trans_b=True, epilogue=L.EPI_DCN_FINAL, c=G[1], beta=1.0, aux2=dx0,
                       col_groups=sc[1] if sc else (), col_group_width=sc[0] if sc else 0)
                wgrad("w0", cur, xs[0])
        if conc:
            main.wait_stream(dws)  # weight updates / grads complete before the caller goes on
        if fused and self._tail_main:
            main.wait_stream(side)  # bias column sums (side stream) before the optimizer reads them
        self.grads.update(bias)
        return dx

    def _colsum_part(self, rows, M, dev):
        """Buffer of the fused bias-gradient partials (DCN_BWD epilogue), or None
        when the width does not allow the fused form (M % 32 != 0)."""
        if M % 32:
            return None
        key = (rows, M)
        if getattr(self, "_part_key", None) != key:
            self._part = torch.empty((K.colsum_rows(rows), M), dtype=torch.float32, device=dev)
            self._part_key = key
        return self._part

    def _dcn_bwd_pairs(self, gy, weight_grad):
        """Crossnet backward without an fp32 dx0 accumulator (L <= 4 layers):
            g_L = gy Wp;  gu_l = g_{l+1} * x0;  g_l = gu_l W_l + g_{l+1}
            dX = gu_0 W_0 + g_1 + sum_l g_{l+1} * u_l     (one DCN_FINAL epilogue)
        Every g_l is kept (bf16), so the per-layer epilogues move 8 bytes per
        element (x0, g_{l+1} in; g_l, gu out) instead of 18, and the bias
        gradients colsum(gu_l) are folded in the same epilogues (per-tile
        partials + one deterministic reduce) when the width is a multiple of 32."""
        xs, us = self._saved
        x0 = xs[0]
        rows, M = x0.shape
        L_ = self.cfg.cross_layers
        dev, dt = x0.device, self.dtype
        G = [None] + [torch.empty((rows, M), dtype=dt, device=dev) for _ in range(L_)]
        gu = [torch.empty((rows, M), dtype=dt, device=dev) for _ in range(2)]
        part = self._colsum_part(rows, M, dev)

        def bias_grad(name, t):
            self.grads[name] = K.column_sum_parts(part) if part is not None else K.column_sum(t)

        K.gemm(gy, self.w["w_proj"], G[L_], trans_b=True, epilogue=L.EPI_DCN_BWD, x0=x0, aux=gu[(L_ - 1) % 2],
               colsum_part=part)
        weight_grad("w_proj", gy, xs[-1])
        self.grads["b_proj"] = K.column_sum(gy)
        dx = self._new_dx(x0)
        for layer in range(L_ - 1, -1, -1):
            cur = gu[layer % 2]
            bias_grad(f"b{layer}", cur)  # before the next GEMM overwrites the partials
            if layer > 0:
                K.gemm(cur, self.w[f"w{layer}"], G[layer], trans_b=True, epilogue=L.EPI_DCN_BWD, c=G[layer + 1],
                       beta=1.0, x0=x0, aux=gu[(layer - 1) % 2], colsum_part=part)
            else:
                K.gemm(cur, self.w["w0"], dx, trans_b=True, epilogue=L.EPI_DCN_FINAL, c=G[1], beta=1.0,
                       pairs=[(G[j + 1], us[j]) for j in range(L_)])
            weight_grad(f"w{layer}", cur, xs[layer])
        return dx

    def sgd_step(self, lr: float) -> None:
        for k, g in self.grads.items():
            K.sgd_dense(self.w[k], g.contiguous(), lr)

    def host_weights(self):
        """Current weights back as reference-typed numpy dataclasses."""
        h = {k: v.double().cpu().numpy() for k, v in self.w.items()}
        if self.cfg.kind == DLRM:
            return DLRMWeights(h["w_flat"], h["b_flat"], h["w_feat"], h["b_feat"])
        cross = tuple((h[f"w{i}"], h[f"b{i}"]) for i in range(self.cfg.cross_layers))
        return DCNWeights(cross, h["w_proj"], h["b_proj"])


def _compute_dtype(embs: np.ndarray):
    return torch.float32  # f64 inputs run as fp32 (3xTF32); bf16 via TowerModule(dtype=...)


def tm_forward(embs: np.ndarray, cfg: TMConfig, weights) -> np.ndarray:
    """towermod.py:161-166 on the GPU; (B, F, N) -> (B, O) float64."""
    embs = np.asarray(embs)
    if embs.ndim != 3:
        raise ShapeError(f"embs must be 3-D, got {embs.shape}")
    B, F, N = embs.shape
    if cfg.kind == PASSTHROUGH:
        return embs.reshape(B, -1).astype(np.float64)
    _check_weight_shapes(cfg, weights, F, N)
    tm = TowerModule(cfg, F, N, weights, dtype=_compute_dtype(embs))
    x = torch.from_numpy(np.ascontiguousarray(embs.reshape(B, F * N))).to(tm.device, torch.float32)
    return tm.forward(x).double().cpu().numpy()


def _check_weight_shapes(cfg, w, F, N):
    if cfg.kind == DLRM:
        if w.w_flat.shape[1] != F * N:
            raise ShapeError(f"w_flat expects input width {w.w_flat.shape[1]}, got {F * N}")
        if w.w_feat.shape[1] != N:
            raise ShapeError(f"w_feat expects input width {w.w_feat.shape[1]}, got {N}")
    else:
        if w.w_proj.shape[1] != F * N:
            raise ShapeError(f"projection expects input width {w.w_proj.shape[1]}, got {F * N}")


def tm_dlrm_forward(embs, cfg, weights):
    """towermod.py:110-129 (GPU)."""
    return tm_forward(embs, cfg, weights)


def tm_dcn_forward(embs, cfg, weights):
    """towermod.py:142-158 (GPU)."""
    return tm_forward(embs, cfg, weights)


def crossnet_layer(x0: np.ndarray, xl: np.ndarray, w: np.ndarray, b: np.ndarray) -> np.ndarray:
    """towermod.py:132-139 on the GPU: x0 * (xl W^T + b) + xl (fused epilogue)."""
    x0, xl = np.asarray(x0), np.asarray(xl)
    if x0.shape != xl.shape:
        raise ShapeError(f"x0 {x0.shape} and xl {xl.shape} must match")
    m = x0.shape[-1]
    if w.shape != (m, m) or b.shape != (m,):
        raise ShapeError(f"cross layer weights {w.shape}/{b.shape} do not match width {m}")
    dev = torch.device("cuda")
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).to(dev, torch.float32)
    x0t, xlt = t(x0.reshape(-1, m)), t(xl.reshape(-1, m))
    out = torch.empty_like(xlt)
    K.gemm(xlt, t(w), out, bias=t(b), epilogue=L.EPI_CROSS, x0=x0t, xl=xlt)
    return out.double().cpu().numpy().reshape(x0.shape)
