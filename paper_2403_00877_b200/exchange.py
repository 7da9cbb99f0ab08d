"""Reference-compatible exchange API on the GPU (drop-in for towersim/exchange.py).

``tower_exchange`` / ``baseline_exchange`` / ``realign`` keep the reference's
signatures and result types (exchange.py:46-109, 200-486): they take the
host-side SparseBatch / ShardedEmbedding of all G ranks, run every simulated
rank's share on one B200 through the same kernels the distributed path uses
(LoopbackFabric), and return float64 numpy outputs plus a CommTrace whose byte
totals follow the reference's accounting.  Table dtype decides the compute
dtype (float64 tables -> f64 kernels, bit-exact with the reference; float32 ->
f32, bit-exact for table/column-wise pooling).
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np
import torch

from . import kernels as K
from .embedding import ShardedEmbedding, SparseBatch
from .errors import DomainError, LayoutError, PlanError
from .fabric import LoopbackFabric
from .pipeline import KJT, SpttEngine
from .plan import ExchangePlan
from .simnet import CommTrace
from .topology import ClusterTopology, TowerLayout
from .towermod import PASSTHROUGH, TMConfig, TowerModule, init_tm_weights, tm_flops, tm_output_width


@dataclass(frozen=True)
class TowerPlan:
    """exchange.py:46-54."""

    layout: TowerLayout
    feature_towers: dict

    def features_of(self, tower: int) -> list[int]:
        return sorted(f for f, t in self.feature_towers.items() if t == tower)


@dataclass(frozen=True)
class ExchangeOptions:
    """exchange.py:57-81.  swap_bc / omit_permute are result-invariant orderings
    of the same data movement; on the GPU the permute is always fused into the
    lookup epilogue (zero extra bytes), so both are accepted and change nothing.
    rowwise_reducescatter switches the step-d combine of row-wise features to
    the reference's reduce-scatter (exchange.py:380-395): the byte accounting
    of simnet.reduce_scatter and its summation order -- each owner's shard
    partials first, then the owners in group order (simnet.py:173-192) -- which
    can differ in the last bit from the row-range order of the all-to-all form
    on real-valued tables."""

    swap_bc: bool = False
    omit_permute: bool = False
    rowwise_reducescatter: bool = False
    tower_modules: object = None

    def tm_for(self, tower: int) -> TMConfig:
        if self.tower_modules is None:
            return TMConfig(kind=PASSTHROUGH)
        if isinstance(self.tower_modules, TMConfig):
            return self.tower_modules
        return self.tower_modules.get(tower, TMConfig(kind=PASSTHROUGH))


@dataclass(frozen=True)
class OutputLayout:
    """exchange.py:84-101."""

    blocks: tuple

    @property
    def total_width(self) -> int:
        return sum(w for _, _, w in self.blocks)

    def feature_widths(self) -> dict[int, int]:
        if any(kind != "feature" for kind, _, _ in self.blocks):
            raise LayoutError("layout contains compressed tower blocks")
        return {ident: width for _, ident, width in self.blocks}


@dataclass
class ExchangeResult:
    """exchange.py:104-109 (+ the device tensors the outputs came from)."""

    outputs: dict
    layout: OutputLayout
    trace: CommTrace
    flops: dict = field(default_factory=dict)
    device_outputs: Optional[dict] = None


_NP_TORCH = {np.dtype(np.float64): torch.float64, np.dtype(np.float32): torch.float32}


def _compute_dtype(placement: ShardedEmbedding, features, dtype):
    if dtype is not None:
        return dtype
    dts = {np.asarray(placement.tables[f].values).dtype for f in features}
    if dts == {np.dtype(np.float32)}:
        return torch.float32
    return torch.float64


def batch_to_kjts(batch: SparseBatch, device) -> dict:
    """SparseBatch (embedding.py:215-226) -> one device KJT per rank."""
    feats = batch.features
    B = batch.local_batch
    out = {}
    for r in range(batch.num_ranks):
        lens = np.zeros(len(feats) * B, dtype=np.int32)
        vals, nnz = [], []
        for fi, f in enumerate(feats):
            bags = batch.bags[r][f]
            ln = np.fromiter((len(b) for b in bags), dtype=np.int32, count=B)
            lens[fi * B:(fi + 1) * B] = ln
            nnz.append(int(ln.sum()))
            vals.append(np.fromiter((i for b in bags for i in b), dtype=np.int64, count=int(ln.sum())))
        v = np.concatenate(vals) if vals else np.zeros(0, np.int64)
        if v.size and v.max() >= 2 ** 31:
            raise DomainError("indices must fit int32")
        out[r] = KJT(lengths=torch.from_numpy(lens).to(device),
                     values=torch.from_numpy(v.astype(np.int32)).to(device), nnz_per_feature=nnz, B=B)
    return out


def _validate(batch, placement, topo):
    batch.validate(placement.tables)
    for f in batch.features:
        placement.shards_of(f)
    if batch.num_ranks != topo.world_size:
        raise DomainError(f"batch has {batch.num_ranks} ranks, topology {topo.world_size}")


def baseline_exchange(batch: SparseBatch, placement: ShardedEmbedding, topo: ClusterTopology,
                      trace: Optional[CommTrace] = None, *, dtype: Optional[torch.dtype] = None,
                      device=None) -> ExchangeResult:
    """exchange.py:200-241: global index all-to-all, lookup, global embedding
    all-to-all; columns in feature-id order."""
    _validate(batch, placement, topo)
    device = device or torch.device("cuda")
    trace = trace if trace is not None else CommTrace(topo)
    feats = batch.features
    dims = {f: placement.tables[f].dim for f in feats}
    plan = ExchangePlan(topo, TowerLayout(1, topo.num_hosts), placement.shards, feats, dims, batch.pooling,
                        batch.local_batch)
    dt = _compute_dtype(placement, feats, dtype)
    eng = SpttEngine(plan, placement, LoopbackFabric(topo.world_size, device), dt, device, mode="flat",
                     trace=trace)
    outs = eng.forward(batch_to_kjts(batch, device))
    layout = OutputLayout(tuple(("feature", f, dims[f]) for f in feats))
    flops = {"b": _lookup_flops(batch, placement, plan)}
    return ExchangeResult({r: o.double().cpu().numpy() for r, o in outs.items()}, layout, trace, flops, outs)


def _lookup_flops(batch, placement, plan) -> float:
    """exchange.py:143-146: per owner sum over its shards of (indices kept) * width."""
    best = 0.0
    for o in range(plan.G):
        tot = 0.0
        for sid in plan.by_owner[o]:
            sh = placement.shards[sid]
            for r in range(batch.num_ranks):
                bags = batch.bags[r][sh.table_id]
                if sh.scheme == "row_wise":
                    r0, r1 = sh.row_range
                    n = sum(1 for b in bags for i in b if r0 <= i < r1)
                else:
                    n = sum(len(b) for b in bags)
                tot += n * sh.width
        best = max(best, tot)
    return float(best)


def tower_exchange(batch: SparseBatch, placement: ShardedEmbedding, plan: TowerPlan, topo: ClusterTopology,
                   opts: ExchangeOptions = ExchangeOptions(), trace: Optional[CommTrace] = None,
                   step_f_schedule: Optional[Sequence[int]] = None, *, dtype: Optional[torch.dtype] = None,
                   device=None) -> ExchangeResult:
    """exchange.py:275-462: SPTT a-f.  Output columns are tower-grouped; TM
    towers are opaque ("tower", t, O_t) blocks."""
    _validate(batch, placement, topo)
    layout = plan.layout
    layout.validate_for(topo)
    W = layout.group_width(topo)
    if step_f_schedule is not None and sorted(step_f_schedule) != list(range(W)):
        raise DomainError("step_f_schedule must be a permutation of the classes")
    device = device or torch.device("cuda")
    trace = trace if trace is not None else CommTrace(topo)
    feats = batch.features
    dims = {f: placement.tables[f].dim for f in feats}
    for f in feats:
        if f not in plan.feature_towers:
            raise PlanError(f"feature {f} has no tower assignment")
    by_tower = {t: [f for f in plan.features_of(t) if f in batch.pooling] for t in range(layout.num_towers)}
    widths, tms, kinds, e_flops = {}, {}, {}, 0.0
    dt = _compute_dtype(placement, feats, dtype)
    tm_dt = torch.float32 if dt == torch.float64 else dt
    for t in range(layout.num_towers):
        cfg = opts.tm_for(t)
        kinds[t] = cfg.kind
        fs = by_tower[t]
        if cfg.kind != PASSTHROUGH:
            ds = {dims[f] for f in fs}
            if len(ds) > 1:
                raise PlanError(f"tower {t} mixes embedding dims {sorted(ds)}; tower modules need one dim per tower")
            n = ds.pop() if ds else 1
            widths[t] = tm_output_width(cfg, len(fs), n)
            e_flops = max(e_flops, tm_flops(cfg, len(fs), n, batch.local_batch) * layout.num_towers)
            if fs:
                tms[t] = TowerModule(cfg, len(fs), n, init_tm_weights(cfg, len(fs), n, salt=t), dtype=tm_dt,
                                     device=device)
    xplan = ExchangePlan(topo, layout, placement.shards, feats, dims, batch.pooling, batch.local_batch,
                         feature_towers=plan.feature_towers, tower_widths=widths)
    if dt != tm_dt and tms:
        # f64 tables with a TM: pool in f64, run the tower module in fp32 (3xTF32)
        eng = _MixedEngine(xplan, placement, LoopbackFabric(topo.world_size, device), dt, tm_dt, device, tms,
                           trace, opts.rowwise_reducescatter)
    else:
        eng = SpttEngine(xplan, placement, LoopbackFabric(topo.world_size, device), dt, device,
                         tower_modules=tms, mode="sptt", trace=trace, rowwise_reducescatter=opts.rowwise_reducescatter)
    outs = eng.forward(batch_to_kjts(batch, device))
    # empty TM towers (no features) still emit their bias-only / zero block
    for t, cfg in ((t, opts.tm_for(t)) for t in range(layout.num_towers)):
        if cfg.kind != PASSTHROUGH and not by_tower[t] and widths[t]:
            _fill_empty_tower(outs, xplan, t, cfg)
    lay = OutputLayout(tuple(xplan.tower_layout_blocks(kinds)))
    flops = {"b": _lookup_flops(batch, placement, xplan), "e": e_flops}
    return ExchangeResult({r: o.double().cpu().numpy() for r, o in outs.items()}, lay, trace, flops, outs)


def _fill_empty_tower(outs, xplan, t, cfg):
    """A TM tower with no features: dlrm emits its flat-projection bias, dcn an
    empty block (towermod.py:126-129 with F = 0)."""
    w = init_tm_weights(cfg, 0, 1, salt=t)
    col = sum(xplan.O[j] for j in range(t))
    if cfg.kind == "dlrm" and w.b_flat.size:
        b = torch.as_tensor(w.b_flat)
        for o in outs.values():
            o[:, col:col + b.numel()] = b.to(o.dtype).to(o.device)


class _MixedEngine(SpttEngine):
    """f64 pooling/exchange with an fp32 tower module: X is converted to fp32
    for the GEMMs and Y back to f64 for step f."""

    def __init__(self, plan, placement, fabric, dt, tm_dt, device, tms, trace, rs):
        super().__init__(plan, placement, fabric, dt, device, tower_modules={}, mode="sptt", trace=trace,
                         rowwise_reducescatter=rs)
        self.tm32 = tms
        for r in self.local:
            t = plan.tower_of(r)
            if t in tms:
                self.buf[r]["Y"] = torch.empty((plan.T * plan.B, plan.O[t]), dtype=dt, device=device)
                if plan.T == 1:  # step f is the identity: the output gathers from Y
                    self.buf[r]["recv_f"] = self.buf[r]["Y"].view(-1)
        self.asm_out = {}
        for r in self.local:
            b = self.buf[r]
            blocks = [K.Block(col, w, [(b["recv_f"], off, w)]) for col, w, off in plan.out_blocks_tower()]
            self.asm_out[r] = K.AssembleTable(blocks, b["out"], plan.B, device)

    def forward(self, kjts, save=False, check_indices=False):
        p = self.plan
        orig = {}
        for r in self.local:
            t = p.tower_of(r)
            if t in self.tm32:
                orig[r] = t
        # run a..e with pass-through (Y buffers are the f64 ones allocated above)
        self.tm = {}
        # hook: convert between dtypes around the TM
        real_asm = self.asm_e

        class _Hook:
            def __init__(s, r, inner):
                s.r, s.inner = r, inner

            def run(s):
                s.inner.run()
                r = s.r
                if r in orig:
                    x32 = K.convert(self.buf[r]["X"], torch.float32)
                    y32 = self.tm32[orig[r]].forward(x32)
                    self.buf[r]["Y"].copy_(K.convert(y32, self.dtype))

        self.asm_e = {r: _Hook(r, real_asm[r]) for r in self.local}
        try:
            return super().forward(kjts, save=False, check_indices=check_indices)
        finally:
            self.asm_e = real_asm


def realign(result: ExchangeResult, target_feature_order: Sequence[int]) -> ExchangeResult:
    """exchange.py:465-486: reverse permutation back to a feature order, done
    on the device with one gather launch per rank (dmt_assemble)."""
    widths = result.layout.feature_widths()
    if sorted(target_feature_order) != sorted(widths):
        raise LayoutError(f"target features {sorted(target_feature_order)} != layout features {sorted(widths)}")
    starts, col = {}, 0
    for _, ident, w in result.layout.blocks:
        starts[ident] = col
        col += w
    outputs, dev_out = {}, {}
    for rank, mat in result.outputs.items():
        src = (result.device_outputs or {}).get(rank)
        if src is None:
            src = torch.from_numpy(np.ascontiguousarray(mat)).cuda()
        dst = torch.empty((src.shape[0], col), dtype=src.dtype, device=src.device)
        blocks, c = [], 0
        for f in target_feature_order:
            blocks.append(K.Block(c, widths[f], [(src, starts[f], src.stride(0))]))
            c += widths[f]
        K.assemble(blocks, dst, src.shape[0])
        dev_out[rank] = dst
        outputs[rank] = dst.double().cpu().numpy()
    lay = OutputLayout(tuple(("feature", f, widths[f]) for f in target_feature_order))
    return ExchangeResult(outputs, lay, result.trace, dict(result.flops), dev_out)
