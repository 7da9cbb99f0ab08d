"""SPTT training module: the distributed forward/backward + optimizer step of
the DMT embedding path (e).

One process per GPU (NcclFabric) or every rank on one GPU (LoopbackFabric).
A step is: step a-f forward (towersim/exchange.py:275-462 semantics), tower
modules on each tower's data-parallel ranks, the reverse exchange, TM weight
gradients all-reduced inside the tower and a fused
sort/segment-reduce/SGD-or-row-wise-Adagrad update of every embedding shard on
its owner.
"""

from __future__ import annotations

import os

from typing import Optional

import numpy as np
import torch

from . import _lib as L
from . import kernels as K
from .errors import DomainError
from .embedding import EmbeddingTable, ShardedEmbedding, TablePlan, shard_tables
from .fabric import Fabric, LoopbackFabric, peer_allreduce_sgd
from .pipeline import KJT, SpttEngine
from .plan import ExchangePlan
from .topology import ClusterTopology, TowerLayout
from .towermod import PASSTHROUGH, TMConfig, TowerModule, init_tm_weights, tm_output_width


class SPTT:
    def __init__(self, topo: ClusterTopology, layout: TowerLayout, placement: ShardedEmbedding,
                 feature_towers: dict, pooling: dict, local_batch: int, fabric: Fabric,
                 tm: Optional[object] = None, dtype: torch.dtype = torch.float32, device=None,
                 mode: str = "sptt", lr: float = 0.01, optimizer: str = "sgd", eps: float = 1e-8,
                 trace=None, top: Optional[TMConfig] = None, dense_lr: Optional[float] = None,
                 check_indices: bool = False):
        """``lr`` drives the embedding (sparse) update; ``dense_lr`` (default:
        ``lr``) the tower modules, the flat baseline's global TM and the top
        head -- recommendation models train the two at very different rates."""
        self.topo, self.layout, self.placement = topo, layout, placement
        self.device = device or torch.device("cuda")
        feats = sorted(pooling)
        dims = {f: placement.tables[f].dim for f in feats}
        T = layout.num_towers
        by_tower = {t: [f for f in feats if feature_towers[f] == t] for t in range(T)}
        widths, tms = {}, {}
        self.tm_cfg = {}
        for t in range(T):
            cfg = tm.get(t) if isinstance(tm, dict) else tm
            cfg = cfg or TMConfig(kind=PASSTHROUGH)
            self.tm_cfg[t] = cfg
            if cfg.kind != PASSTHROUGH and mode == "sptt":
                n = dims[by_tower[t][0]] if by_tower[t] else 1
                widths[t] = tm_output_width(cfg, len(by_tower[t]), n)
                local_towers = {r // layout.group_width(topo) for r in fabric.local_ranks}
                if by_tower[t] and t in local_towers:
                    tms[t] = TowerModule(cfg, len(by_tower[t]), n, init_tm_weights(cfg, len(by_tower[t]), n, salt=t),
                                         dtype=dtype, device=self.device)
        self.plan = ExchangePlan(topo, layout, placement.shards, feats, dims, pooling, local_batch,
                                 feature_towers=feature_towers if mode == "sptt" else None, tower_widths=widths)
        self.engine = SpttEngine(self.plan, placement, fabric, dtype, self.device, tower_modules=tms, mode=mode,
                                 trace=trace)
        self.tms = tms
        self.fabric = fabric
        # flat baseline with the same dense work: one global TM over all
        # features after the flat all-to-all (what the DMT paper compares to)
        self.global_tm = None
        if mode == "flat" and tm is not None and not isinstance(tm, dict) and tm.kind != PASSTHROUGH:
            ds = {dims[f] for f in feats}
            n = ds.pop()
            self.global_tm = TowerModule(tm, len(feats), n, init_tm_weights(tm, len(feats), n, salt=0),
                                         dtype=dtype, device=self.device)
        # the flat global TM's world all-reduce + SGD over NVLink peer memory
        # when the exchange runs over peers too (same transport as SPTT's
        # tower reduction; rank-order fp32 sum, bit-identical replicas)
        self._peer_dense = None
        if (self.global_tm is not None and getattr(fabric, "p2p", False) and len(fabric.local_ranks) == 1
                and 1 < topo.world_size <= L.MAX_PEER_SRCS):
            bufs = {k: torch.empty(v.shape, dtype=torch.float32, device=self.device)
                    for k, v in self.global_tm.w.items() if v.numel()}
            shared = {"gtm_" + k: v for k, v in bufs.items()}
            shared.update({"gtw_" + k: self.global_tm.w[k] for k in bufs})
            self._peer_dense = (bufs, fabric.share(shared))
        # dense head above the exchange (data parallel, replicated on every
        # rank): the full DCN + SPTT model's top crossnet + logit projection,
        # a TowerModule over one "feature" of the whole SPTT output width
        self.top = None
        if top is not None:
            w_in = self.out_width
            if top.kind == PASSTHROUGH or tm_output_width(top, 1, w_in) != 1:
                raise DomainError("the top model must project to one logit (dcn out_dim=1 / dlrm c=1, p=0, "
                                  "out_dim=1)")
            self.top = TowerModule(top, 1, w_in, init_tm_weights(top, 1, w_in, salt=1_000_003), dtype=dtype,
                                   device=self.device)
            self._labels_loss = {}
        self.lr, self.eps = lr, eps
        self.dense_lr = lr if dense_lr is None else dense_lr
        # debug: validate every index against its table (TableLookupError, the
        # reference's embedding.py:74-77 check); costs a host sync per step
        self.check_indices = check_indices
        self.opt = L.OPT_ROWWISE_ADAGRAD if optimizer == "adagrad" else L.OPT_SGD
        if self.opt == L.OPT_ROWWISE_ADAGRAD:
            self.engine.enable_adagrad()

    def set_capacity(self, capacity) -> None:
        """Ragged batches without a host sync (and under CUDA graphs): see
        SpttEngine.set_capacity; ``capacity[f]`` >= feature f's nnz per rank."""
        self.engine.set_capacity(capacity)

    @property
    def out_width(self) -> int:
        if self.global_tm is not None:
            return self.global_tm.width
        return self.plan.out_width() if self.plan.feature_towers is not None else self.plan.flat_width()

    def forward(self, kjts: dict, save: bool = True) -> dict:
        outs = self.engine.forward(kjts, save=save, check_indices=self.check_indices)
        if self.global_tm is None:
            return outs
        self._gsaved = {}
        ys = {}
        for r, o in outs.items():
            with self.engine._t("tm_fwd"):
                ys[r] = self.global_tm.forward(o, save=save)
            self._gsaved[r] = self.global_tm._saved
        return ys

    def backward(self, grads: dict, dense_hook=None) -> None:
        if self.global_tm is None:
            self.engine.backward(grads, self.lr, self.opt, self.eps, tm_lr=self.dense_lr, dense_hook=dense_hook)
            return
        dx, acc = {}, {}
        for r, g in grads.items():
            self.global_tm._saved = self._gsaved[r]
            # peer fabric: the global TM's dX GEMM stores step c^-1 straight
            # into the owners' gradient buffers (same fusion as SPTT's d^-1)
            scatter = self.engine.flat_dx_scatter(r)
            with self.engine._t("tm_bwd"):
                dx[r] = self.global_tm.backward(g, dx_scatter=scatter)
            self.engine.c_bwd_fused = scatter is not None and self.global_tm._dx_scatter is not None
            for k, v in self.global_tm.grads.items():
                acc[k] = v.clone() if k not in acc else acc[k].add_(v)

        if self._peer_dense is not None:
            bufs = self._peer_dense[0]
            for k, v in acc.items():
                if k in bufs:
                    bufs[k].view(v.shape).copy_(v)

        def dense_step():  # world all-reduce of the global TM grads + SGD
            world = list(range(self.plan.G))
            if self._peer_dense is not None:
                bufs, peers = self._peer_dense
                peer_allreduce_sgd(self.fabric, world, {k: self.global_tm.w[k] for k in bufs},
                                   {m: {k: peers[m]["gtm_" + k] for k in bufs} for m in world},
                                   {m: {k: peers[m]["gtw_" + k] for k in bufs} for m in world},
                                   self.dense_lr, self.device)
                self.global_tm.grads = {}  # the summed gradient is never materialised
            else:
                self.fabric.all_reduce_(world, acc)
                self.global_tm.grads = acc
                self.global_tm.sgd_step(self.dense_lr)
            if dense_hook is not None:
                dense_hook()

        self.engine.backward(dx, self.lr, self.opt, self.eps, tm_lr=self.dense_lr, dense_hook=dense_step)

    def train_step(self, kjts: dict, grads: dict) -> dict:
        outs = self.forward(kjts, save=True)
        self.backward(grads)
        return outs

    def train_step_bce(self, kjts: dict, labels: dict) -> dict:
        """Full model step with a loss: SPTT forward, top head -> logit, binary
        cross-entropy against ``labels[r]`` (B,) fp32 (mean over the global
        batch), top backward, SPTT backward with the top's gradient all-reduce
        + SGD overlapped with the embedding update.  Returns {rank: loss (1,)}
        (rank r's share of the global mean loss)."""
        if self.top is None:
            raise DomainError("train_step_bce needs SPTT(top=...)")
        outs = self.forward(kjts, save=True)
        scale = 1.0 / (self.plan.G * self.plan.B)
        saved, gx, losses, acc = {}, {}, {}, {}
        for r, o in outs.items():
            with self.engine._t("top_fwd"):
                z = self.top.forward(o, save=True)
            buf = self._labels_loss.get(r)
            if buf is None:
                buf = self._labels_loss[r] = (torch.empty_like(z), torch.zeros(1, dtype=torch.float32,
                                                                               device=self.device))
            K.bce_with_logits(z, labels[r], scale, dz=buf[0], loss=buf[1])
            losses[r] = buf[1]
            with self.engine._t("top_bwd"):
                gx[r] = self.top.backward(buf[0])
            for k, v in self.top.grads.items():
                acc[k] = v.clone() if k not in acc else acc[k].add_(v)

        def top_step():  # world all-reduce of the head's grads + SGD
            self.fabric.all_reduce_(list(range(self.plan.G)), acc)
            self.top.grads = acc
            self.top.sgd_step(self.dense_lr)

        self.backward(gx, dense_hook=top_step)
        return losses

    def capture(self, kjts: dict, grads: Optional[dict], warmup: int = 2, timers=None, labels: Optional[dict] = None,
                step=None):
        """Capture one full train step (forward a-f, backward, optimizer
        updates) as a CUDA graph over the given static input buffers.

        Returns (replay, outs): copy the next batch into ``kjts``' lengths /
        values in place, then call replay().  Requires fixed per-feature nnz
        (uniform_nnz: no step-a counts exchange / host sync), or, for ragged
        batches, per-feature capacities (set_capacity; the static values
        buffer then holds sum(capacity) entries), and a fixed batch shape.  Every launch inside is a libdmt kernel or an NCCL collective on
        the capture stream; descriptor tables are content-cached, so replay
        issues no host work besides the graph launch."""
        self.engine.uniform_nnz = True
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        if step is None:  # a full-model step (e.g. dlrm.DLRM.train_step) may be passed in
            step = (lambda: self.train_step_bce(kjts, labels)) if labels is not None else (
                lambda: self.train_step(kjts, grads))
        with torch.cuda.stream(s):
            for _ in range(warmup):
                step()
        torch.cuda.current_stream().wait_stream(s)
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        self.engine.timers = timers  # external events -> graph nodes
        # the main chain is captured on a high-priority stream while the side
        # streams (embedding-backward prepare, crossnet backward tail) keep the
        # default lowest priority, so pending GEMM CTAs are scheduled ahead of
        # side-kernel CTAs: C2 step 2.89-2.93 -> 2.82-2.86 ms, tm_fwd 0.70 ->
        # 0.64 ms (same box).  DMT_CAPTURE_PRIORITY=default keeps the pool stream.
        cap = None if os.environ.get("DMT_CAPTURE_PRIORITY") == "default" else torch.cuda.Stream(priority=-1)
        try:
            with torch.cuda.graph(graph, stream=cap):
                outs = step()
        finally:
            self.engine.timers = None
        return graph.replay, outs


def build_world(G_hosts: int, ranks_per_host: int, hosts_per_tower: int, num_tables: int, rows: int, dim: int,
                seed: int = 0, dtype=np.float32, scheme: str = "table_wise", shards_per_table: int = 1,
                assignment: Optional[dict] = None):
    """Synthetic world: uniform(-1, 1) tables (embedding.py:58-60 generator),
    contiguous balanced feature->tower assignment, round-robin placement."""
    topo = ClusterTopology(G_hosts, ranks_per_host)
    W = ranks_per_host * hosts_per_tower
    layout = TowerLayout(topo.world_size // W, hosts_per_tower)
    T = layout.num_towers
    tables = {}
    for t in range(num_tables):
        vals = np.random.default_rng([seed, t]).uniform(-1.0, 1.0, size=(rows, dim)).astype(dtype)
        tables[t] = EmbeddingTable(t, rows, dim, vals)
    if assignment is None:
        base, extra = divmod(num_tables, T)
        assignment, f = {}, 0
        for t in range(T):
            for _ in range(base + (1 if t < extra else 0)):
                assignment[f] = t
                f += 1
    plan = {t: TablePlan(scheme, 1 if scheme == "table_wise" else shards_per_table, assignment[t]) for t in tables}
    return topo, layout, shard_tables(tables, plan, topo, layout), assignment


def device_world(G_hosts: int, ranks_per_host: int, hosts_per_tower: int, num_tables: int, rows: int, dim: int,
                 dtype: torch.dtype, local_ranks, seed: int = 0, device=None):
    """Large synthetic world whose tables are generated directly in HBM (the
    bench: 26 x 1M x 128 does not need a host copy).  Host-side EmbeddingTable
    values are zero-stride placeholders; only the shards owned by
    ``local_ranks`` are materialised, each filled with U(-1, 1) from a
    per-table seeded device generator."""
    topo = ClusterTopology(G_hosts, ranks_per_host)
    W = ranks_per_host * hosts_per_tower
    layout = TowerLayout(topo.world_size // W, hosts_per_tower)
    T = layout.num_towers
    tables = {}
    for t in range(num_tables):
        tab = object.__new__(EmbeddingTable)
        for k, v in (("table_id", t), ("rows", rows), ("dim", dim),
                     ("values", np.broadcast_to(np.float32(0), (rows, dim)))):
            object.__setattr__(tab, k, v)
        tables[t] = tab
    base, extra = divmod(num_tables, T)
    assignment, f = {}, 0
    for t in range(T):
        for _ in range(base + (1 if t < extra else 0)):
            assignment[f] = t
            f += 1
    from .embedding import Shard

    cursor = [0] * T
    shards = []
    for tid in range(num_tables):
        tw = assignment[tid]
        ranks = layout.tower_ranks(tw, topo)
        shards.append(Shard(tid, ranks[cursor[tw] % len(ranks)], "table_wise", (0, rows), (0, dim)))
        cursor[tw] += 1
    placement = ShardedEmbedding(tables, shards)
    device = device or torch.device("cuda")
    for sid, sh in enumerate(shards):
        if sh.rank in local_ranks:
            g = torch.Generator(device=device).manual_seed(seed * 1_000_003 + sh.table_id)
            w = torch.empty((rows, dim), dtype=torch.float32, device=device).uniform_(-1.0, 1.0, generator=g)
            placement._dev[(sid, dtype, str(device))] = w.to(dtype).contiguous()
            del w
    return topo, layout, placement, assignment


def random_kjt(F: int, B: int, rows: int, L_: int, gen: torch.Generator, device) -> KJT:
    """Fixed pooling factor L (C2/C3: L = 20), uniform indices (embedding.py:290)."""
    lengths = torch.full((F * B,), L_, dtype=torch.int32, device=device)
    values = torch.randint(0, rows, (F * B * L_,), generator=gen, device=device, dtype=torch.int32)
    return KJT(lengths=lengths, values=values, nnz_per_feature=[B * L_] * F, B=B)


def powerlaw_lengths(F: int, B: int, seed: int, mean: float = 20.0, cap: int = 200, alpha: float = 2.0) -> np.ndarray:
    """C5 pooling factors: a seeded Pareto(alpha) with scale
    chosen for the requested mean, truncated at ``cap`` and floored at 1,
    (F, B) int32.  The reference's make_batch only draws uniform [lo, hi]
    lengths (embedding.py:259-295); this builds the batch directly."""
    rng = np.random.default_rng(seed)
    xm = mean * (alpha - 1.0) / alpha
    x = xm * (1.0 - rng.random((F, B))) ** (-1.0 / alpha)
    return np.clip(np.floor(x), 1, cap).astype(np.int32)


def random_kjt_lengths(lengths: np.ndarray, rows: int, gen: torch.Generator, device) -> KJT:
    """KJT with the given (F, B) lengths and uniform indices in [0, rows);
    per-feature nnz known on the host (no device sync for step-a splits)."""
    F, B = lengths.shape
    nnz = [int(x) for x in lengths.sum(axis=1)]
    lens = torch.from_numpy(lengths.reshape(-1).copy()).to(device)
    values = torch.randint(0, rows, (max(1, sum(nnz)),), generator=gen, device=device, dtype=torch.int32)[:sum(nnz)]
    return KJT(lengths=lens, values=values, nnz_per_feature=nnz, B=B)
