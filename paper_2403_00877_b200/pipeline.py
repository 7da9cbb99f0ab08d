"""Device pipeline of the SPTT forward/backward and the flat baseline.

One engine instance serves the ranks hosted by this process: every rank on a
single GPU (LoopbackFabric, used by the reference-API drop-in and the parity
tests) or exactly one rank per GPU (NcclFabric, the distributed training
path).  Both run the same phases in the same order:

  forward  a  bucketize (dmt_kjt_bucketize) + all-to-all(v) of lengths/values
           b  offsets scan + pooled lookup straight into the step-d send buffer
              (class-order permute and stacking fused: dmt_pooled_lookup_fwd)
           d  tower all-to-all(v)                          (SPTT)   | c  world all-to-all (flat)
           e  assemble / regroup (dmt_assemble) + tower module GEMMs (dmt_gemm)
           f  per-class all-to-all, then output gather (dmt_assemble)
  backward f^-1 pack + class all-to-all, TM backward + tower all-reduce of the
           TM weight grads, d^-1 pack + tower all-to-all, then the fused
           sort/segment-reduce/optimizer embedding update (dmt_pooled_lookup_bwd)
           on the owner (no a^-1 exchange: the owner already holds the indices).

Reference: towersim/exchange.py:149-462 (forward only; the backward is new).
"""

from __future__ import annotations

import os
from dataclasses import dataclass
from typing import Optional, Sequence

import torch

from . import _lib as L
from . import kernels as K
from .embedding import POOL_MEAN, ROW_WISE, ShardedEmbedding
from .errors import DomainError
from .fabric import Fabric, peer_allreduce_sgd
from .plan import ExchangePlan
from .simnet import CommTrace


class PhaseTimers:
    """CUDA events around pipeline phases, on the stream the kernels run on
    (the current stream), for the bench's per-kernel roofline.  With
    ``external=True`` the events are recorded as CUDA-graph nodes, so a
    captured step reports its phases on every replay."""

    def __init__(self, external: bool = False):
        self.events: dict = {}
        self.external = external

    def scope(self, name: str):
        return _Scope(self, name)

    def reset(self) -> None:
        self.events = {}

    def ms(self) -> dict:
        out = {k: sum(a.elapsed_time(b) for a, b in v) for k, v in self.events.items()}
        ex = [v for k, v in out.items() if k.startswith("exchange_")]
        if ex:
            out["exchange"] = sum(ex)
        return out

    def count(self, name: str) -> int:
        return len(self.events.get(name, ()))


class _Scope:
    def __init__(self, timers, name):
        self.t, self.name = timers, name

    def __enter__(self):
        if self.t is not None:
            self.a = torch.cuda.Event(enable_timing=True, external=self.t.external)
            self.a.record()
        return self

    def __exit__(self, *exc):
        if self.t is not None:
            b = torch.cuda.Event(enable_timing=True, external=self.t.external)
            b.record()
            self.t.events.setdefault(self.name, []).append((self.a, b))
        return False


@dataclass
class KJT:
    """A rank's keyed jagged tensor, keys (features) major.

    lengths (F*B,) int32 and values (nnz,) int32 on the device; the host keeps
    the per-feature nnz (as TorchRec's length_per_key) so the step-a value
    splits need no device sync when every rank knows its own counts."""

    lengths: torch.Tensor
    values: torch.Tensor
    nnz_per_feature: list
    B: int
    offsets: Optional[torch.Tensor] = None

    @property
    def F(self) -> int:
        return len(self.nnz_per_feature)

    def ensure_offsets(self) -> torch.Tensor:
        if self.offsets is None:
            self.offsets = K.lengths_to_offsets(self.lengths)
        return self.offsets


def _too_many_towers(plan) -> bool:
    """Step-f fusion needs at most DMT_GEMM_MAX_OUT_GROUPS towers."""
    return plan.T > L.GEMM_MAX_OUT_GROUPS


class SpttEngine:
    def __init__(self, plan: ExchangePlan, placement: ShardedEmbedding, fabric: Fabric, dtype: torch.dtype,
                 device=None, tower_modules: Optional[dict] = None, mode: str = "sptt",
                 trace: Optional[CommTrace] = None, rowwise_reducescatter: bool = False):
        if mode not in ("sptt", "flat"):
            raise DomainError(f"unknown mode {mode!r}")
        if mode == "sptt" and plan.feature_towers is None:
            raise DomainError("SPTT mode needs feature_towers")
        self.plan, self.placement, self.fabric = plan, placement, fabric
        self.dtype = dtype
        self.es = torch.empty((), dtype=dtype).element_size()
        self.device = device or torch.device("cuda")
        self.tm = tower_modules or {}
        self.mode = mode
        self.trace = trace
        self.rs = rowwise_reducescatter
        self.local = list(fabric.local_ranks)
        p = plan
        dev = self.device
        self.weights = {sid: placement.device_shard(sid, dtype, dev) for r in self.local for sid in p.by_owner[r]}
        self.state = {}
        self.slot_feature = torch.tensor(p.a_slot_feature or [0], dtype=torch.int32, device=dev)
        # persistent buffers + descriptor tables (built once; pointers stay valid)
        self.buf = {}
        self.seg_fwd, self.seg_bwd = {}, {}
        self.asm_e, self.asm_out, self.asm_c = {}, {}, {}
        self.direct_x = {}
        sptt = mode == "sptt"
        for r in self.local:
            nsend = p.send_d_size(r) if sptt else p.send_c_size(r)
            b = {"send_x": torch.empty(max(1, nsend), dtype=dtype, device=dev),
                 "grad_x": torch.empty(max(1, nsend), dtype=dtype, device=dev)}
            if sptt:
                # singleton tower (W = 1): step d is the identity -> alias
                b["recv_d"] = (b["send_x"] if p.W == 1 else
                               torch.empty(max(1, sum(p.d_recv_splits(r))), dtype=dtype, device=dev))
                b["X"] = torch.empty((p.T * p.B, p.x_width(r)), dtype=dtype, device=dev)
                t = p.tower_of(r)
                if t not in self.tm and p.O[t] == p.x_width(r):
                    b["Y"] = b["X"]  # pass-through tower: X is the step-f send buffer
                else:
                    b["Y"] = torch.zeros((p.T * p.B, p.O[t]), dtype=dtype, device=dev)
                # singleton class (T = 1): step f is the identity -> alias
                b["recv_f"] = (b["Y"].view(-1) if p.T == 1 else
                               torch.empty(max(1, sum(p.f_recv_splits(r))), dtype=dtype, device=dev))
                # one tower: the tower-grouped output IS Y (no output gather)
                b["out"] = b["Y"] if p.T == 1 else torch.empty((p.B, p.out_width()), dtype=dtype, device=dev)
            else:
                b["recv_c"] = (b["send_x"] if p.G == 1 else
                               torch.empty(max(1, sum(p.c_recv_splits(r))), dtype=dtype, device=dev))
                b["out"] = torch.empty((p.B, p.flat_width()), dtype=dtype, device=dev)
            self.buf[r] = b
            xmap = self._direct_x_map(r) if sptt else None
            if xmap is not None:
                # one-rank tower (W = 1): steps c, d and the step-e regroup are
                # all identities up to layout, so the lookup pools straight into
                # the TM input X and the embedding backward reads its gradient
                # rows straight from dX (no assemble / scatter copies)
                b["gX"] = torch.empty_like(b["X"])
                self.direct_x[r] = xmap
                self.seg_fwd[r] = self._segments(r, b["X"], xmap=xmap)
                self.seg_bwd[r] = self._segments(r, b["gX"], with_keys=True, xmap=xmap)
            else:
                self.seg_fwd[r] = self._segments(r, b["send_x"])
                self.seg_bwd[r] = self._segments(r, b["grad_x"], with_keys=True)
            if sptt:
                self.asm_e[r] = self._assemble_table(p.e_blocks(r, rs=self.rs), b["recv_d"], b["X"], p.T * p.B)
                blocks = [K.Block(col, w, [(b["recv_f"], off, w)]) for col, w, off in p.out_blocks_tower()]
                self.asm_out[r] = K.AssembleTable(blocks, b["out"], p.B, dev)
            else:
                self.asm_c[r] = self._assemble_table(p.c_blocks(), b["recv_c"], b["out"], p.B)
        self._bwd_ws = {}
        self.timers: Optional[PhaseTimers] = None
        self.uniform_nnz = False
        self.capacity: Optional[list] = None  # per-feature value capacity (set_capacity)
        self.p2p_a = False
        # DMT_FUSE_F=0 / DMT_FUSE_D_BWD=0: keep step f / d^-1 as separate
        # peer-copy launches instead of fusing them into the TM GEMM epilogues
        self.fuse_f = os.environ.get("DMT_FUSE_F", "1") == "1"
        self.fuse_d_bwd = os.environ.get("DMT_FUSE_D_BWD", "1") == "1"
        self.c_bwd_fused = False
        # DMT_PEER_STEP_A=0 keeps step a on NCCL all-to-alls with the peer fabric
        self.peer_step_a = os.environ.get("DMT_PEER_STEP_A", "1") == "1"
        self._side = None
        self._prepared: dict = {}
        self.p2p_d = self.p2p_f = self.p2p_tm = self.p2p_c = False
        self.direct_peer_x = False
        if getattr(fabric, "p2p", False) and sptt:
            self._init_peer_links()
        elif getattr(fabric, "p2p", False) and plan.G > 1:
            self._init_peer_links_flat()

    # ------------------------------------------------------- NVLink peers ----
    def _init_peer_links(self) -> None:
        """Map every rank's exchange buffers (PeerFabric.share) and build the
        descriptor tables whose destinations are *peer* addresses: the pooled
        lookup writes its step-d blocks straight into the tower members'
        receive buffers (step c + d fused into the gather), and step f, f^-1
        and d^-1 become one peer-store launch each.  One rank per process."""
        p, dev = self.plan, self.device
        (r,) = self.local
        b = self.buf[r]
        self.p2p_d = p.W > 1
        self.p2p_f = p.T > 1
        share = {"recv_d": b["recv_d"], "recv_f": b["recv_f"], "grad_x": b["grad_x"], "X": b["X"]}
        if self.p2p_f:
            share["g_y"] = self._persist(r, "g_y", b["Y"])
        # TM gradients of a multi-rank tower: persistent fp32 buffers the tower
        # members read over NVLink (all-reduce fused with the SGD step)
        t = p.tower_of(r)
        # (dmt_peer_sum_sgd sums at most DMT_MAX_PEER_SRCS members; wider
        # towers keep the NCCL all-reduce + SGD)
        self.p2p_tm = 1 < p.W <= L.MAX_PEER_SRCS and t in self.tm
        self.tm_gbuf = {}
        if self.p2p_tm:
            # zero-size weights (e.g. DLRM w_flat with flat_outputs = 0) have no
            # gradient to exchange: a null pointer cannot be IPC-exported
            self.tm_gbuf = {k: torch.empty(v.shape, dtype=torch.float32, device=dev)
                            for k, v in self.tm[t].w.items() if v.numel()}
            share.update({"tmg_" + k: v for k, v in self.tm_gbuf.items()})
            share.update({"tmw_" + k: self.tm[t].w[k] for k in self.tm_gbuf})
        self.peer = self.fabric.share(share)
        if self.p2p_d:
            # without row-wise shards (no summed pieces) the lookup stores each
            # block straight into the member's TM input X (step e regroup
            # fused too); otherwise into its step-d receive buffer
            blocks = p.e_blocks(r)  # same feature layout for every member of the tower
            self.direct_peer_x = not any(fb.rowwise for fb in blocks)
            where = {pc.sid: fb.dst_col + pc.c0 for fb in blocks for pc in fb.pieces}
            xw = p.x_width(r)
            segs = []
            for seg, (pp, k, off, w) in zip(self.seg_fwd[r].segments, p.lookup_out_offsets(r, True)):
                c, j = pp % p.W, pp // p.W
                m = p.tower_of(r) * p.W + c
                if self.direct_peer_x:
                    dst, doff, dld = self.peer[m]["X"], j * p.B * xw + where[p.by_owner[r][k]], xw
                else:
                    dst, doff, dld = self.peer[m]["recv_d"], p.d_recv_offset(m, r, k) + j * p.B * w, w
                segs.append(K.Segment(weights=seg.weights, out=dst, out_offset=doff,
                                      out_ld=dld, bag_begin=seg.bag_begin, nbags=seg.nbags, pooling=seg.pooling,
                                      row_begin=seg.row_begin, row_filter=seg.row_filter, key_base=seg.key_base,
                                      table_rows=seg.table_rows))
            self.seg_fwd_p2p = K.SegmentTable(segs, dev)

    def _init_peer_links_flat(self) -> None:
        """The flat baseline over the same NVLink peer-store transport as SPTT
        (a fair comparison of the two exchange algorithms): the lookup stores
        every destination rank's block straight into that rank's step-c
        receive buffer, and c^-1 stores each gradient block straight into its
        owner's gradient buffer; a barrier completes each."""
        p, dev = self.plan, self.device
        (r,) = self.local
        b = self.buf[r]
        self.p2p_c = True
        self.peer = self.fabric.share({"recv_c": b["recv_c"], "grad_x": b["grad_x"]})
        segs = []
        for seg, (pp, k, off, w) in zip(self.seg_fwd[r].segments, p.lookup_out_offsets(r, False)):
            segs.append(K.Segment(weights=seg.weights, out=self.peer[pp]["recv_c"], out_offset=p.c_recv_offset(r, k),
                                  out_ld=w, bag_begin=seg.bag_begin, nbags=seg.nbags, pooling=seg.pooling,
                                  row_begin=seg.row_begin, row_filter=seg.row_filter, key_base=seg.key_base,
                                  table_rows=seg.table_rows))
        self.seg_fwd_p2p = K.SegmentTable(segs, dev)

    def flat_dx_scatter(self, r: int):
        """The flat baseline's c^-1 as a column scatter of the global TM's dX
        GEMM (see _d_bwd_fused_scatter); None unless fusable."""
        if not (self.p2p_c and self.fuse_d_bwd):
            return None
        p = self.plan
        groups, col, width = [], 0, None
        for fb in p.c_blocks():
            for pc in fb.pieces:
                if fb.rowwise or fb.dst_col + pc.c0 != col:
                    return None
                width = width or pc.width
                if pc.width != width or pc.ld != width:
                    return None
                o = self.placement.shards[pc.sid].rank
                k = p.k_of(pc.sid)
                off = r * p.B * p.SW[o] + p.B * p.pre[o][k]
                groups.append((self.peer[o]["grad_x"].data_ptr() + off * self.es, pc.ld))
                col += pc.width
        if not groups or width % 32 or len(groups) > L.GEMM_MAX_COL_GROUPS or col != p.flat_width():
            return None
        return width, groups

    def _d_bwd_fused_scatter(self, r: int):
        """(width, [(owner gradient-buffer address, row stride)] per dX column
        block) for the DCN's final dX GEMM to store d^-1 straight into the
        owners over NVLink; None unless every piece has one width (a multiple
        of 32) and the pieces tile X's columns in order."""
        if not self.fuse_d_bwd:
            return None
        p = self.plan
        c = r % p.W
        groups, col, width = [], 0, None
        for fb in p.e_blocks(r):
            for pc in fb.pieces:
                if fb.rowwise or fb.dst_col + pc.c0 != col:
                    return None
                if width is None:
                    width = pc.width
                if pc.width != width or pc.ld != width:
                    return None
                o = self.placement.shards[pc.sid].rank
                k = p.k_of(pc.sid)
                off = c * p.T * p.B * p.SW[o] + p.T * p.B * p.pre[o][k]
                groups.append((self.peer[o]["grad_x"].data_ptr() + off * self.es, pc.ld))
                col += pc.width
        if not groups or width % 32 or len(groups) > L.GEMM_MAX_COL_GROUPS or col != p.x_width(r):
            return None
        return width, groups

    def _f_fused_groups(self, r: int):
        """(B, [address of block j in the tower-j class member's step-f receive
        buffer]) for the TM projection GEMM to store into directly over NVLink
        (step f fused into the GEMM epilogue); None when not applicable."""
        if not self.fuse_f or _too_many_towers(self.plan):
            return None
        p = self.plan
        t, c = p.tower_of(r), r % p.W
        es = self.es
        off_recv = p.B * sum(p.O[t2] for t2 in range(t))
        return p.B, [self.peer[j * p.W + c]["recv_f"].data_ptr() + off_recv * es for j in range(p.T)]

    def _f_peer_copies(self, r: int) -> K.CopyTable:
        """Step f: Y block j -> the class member in tower j (its recv_f slot)."""
        p = self.plan
        t, c = p.tower_of(r), r % p.W
        Y = self.buf[r]["Y"]
        es = Y.element_size()
        blk = p.B * p.O[t]
        off_recv = p.B * sum(p.O[t2] for t2 in range(t))
        copies = []
        for j in range(p.T):
            dst = self.peer[j * p.W + c]["recv_f"]
            copies.append((Y.data_ptr() + j * blk * es, dst.data_ptr() + off_recv * es, blk * es))
        return K.CopyTable(copies, self.device)

    def _record_d(self, r: int) -> None:
        if self.trace is not None:
            for m in self.plan.group_of(r):
                self.trace.record_elements("d", r, m, self.plan.d_send_splits(r)[0], self.es)

    def _record_f(self, r: int) -> None:
        if self.trace is not None:
            for m in self.plan.class_group_of(r):
                self.trace.record_elements("f", r, m, self.plan.f_send_splits(r)[0], self.es)

    def _t(self, name: str):
        return _Scope(self.timers, name)

    def _persist(self, r: int, name: str, like: torch.Tensor) -> torch.Tensor:
        """Backward scratch kept across steps (stable pointers -> cached
        descriptor tables, capturable)."""
        t = self.buf[r].get(name)
        if t is None:
            t = torch.empty_like(like)
            self.buf[r][name] = t
        return t

    # ----------------------------------------------------------- tables ----
    def _direct_x_map(self, r: int) -> Optional[dict]:
        """{(src block p, shard k): (element offset in X, row stride)} when rank r
        is a one-rank tower whose TM input X can take the lookup output directly
        (no row-wise shard sums, every shard of r inside its tower), else None."""
        p = self.plan
        t = p.tower_of(r)
        if p.W != 1 or t not in self.tm:
            return None
        xw = p.x_width(r)
        where = {}
        for fb in p.e_blocks(r):
            if fb.rowwise:
                return None
            for pc in fb.pieces:
                where[pc.sid] = fb.dst_col + pc.c0
        xmap = {}
        for (pp, k, off, w) in p.lookup_out_offsets(r, True):
            sid = p.by_owner[r][k]
            if sid not in where:
                return None
            xmap[(pp, k)] = (pp * p.B * xw + where[sid], xw)
        return xmap

    def _segments(self, r: int, out: torch.Tensor, with_keys: bool = False,
                  xmap: Optional[dict] = None) -> K.SegmentTable:
        p = self.plan
        segs = []
        key_base, kb = {}, 0
        for sid in p.by_owner[r]:
            key_base[sid] = kb
            kb += self.placement.shards[sid].rows
        self.key_space = getattr(self, "key_space", {})
        self.key_space[r] = kb
        for (pp, k, off, w) in p.lookup_out_offsets(r, self.mode == "sptt"):
            if xmap is not None:
                off, w = xmap[(pp, k)]
            sid = p.by_owner[r][k]
            sh = self.placement.shards[sid]
            pool = p.pooling[sh.table_id]
            code = L.POOL_SUM if sh.scheme == ROW_WISE else L.POOL_CODE[pool]
            if sh.scheme == ROW_WISE and pool == POOL_MEAN:
                raise DomainError("mean pooling over row-wise shards is not defined (partials sum)")
            segs.append(K.Segment(weights=self.weights[sid], out=out, out_offset=off, out_ld=w,
                                  bag_begin=(pp * p.S[r] + k) * p.B, nbags=p.B, pooling=code,
                                  row_begin=sh.row_range[0], row_filter=sh.scheme == ROW_WISE,
                                  key_base=key_base[sid], state=self.state.get(sid),
                                  table_rows=self.placement.tables[sh.table_id].rows if sh.scheme == ROW_WISE
                                  else 0))
        return K.SegmentTable(segs, self.device)

    def _assemble_table(self, fblocks, src: torch.Tensor, dst: torch.Tensor, rows: int) -> K.AssembleTable:
        blocks = []
        for fb in fblocks:
            if fb.rowwise:
                blocks.append(K.Block(fb.dst_col, fb.width, [(src, pc.offset, pc.ld) for pc in fb.pieces],
                                      fb.groups))
            else:
                for pc in fb.pieces:
                    blocks.append(K.Block(fb.dst_col + pc.c0, pc.width, [(src, pc.offset, pc.ld)]))
        return K.AssembleTable(blocks, dst, rows, self.device)

    def enable_adagrad(self) -> None:
        """Allocate row-wise Adagrad accumulators (one fp32 per row) and
        rebuild the backward segment tables to point at them."""
        for r in self.local:
            for sid in self.plan.by_owner[r]:
                if sid not in self.state:
                    self.state[sid] = torch.zeros(self.placement.shards[sid].rows, dtype=torch.float32,
                                                  device=self.device)
            if self.direct_x.get(r):
                self.seg_bwd[r] = self._segments(r, self.buf[r]["gX"], with_keys=True, xmap=self.direct_x[r])
            else:
                self.seg_bwd[r] = self._segments(r, self.buf[r]["grad_x"], with_keys=True)

    def set_capacity(self, capacity: Optional[Sequence[int]]) -> None:
        """Capacity-padded step a for ragged batches (C5 power-law pooling)
        without a host sync: every rank's send slot of feature f holds
        ``capacity[f]`` values (>= that feature's nnz on any rank in any step),
        so the step-a splits are static, the owner packs the received regions
        on the device (dmt_kjt_compact) and the embedding backward sorts the
        padded count with the unused slots keyed invalid.  A feature exceeding
        its capacity sets a device flag (capacity_overflowed()).  None = off."""
        p = self.plan
        if capacity is None:
            self.capacity = None
            return
        if len(capacity) != len(p.features):
            raise DomainError("one capacity per feature position")
        self.capacity = [int(c) for c in capacity]
        dev = self.device
        self._cap_dev = K.device_ints(self.capacity, torch.int64, dev)
        self._cap_flag = torch.zeros(1, dtype=torch.int32, device=dev)
        self._cap_seg = {}
        # device byte counters of step a: owner o's slots are a_slots[b_o:e_o]
        bounds, s0 = [], 0
        for o in range(p.G):
            bounds.append((s0, s0 + len(p.by_owner[o])))
            s0 += len(p.by_owner[o])
        self._owner_slot_begin = torch.tensor([b for b, _ in bounds], dtype=torch.long, device=dev)
        self._owner_slot_end = torch.tensor([e for _, e in bounds], dtype=torch.long, device=dev)
        for r in self.local:
            caps = [self.capacity[p.fpos[p.shards[sid].table_id]] for sid in p.by_owner[r]]
            C_r = sum(caps)
            starts, acc = [], 0
            for c in caps:
                starts.append(acc)
                acc += c
            self._cap_seg[r] = K.device_ints([pp * C_r + s for pp in range(p.G) for s in starts] or [0],
                                             torch.int64, dev)

    def capacity_overflowed(self) -> bool:
        """True if a capacity-padded step saw a feature over its capacity
        (host sync; check it outside the timed loop)."""
        return self.capacity is not None and bool(self._cap_flag.item())

    def _init_peer_step_a(self, nnz_pf) -> None:
        """Step a over NVLink peer stores (uniform or capacity-padded value
        counts, so every slot's place in its owner's receive buffer is
        static): persistent receive buffers shared with the world, and the
        per-slot destination table of dmt_kjt_bucketize_peer.  Collective
        (every rank calls it in the same step, outside graph capture)."""
        p, dev = self.plan, self.device
        (r,) = self.local
        fpos = lambda sid: p.fpos[p.shards[sid].table_id]
        C = {o: sum(int(nnz_pf[fpos(sid)]) for sid in p.by_owner[o]) for o in range(p.G)}
        a_len = torch.empty(max(1, p.owner_bags(r)), dtype=torch.int32, device=dev)
        a_val = torch.empty(max(1, p.G * C[r]), dtype=torch.int32, device=dev)
        peers = self.fabric.share({"a_len": a_len, "a_val": a_val})
        slots = []
        for o, sid in p.a_slots:
            k = p.by_owner[o].index(sid)
            off = sum(int(nnz_pf[fpos(s2)]) for s2 in p.by_owner[o][:k])
            slots.append(L.SlotDst(len=peers[o]["a_len"].data_ptr() + 4 * (r * p.S[o] + k) * p.B,
                                   val=peers[o]["a_val"].data_ptr() + 4 * (r * C[o] + off),
                                   room=int(nnz_pf[fpos(sid)])))
        self._a_table, _ = K.device_table(L.SlotDst, slots, dev)
        self._a_bufs = (a_len, a_val)
        self._a_key = tuple(int(x) for x in nnz_pf)
        self.p2p_a = True

    # ---------------------------------------------------------- forward ----
    def forward(self, kjts: dict, save: bool = False, check_indices: bool = False) -> dict:
        p, fab, dev = self.plan, self.fabric, self.device
        world = list(range(p.G))
        # step a over NVLink peers when every slot's place is static
        peer_a = (getattr(fab, "p2p", False) and p.G > 1 and len(self.local) == 1 and bool(p.a_slots)
                  and (self.uniform_nnz or self.capacity is not None) and self.peer_step_a)
        if peer_a:
            (r,) = self.local
            nnz_pf = kjts[r].nnz_per_feature if self.capacity is None else self.capacity
            if getattr(self, "_a_key", None) != tuple(int(x) for x in nnz_pf):
                if torch.cuda.is_current_stream_capturing():
                    raise DomainError("step-a peer buffers must be set up by an eager step before capture")
                self._init_peer_step_a(nnz_pf)
            return self._forward_after_a(kjts, save, check_indices, peer_a=True)
        return self._forward_after_a(kjts, save, check_indices, peer_a=False)

    def _forward_after_a(self, kjts: dict, save: bool, check_indices: bool, peer_a: bool) -> dict:
        p, fab, dev = self.plan, self.fabric, self.device
        world = list(range(p.G))
        if (p.G == 1 and len(self.local) == 1 and self.capacity is None and self.trace is None
                and list(p.a_slot_feature) == list(range(len(p.features)))):
            # one rank whose slots are the features in order: the bucketized
            # KJT is the input KJT itself (no bucketize pass, offsets reused)
            (r,) = self.local
            kj = kjts[r]
            if kj.B != p.B or kj.F != len(p.features):
                raise DomainError("KJT shape does not match the plan")
            offs = kj.offsets if kj.offsets is not None else K.lengths_to_offsets(kj.lengths)
            return self._forward_from_b({r: kj.lengths}, {r: kj.values},
                                        {r: p.a_send_value_splits(kj.nnz_per_feature)}, save, check_indices,
                                        recv_offs={r: offs})
        # step a: bucketize per src, exchange lengths then values
        send_len, send_val, len_splits, val_splits = {}, {}, {}, {}
        for r in self.local:
            kj = kjts[r]
            if kj.B != p.B or kj.F != len(p.features):
                raise DomainError("KJT shape does not match the plan")
            offs = kj.offsets if kj.offsets is not None else K.lengths_to_offsets(kj.lengths)
            nnz_pf = kj.nnz_per_feature if self.capacity is None else self.capacity
            if self.capacity is not None:
                K.kjt_check_capacity(offs, p.B, self._cap_dev, self._cap_flag)
            if peer_a:
                # every slot straight into its owner's receive buffers, then a
                # world barrier (replaces the lengths + values all-to-alls)
                K.kjt_bucketize_peer(kj.lengths, offs, kj.values, p.B, self.slot_feature, self._a_table)
                if self.trace is not None:
                    if self.capacity is not None:
                        self._record_a_device(r, offs, world)
                    else:
                        for j, dst in enumerate(world):
                            self.trace.record_elements("a", r, dst, p.a_send_value_splits(nnz_pf)[j], 4)
                continue
            slot_offs = p.a_slot_value_offsets(nnz_pf)
            total = slot_offs[-1]
            send_len[r] = torch.empty(max(1, len(p.a_slots) * p.B), dtype=torch.int32, device=dev)
            send_val[r] = torch.empty(max(1, total), dtype=torch.int32, device=dev)
            if p.a_slots:
                so = K.device_ints(slot_offs, torch.int64, dev)
                K.kjt_bucketize(kj.lengths, offs, kj.values, p.B, self.slot_feature, so, send_len[r], send_val[r])
                if self.capacity is not None and self.trace is not None:
                    self._record_a_device(r, offs, world)
            len_splits[r] = p.a_send_length_splits()
            val_splits[r] = p.a_send_value_splits(nnz_pf)
        if peer_a:
            (r,) = self.local
            with self._t("exchange_a"):
                fab.barrier_(world)
            recv_len, recv_val = {r: self._a_bufs[0]}, {r: self._a_bufs[1]}
            recv_val_splits = {r: [sum(int(nnz_pf[p.fpos[p.shards[sid].table_id]]) for sid in p.by_owner[r])]
                               * p.G}
            return self._forward_from_b(recv_len, recv_val, recv_val_splits, save, check_indices)
        if self.uniform_nnz or self.capacity is not None:
            # fixed pooling factors: every rank ships the same per-feature nnz,
            # so owner r receives val_splits[r][r] from every source and the
            # ragged step-a splits need no counts exchange (no host sync -> the
            # step is CUDA-graph capturable)
            recv_val_splits = {r: [val_splits[r][r]] * p.G for r in self.local}
        else:
            with self._t("exchange_counts"):
                recv_val_splits = fab.exchange_counts(world, val_splits)
        recv_len, recv_val = {}, {}
        for r in self.local:
            if p.G == 1:  # single rank: step a is the identity
                recv_len[r], recv_val[r] = send_len[r], send_val[r]
                continue
            recv_len[r] = torch.empty(max(1, p.owner_bags(r)), dtype=torch.int32, device=dev)
            recv_val[r] = torch.empty(max(1, sum(recv_val_splits[r])), dtype=torch.int32, device=dev)
        with self._t("exchange_a_len"):
            fab.alltoallv(world, "a_len", send_len, len_splits, recv_len,
                          {r: [p.S[r] * p.B] * p.G for r in self.local})
        with self._t("exchange_a"):
            fab.alltoallv(world, "a", send_val, val_splits, recv_val, recv_val_splits,
                          None if self.capacity is not None else self.trace, 4)
        return self._forward_from_b(recv_len, recv_val, recv_val_splits, save, check_indices)

    def _record_a_device(self, r: int, offs: torch.Tensor, world: list) -> None:
        """Step-a payload bytes from device counters (capacity mode: the host
        only knows capacities; each slot ships its actual nnz)."""
        p = self.plan
        packed = self.buf[r].get("a_slot_packed")
        if packed is None:
            packed = self.buf[r]["a_slot_packed"] = torch.empty(len(p.a_slots) + 1, dtype=torch.int64,
                                                                device=self.device)
        K.kjt_slot_offsets(offs, p.B, self.slot_feature, packed)
        counts = packed[self._owner_slot_end] - packed[self._owner_slot_begin]
        self.trace.record_device("a", r, world, counts, 4)

    def _forward_from_b(self, recv_len: dict, recv_val: dict, recv_val_splits: dict, save: bool,
                        check_indices: bool, recv_offs: Optional[dict] = None) -> dict:
        p, fab, dev = self.plan, self.fabric, self.device
        # step b: lookup (+ fused permute) on every owner
        self._owner = {}
        err = torch.zeros(1, dtype=torch.int32, device=dev) if check_indices else None
        for r in self.local:
            if recv_offs is not None:
                offsets = recv_offs[r]
            else:
                offsets = K.lengths_to_offsets(recv_len[r][: p.owner_bags(r)])
            nnz = sum(recv_val_splits[r])
            if self.capacity is not None:
                # pack the capacity-padded (src, shard) regions back to back
                packed = self._persist(r, "recv_val_packed", recv_val[r])
                K.kjt_compact(recv_val[r], offsets, p.B, self._cap_seg[r][: p.G * p.S[r]], packed)
                recv_val[r] = packed
            if save and self._prepare_with_lookup:
                self._launch_prepare(r, offsets, recv_val[r], nnz)
            with self._t("lookup_fwd"):
                table = self.seg_fwd_p2p if (self.p2p_d or self.p2p_c) else self.seg_fwd[r]
                K.pooled_lookup_fwd(table, offsets, recv_val[r], err)
            self._owner[r] = (offsets, recv_val[r], nnz)
            if save and not self._prepare_with_lookup:
                # the embedding backward's key build + radix sort need only the
                # indices: run them on a side stream, overlapped with the tower
                # module forward/backward and the exchanges (joined in backward)
                self._launch_prepare(r, offsets, recv_val[r], nnz)
        if err is not None:
            K.raise_lookup_errors(err)
        if self.mode == "flat":
            return self._flat_forward()
        # step d: tower all-to-alls (or, over NVLink peers, the lookup already
        # stored every block in its member's receive buffer: barrier only)
        send = {r: self.buf[r]["send_x"] for r in self.local}
        recv = {r: self.buf[r]["recv_d"] for r in self.local}
        for g in self._groups(p.group_of):
            if self.p2p_d:
                self._record_d(self.local[0])
                with self._t("exchange_d"):
                    fab.barrier_(g)
                continue
            self._trace_d(g)
            with self._t("exchange_d"):
                fab.alltoallv(g, "d", send, {r: p.d_send_splits(r) for r in g}, recv,
                              {r: p.d_recv_splits(r) for r in g}, None)
        # step e: regroup + tower module
        for r in self.local:
            if not (self.direct_x.get(r) or self.direct_peer_x):
                self.asm_e[r].run()
            t = p.tower_of(r)
            if t in self.tm:
                groups = self._f_fused_groups(r) if (self.p2p_f and self.tm[t].cfg.kind == "dcn") else None
                with self._t("tm_fwd"):
                    self.tm[t].forward(self.buf[r]["X"], save=save, out=self.buf[r]["Y"], out_groups=groups)
                if save:
                    self.buf[r]["tm_saved"] = self.tm[t]._saved
        # step f: per-class all-to-alls, then tower-grouped output
        send = {r: self.buf[r]["Y"].view(-1) for r in self.local}
        recv = {r: self.buf[r]["recv_f"] for r in self.local}
        for g in self._groups(p.class_group_of):
            if self.p2p_f:
                (r,) = self.local
                self._record_f(r)
                with self._t("exchange_f"):
                    if not self._f_fused_groups(r) or p.tower_of(r) not in self.tm or \
                            self.tm[p.tower_of(r)].cfg.kind != "dcn":
                        if "f_copies" not in self.buf[r]:
                            self.buf[r]["f_copies"] = self._f_peer_copies(r)
                        self.buf[r]["f_copies"].run()  # peer stores over NVLink
                    fab.barrier_(g)
                continue
            with self._t("exchange_f"):
                fab.alltoallv(g, "f", send, {r: p.f_send_splits(r) for r in g}, recv,
                              {r: p.f_recv_splits(r) for r in g}, self.trace, self.es)
        out = {}
        for r in self.local:
            if self.buf[r]["out"] is not self.buf[r]["Y"]:
                self.asm_out[r].run()
            out[r] = self.buf[r]["out"]
        return out

    def _flat_forward(self) -> dict:
        p, fab = self.plan, self.fabric
        world = list(range(p.G))
        send = {r: self.buf[r]["send_x"] for r in self.local}
        recv = {r: self.buf[r]["recv_c"] for r in self.local}
        if self.p2p_c:  # the lookup already stored every block in its receiver
            (r,) = self.local
            if self.trace is not None:
                for j, dst in enumerate(world):
                    self.trace.record_elements("c", r, dst, p.c_send_splits(r)[j], self.es)
            with self._t("exchange_c"):
                fab.barrier_(world)
        else:
            with self._t("exchange_c"):
                fab.alltoallv(world, "c", send, {r: p.c_send_splits(r) for r in world}, recv,
                              {r: p.c_recv_splits(r) for r in world}, self.trace, self.es)
        out = {}
        for r in self.local:
            self.asm_c[r].run()
            out[r] = self.buf[r]["out"]
        return out

    def _groups(self, group_fn) -> list:
        seen, out = set(), []
        for r in self.local:
            g = tuple(group_fn(r))
            if g not in seen:
                seen.add(g)
                out.append(list(g))
        return out

    def _trace_d(self, group) -> None:
        """Step-d byte accounting exactly as the reference records it
        (exchange.py:367-395), including the reduce-scatter form."""
        if self.trace is None:
            return
        p = self.plan
        rs_tables = set()
        if self.rs:
            rs_tables = {f for f in p.features
                         if any(s.scheme == ROW_WISE for s in self.placement.shards if s.table_id == f)}
        tower = p.tower_of(group[0])
        for owner in group:
            for member in group:
                if owner not in self.fabric.local_ranks and member not in self.fabric.local_ranks:
                    continue
                if owner not in self.fabric.local_ranks:
                    continue
                n = sum(p.T * p.B * self.placement.shards[sid].width for sid in p.by_owner[owner]
                        if self.placement.shards[sid].table_id not in rs_tables)
                self.trace.record_elements("d", owner, member, n, self.es)
        for f in p.tower_features[tower]:
            if f not in rs_tables:
                continue
            contributors = sorted({self.placement.shards[sid].rank for sid in p.live
                                   if self.placement.shards[sid].table_id == f})
            for dst in group:
                for src in group:
                    if src in contributors and src in self.fabric.local_ranks:
                        self.trace.record_elements("d", src, dst, p.T * p.B * p.dims[f], self.es)

    # --------------------------------------------------------- backward ----
    def backward(self, grad_out: dict, lr: float, optimizer: int = L.OPT_SGD, eps: float = 1e-8,
                 tm_lr: Optional[float] = None, dense_hook=None) -> None:
        """Backward of the last forward(save=True) + fused optimizer updates."""
        p, fab, dev = self.plan, self.fabric, self.device
        if self.mode == "flat":
            return self._flat_backward(grad_out, lr, optimizer, eps, dense_hook)
        # f^-1: pack the tower-grouped gradient into per-tower blocks (the step-f
        # receive layout), send each block back to the member that produced it
        gsend, grecv = {}, {}
        for r in self.local:
            if self.p2p_f:
                # f^-1 over NVLink: the tower-t column block goes straight into
                # the tower-t class member's g_y rows of this rank's tower
                t_r, c = p.tower_of(r), r % p.W
                copies, col, ow = [], 0, p.out_width()
                for t in range(p.T):
                    dst = self.peer[t * p.W + c]["g_y"]
                    copies.append((grad_out[r], col, ow, dst, t_r * p.B * p.O[t], p.O[t], p.B, p.O[t]))
                    col += p.O[t]
                with self._t("exchange_f_bwd"):
                    K.Copy2DTable(copies, dev).run()
                    fab.barrier_(p.class_group_of(r))
                grecv[r] = self.buf[r]["g_y"]
                continue
            go = grad_out[r]
            if p.T == 1 and go.is_contiguous() and tuple(go.shape) == (p.B, p.O[p.tower_of(r)]):
                # one tower: the output gradient already is the TM's gy layout
                gsend[r], grecv[r] = go.view(-1), go
                continue
            gf = self._persist(r, "g_f", self.buf[r]["recv_f"])
            copies = []
            col, off = 0, 0
            ow = p.out_width()
            for t in range(p.T):
                copies.append((grad_out[r], col, ow, gf, off, p.O[t], p.B, p.O[t]))
                col += p.O[t]
                off += p.B * p.O[t]
            K.Copy2DTable(copies, dev).run()
            gsend[r] = gf
            grecv[r] = (gf.view(p.T * p.B, p.O[p.tower_of(r)]) if p.T == 1 else
                        self._persist(r, "g_y", self.buf[r]["Y"]))
        for g in ([] if self.p2p_f else self._groups(p.class_group_of)):
            with self._t("exchange_f_bwd"):
                fab.alltoallv(g, "f_bwd", gsend, {r: p.f_recv_splits(r) for r in g}, {r: grecv[r].view(-1) for r in self.local},
                              {r: p.f_send_splits(r) for r in g})
        # e^-1: tower module backward (weight grads summed over the tower)
        dX = {}
        tower_grads = {}
        for r in self.local:
            t = p.tower_of(r)
            if t in self.tm:
                self.tm[t]._saved = self.buf[r]["tm_saved"]
                # a one-rank tower needs no gradient all-reduce: fuse the weight
                # SGD into the dW GEMM epilogues
                fused = (tm_lr if tm_lr is not None else lr) if p.W == 1 else None
                scatter = self._d_bwd_fused_scatter(r) if (self.p2p_d and self.tm[t].cfg.kind == "dcn") else None
                with self._t("tm_bwd"):
                    dX[r] = self.tm[t].backward(grecv[r], fused_lr=fused,
                                                dx_out=self.buf[r]["gX"] if self.direct_x.get(r) else None,
                                                dx_scatter=scatter)
                self._d_bwd_fused = scatter is not None and self.tm[t]._dx_scatter is not None
                acc = tower_grads.setdefault(t, {})
                for k, v in self.tm[t].grads.items():
                    if self.p2p_tm:  # one rank per process: into the peer-shared buffer
                        acc[k] = self.tm_gbuf[k].view(v.shape).copy_(v) if v.numel() else v
                    else:
                        acc[k] = v.clone() if k not in acc else acc[k].add_(v)
            else:
                dX[r] = grecv[r]
        # d^-1: scatter dX columns back into the step-d receive layout
        dsend, drecv = {}, {}
        for r in self.local:
            if self.direct_x.get(r):
                continue  # the embedding backward reads gX directly
            if self.p2p_d and getattr(self, "_d_bwd_fused", False):
                with self._t("exchange_d_bwd"):  # the dX GEMM already stored every block
                    fab.barrier_(p.group_of(r))
                continue
            if self.p2p_d:
                # d^-1 over NVLink: scatter dX columns straight into every
                # owner's gradient buffer (its step-d send layout, member block c)
                c = r % p.W
                copies, xw = [], p.x_width(r)
                for fb in p.e_blocks(r):
                    for pc in fb.pieces:
                        o = self.placement.shards[pc.sid].rank
                        k = p.k_of(pc.sid)
                        dst = self.peer[o]["grad_x"]
                        off = c * p.T * p.B * p.SW[o] + p.T * p.B * p.pre[o][k]
                        copies.append((dX[r], fb.dst_col + pc.c0, xw, dst, off, pc.ld, p.T * p.B, pc.width))
                with self._t("exchange_d_bwd"):
                    K.Copy2DTable(copies, dev).run()
                    fab.barrier_(p.group_of(r))
                continue
            gd = self.buf[r]["grad_x"] if p.W == 1 else self._persist(r, "g_d", self.buf[r]["recv_d"])
            copies = []
            xw = p.x_width(r)
            for fb in p.e_blocks(r):
                for pc in fb.pieces:
                    copies.append((dX[r], fb.dst_col + pc.c0, xw, gd, pc.offset, pc.ld, p.T * p.B, pc.width))
            K.Copy2DTable(copies, dev).run()
            dsend[r] = gd
            drecv[r] = self.buf[r]["grad_x"]
        for g in ([] if self.p2p_d else self._groups(p.group_of)):
            if any(self.direct_x.get(r) for r in g):
                continue  # one-rank tower: dX already is the gradient layout
            with self._t("exchange_d_bwd"):
                fab.alltoallv(g, "d_bwd", dsend, {r: p.d_recv_splits(r) for r in g}, drecv,
                              {r: p.d_send_splits(r) for r in g})

        def tm_reduce_and_step():
            for t, grads in tower_grads.items():
                group = p.layout.tower_ranks(t, p.topo)
                if self.p2p_tm:
                    # NVLink reduce-scatter + SGD + all-gather: member i sums
                    # slice i of the members' gradient buffers in tower-rank
                    # order into its replica, then copies the others' updated
                    # slices (bit-identical replicas).  A member overwrites its
                    # gradient buffer / weights only after the next step's
                    # step-d barrier, which every reader passes after this
                    # side stream is joined.
                    ks = [k for k in grads if k in self.tm_gbuf]
                    peer_allreduce_sgd(fab, group, {k: self.tm[t].w[k] for k in ks},
                                       {m: {k: self.peer[m]["tmg_" + k] for k in ks} for m in group},
                                       {m: {k: self.peer[m]["tmw_" + k] for k in ks} for m in group},
                                       tm_lr if tm_lr is not None else lr, dev)
                    # the tower-summed gradient is never materialised on this
                    # path (each member folds the peers' buffers straight into
                    # its weights): leave no rank-local partial behind that a
                    # caller could mistake for the summed gradient
                    self.tm[t].grads = {}
                    continue
                fab.all_reduce_(group, grads)
                self.tm[t].grads = grads
                self.tm[t].sgd_step(tm_lr if tm_lr is not None else lr)
            if dense_hook is not None:  # data-parallel layers above SPTT (world all-reduce + SGD)
                dense_hook()

        self.overlap_with_embedding_update(tm_reduce_and_step, lr, optimizer, eps)

    def overlap_with_embedding_update(self, fn, lr, optimizer, eps) -> None:
        """Run ``fn`` (dense-gradient all-reduce + SGD) on a side stream while the
        fused embedding update runs on the current one.  ``fn``'s collectives are
        enqueued after the backward all-to-alls on the same communicators, so
        they execute while the (HBM-bound) update kernel runs."""
        side = self._side_stream2()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            with self._t("overlapped_allreduce"):  # not exposed: hidden under the update
                fn()
        self._embedding_update(lr, optimizer, eps)
        torch.cuda.current_stream().wait_stream(side)

    def _side_stream2(self):
        if getattr(self, "_side2", None) is None:
            self._side2 = torch.cuda.Stream(device=self.device)
        return self._side2

    def _flat_backward(self, grad_out, lr, optimizer, eps, dense_hook=None):
        p, fab, dev = self.plan, self.fabric, self.device
        world = list(range(p.G))
        gsend = {}
        fw = p.flat_width()
        if self.p2p_c and self.c_bwd_fused:
            self.c_bwd_fused = False
            with self._t("exchange_c_bwd"):  # the global TM's dX GEMM already stored every block
                fab.barrier_(world)
            if dense_hook is None:
                self._embedding_update(lr, optimizer, eps)
            else:
                self.overlap_with_embedding_update(dense_hook, lr, optimizer, eps)
            return
        if self.p2p_c:
            # c^-1 over NVLink: each feature block of this rank's output
            # gradient goes straight into its owner's gradient buffer (the
            # owner's step-c send layout, source block r)
            (r,) = self.local
            copies = []
            for fb in p.c_blocks():
                for pc in fb.pieces:
                    o = self.placement.shards[pc.sid].rank
                    k = p.k_of(pc.sid)
                    copies.append((grad_out[r], fb.dst_col + pc.c0, fw, self.peer[o]["grad_x"],
                                   r * p.B * p.SW[o] + p.B * p.pre[o][k], pc.ld, p.B, pc.width))
            with self._t("exchange_c_bwd"):
                K.Copy2DTable(copies, dev).run()
                fab.barrier_(world)
            if dense_hook is None:
                self._embedding_update(lr, optimizer, eps)
            else:
                self.overlap_with_embedding_update(dense_hook, lr, optimizer, eps)
            return
        for r in self.local:
            gc = self.buf[r]["grad_x"] if p.G == 1 else self._persist(r, "g_c", self.buf[r]["recv_c"])
            copies = []
            for fb in p.c_blocks():
                for pc in fb.pieces:
                    copies.append((grad_out[r], fb.dst_col + pc.c0, fw, gc, pc.offset, pc.ld, p.B, pc.width))
            K.Copy2DTable(copies, dev).run()
            gsend[r] = gc
        with self._t("exchange_c_bwd"):
            fab.alltoallv(world, "c_bwd", gsend, {r: p.c_recv_splits(r) for r in world},
                          {r: self.buf[r]["grad_x"] for r in self.local}, {r: p.c_send_splits(r) for r in world})
        if dense_hook is None:
            self._embedding_update(lr, optimizer, eps)
        else:
            self.overlap_with_embedding_update(dense_hook, lr, optimizer, eps)

    # DMT_PREPARE_INLINE=1: run the embedding-backward prepare (keys + sort)
    # on the launching stream instead of overlapping it with the tower module;
    # DMT_PREPARE_AT=lookup: fork it before the lookup so it overlaps the
    # (HBM-bound) lookup rather than the persistent tower-module GEMMs
    _prepare_inline = os.environ.get("DMT_PREPARE_INLINE", "0") == "1"
    _prepare_with_lookup = os.environ.get("DMT_PREPARE_AT", "tm") == "lookup"

    def _launch_prepare(self, r, offsets, vals, nnz) -> None:
        side = self._side_stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            K.pooled_lookup_bwd_prepare(self.seg_bwd[r], offsets, vals, nnz, self.key_space[r],
                                        self._bwd_workspace(r, nnz))
        self._prepared[r] = True

    def _side_stream(self):
        if self._prepare_inline:
            return torch.cuda.current_stream()
        if self._side is None:
            self._side = torch.cuda.Stream(device=self.device)
        return self._side

    def _bwd_workspace(self, r: int, nnz: int) -> torch.Tensor:
        need = L.lib().dmt_pooled_lookup_bwd_workspace_size(nnz, self.key_space[r], self.plan.owner_bags(r))
        ws = self._bwd_ws.get(r)
        if ws is None or ws.numel() < need:
            ws = torch.empty(max(1, need), dtype=torch.uint8, device=self.device)
            self._bwd_ws[r] = ws
        return ws

    def _embedding_update(self, lr, optimizer, eps):
        if optimizer == L.OPT_ROWWISE_ADAGRAD and not self.state:
            self.enable_adagrad()
            self._prepared = {}  # records must point at the new state arrays
        for r in self.local:
            offsets, vals, nnz = self._owner[r]
            ks = self.key_space[r]
            ws = self._bwd_workspace(r, nnz)
            with self._t("lookup_bwd"):
                if self._prepared.get(r):
                    if self._side is not None:
                        torch.cuda.current_stream().wait_stream(self._side)
                    K.pooled_lookup_bwd_apply(self.seg_bwd[r], nnz, ks, optimizer, lr, eps, ws)
                else:
                    K.pooled_lookup_bwd(self.seg_bwd[r], offsets, vals, nnz, ks, optimizer, lr, eps, ws)
            self._prepared[r] = False
