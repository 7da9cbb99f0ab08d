"""Static routing plan of the exchange (host-side integers only).

Everything the device pipeline needs that does not depend on the index
*values*: which shard lives where, the step-a send slots, every buffer's
element layout and every collective's split sizes, for the SPTT pipeline
(towersim/exchange.py:275-462) and the flat baseline (exchange.py:200-241).
Pure Python -- unit-tested on CPU and under gloo without a GPU.

Buffer layouts (elements of the compute dtype unless noted):

* step a, src r -> owner o: for each shard sid in ``by_owner[o]`` (shard-id
  order) the B bag lengths of the shard's feature, then its values
  (exchange.py:172-178: the full bag list goes to every shard owner).
* owner r's received KJT: bag (p, k, b) = (p*S_r + k)*B + b for source p in
  rank order and its k-th shard.
* SPTT step-d send buffer of owner r (lookup output, step c fused):
  member c block = [shard k: (T*B, w_k)] with row j*B + b holding dest rank
  j*W + c -- the class-order stacking of exchange.py:319-365.
* step-d receive buffer of member m: owners of m's tower in group order, each
  [shard k: (T*B, w_k)].
* step-e X: (T*B, sum N_f over tower features ascending); TM maps it to
  Y (T*B, O_t) = step-f send buffer (block j -> tower-j class member).
* step-f receive: tower j block (B, O_j), j ascending -> output (B, sum O_j),
  tower-grouped like exchange.py:451-460.
* flat step-c send buffer of owner r: dest p block = [shard k: (B, w_k)];
  receive: owners in rank order, each [shard k: (B, w_k)].
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Optional, Sequence

from .embedding import ROW_WISE, Shard
from .errors import PlanError
from .topology import ClusterTopology, TowerLayout


@dataclass(frozen=True)
class Piece:
    """One source of an assembled feature: a shard block inside a buffer."""

    sid: int
    offset: int  # element offset of row 0 in the source buffer
    ld: int      # row stride (= shard width)
    c0: int      # shard column range start (within the feature)
    width: int


@dataclass(frozen=True)
class FeatureBlock:
    """Destination columns of one feature, and its pieces in combine order
    (exchange.py:112-127: row shards summed by row range, column shards
    concatenated by column range)."""

    feature: int
    dst_col: int
    width: int
    rowwise: bool
    pieces: tuple
    groups: int = 0  # row-wise reduce-scatter order: bit s = piece s starts an owner's partial


@dataclass
class ExchangePlan:
    topo: ClusterTopology
    layout: TowerLayout
    shards: list            # all placement shards (sid-indexed)
    features: list          # sorted batch features
    dims: dict              # feature -> embedding dim
    pooling: dict           # feature -> none|sum|mean
    B: int
    feature_towers: Optional[dict] = None
    tower_widths: Optional[dict] = None   # tower -> O_t (None = pass-through widths)
    G: int = 0
    W: int = 0
    T: int = 0
    fpos: dict = field(default_factory=dict)
    live: list = field(default_factory=list)
    by_owner: dict = field(default_factory=dict)
    S: dict = field(default_factory=dict)          # shards per owner
    SW: dict = field(default_factory=dict)         # sum of shard widths per owner
    pre: dict = field(default_factory=dict)        # owner -> prefix widths per k
    a_slots: list = field(default_factory=list)    # [(owner, sid)] owner-major
    a_slot_feature: list = field(default_factory=list)
    tower_features: dict = field(default_factory=dict)
    O: dict = field(default_factory=dict)          # tower -> output width

    def __post_init__(self) -> None:
        self.layout.validate_for(self.topo)
        self.G = self.topo.world_size
        self.W = self.layout.group_width(self.topo)
        self.T = self.layout.num_towers
        self.fpos = {f: i for i, f in enumerate(self.features)}
        fset = set(self.features)
        for f in self.features:
            if not any(s.table_id == f for s in self.shards):
                raise PlanError(f"table {f} has no shards")
        self.live = [sid for sid, s in enumerate(self.shards) if s.table_id in fset]
        self.by_owner = {o: [sid for sid in self.live if self.shards[sid].rank == o] for o in range(self.G)}
        for o in range(self.G):
            ws = [self.shards[sid].width for sid in self.by_owner[o]]
            self.S[o] = len(ws)
            self.SW[o] = sum(ws)
            acc, pre = 0, []
            for w in ws:
                pre.append(acc)
                acc += w
            self.pre[o] = pre
        self.a_slots = [(o, sid) for o in range(self.G) for sid in self.by_owner[o]]
        self.a_slot_feature = [self.fpos[self.shards[sid].table_id] for _, sid in self.a_slots]
        if self.feature_towers is not None:
            for f in self.features:
                if f not in self.feature_towers:
                    raise PlanError(f"feature {f} has no tower assignment")
                t = self.feature_towers[f]
                ranks = set(self.layout.tower_ranks(t, self.topo))
                owners = {s.rank for s in self.shards if s.table_id == f}
                if not owners <= ranks:
                    raise PlanError(f"feature {f} mapped to tower {t} but sharded on {sorted(owners)}")
            self.tower_features = {t: [f for f in self.features if self.feature_towers[f] == t]
                                   for t in range(self.T)}
            for t in range(self.T):
                pw = sum(self.dims[f] for f in self.tower_features[t])
                self.O[t] = (self.tower_widths or {}).get(t, pw)

    # ------------------------------------------------------------ step a ----
    def k_of(self, sid: int) -> int:
        return self.by_owner[self.shards[sid].rank].index(sid)

    def a_send_length_splits(self) -> list[int]:
        """Lengths (elements) src -> each owner (same for every src)."""
        return [self.S[o] * self.B for o in range(self.G)]

    def a_send_value_splits(self, nnz_of_feature: Sequence[int]) -> list[int]:
        """Values src -> each owner, given the src's nnz per feature position."""
        out = []
        for o in range(self.G):
            out.append(sum(int(nnz_of_feature[self.fpos[self.shards[sid].table_id]]) for sid in self.by_owner[o]))
        return out

    def a_slot_value_offsets(self, nnz_of_feature: Sequence[int]) -> list[int]:
        offs, acc = [], 0
        for f in self.a_slot_feature:
            offs.append(acc)
            acc += int(nnz_of_feature[f])
        offs.append(acc)
        return offs

    # ------------------------------------------------------------ step b ----
    def owner_bags(self, r: int) -> int:
        return self.G * self.S[r] * self.B

    def lookup_out_offsets(self, r: int, sptt: bool) -> list[tuple[int, int, int, int]]:
        """[(p, k, element offset of bag 0, row stride)] for owner r's segments."""
        B, T, W = self.B, self.T, self.W
        out = []
        for p in range(self.G):
            for k, sid in enumerate(self.by_owner[r]):
                w = self.shards[sid].width
                if sptt:
                    c, j = p % W, p // W
                    off = c * T * B * self.SW[r] + T * B * self.pre[r][k] + j * B * w
                else:
                    off = p * B * self.SW[r] + B * self.pre[r][k]
                out.append((p, k, off, w))
        return out

    def send_d_size(self, r: int) -> int:
        return self.W * self.T * self.B * self.SW[r]

    def send_c_size(self, r: int) -> int:
        return self.G * self.B * self.SW[r]

    # ------------------------------------------------------------ step d ----
    def tower_of(self, r: int) -> int:
        return r // self.W

    def group_of(self, r: int) -> list[int]:
        return self.layout.tower_ranks(self.tower_of(r), self.topo)

    def class_group_of(self, r: int) -> list[int]:
        c = r % self.W
        return [t * self.W + c for t in range(self.T)]

    def d_send_splits(self, r: int) -> list[int]:
        return [self.T * self.B * self.SW[r]] * self.W

    def d_recv_splits(self, r: int) -> list[int]:
        return [self.T * self.B * self.SW[o] for o in self.group_of(r)]

    def d_recv_offset(self, r: int, owner: int, k: int) -> int:
        off = 0
        for o in self.group_of(r):
            if o == owner:
                return off + self.T * self.B * self.pre[o][k]
            off += self.T * self.B * self.SW[o]
        raise PlanError(f"owner {owner} not in rank {r}'s tower")

    def _feature_blocks(self, feats, recv_offset, rs: bool = False) -> list[FeatureBlock]:
        """``rs``: row-wise features combine in the reduce-scatter order of
        exchange.py:380-395 -- each owner's shards summed in shard order, then
        the owners' partials in group (rank) order (simnet.py:173-192) -- instead
        of one sum in row-range order (_combine_pieces, exchange.py:112-127)."""
        blocks, col = [], 0
        for f in feats:
            sids = [sid for sid in self.live if self.shards[sid].table_id == f]
            schemes = {self.shards[s].scheme for s in sids}
            if ROW_WISE in schemes and schemes != {ROW_WISE}:
                raise PlanError("a table mixes row-wise and column-wise shards")
            rowwise = schemes == {ROW_WISE}
            if rowwise and rs:
                key = lambda s: (self.shards[s].rank, s)
            elif rowwise:
                key = lambda s: self.shards[s].row_range
            else:
                key = lambda s: self.shards[s].col_range
            pieces, groups, prev = [], 0, None
            for j, sid in enumerate(sorted(sids, key=key)):
                sh: Shard = self.shards[sid]
                pieces.append(Piece(sid, recv_offset(sh.rank, self.k_of(sid)), sh.width,
                                    0 if rowwise else sh.col_range[0], sh.width))
                if rowwise and rs and prev is not None and sh.rank != prev:
                    groups |= 1 << j
                prev = sh.rank
            if groups and len(pieces) > 32:
                raise PlanError("reduce-scatter order supports at most 32 row shards per table")
            blocks.append(FeatureBlock(f, col, self.dims[f], rowwise, tuple(pieces), groups))
            col += self.dims[f]
        return blocks

    def e_blocks(self, r: int, rs: bool = False) -> list[FeatureBlock]:
        """Step-d assemble / step-e regroup into X (T*B, sum N) for member r."""
        return self._feature_blocks(self.tower_features[self.tower_of(r)],
                                    lambda o, k: self.d_recv_offset(r, o, k))

    def x_width(self, r: int) -> int:
        return sum(self.dims[f] for f in self.tower_features[self.tower_of(r)])

    # ------------------------------------------------------------ step f ----
    def f_send_splits(self, r: int) -> list[int]:
        return [self.B * self.O[self.tower_of(r)]] * self.T

    def f_recv_splits(self, r: int) -> list[int]:
        return [self.B * self.O[t] for t in range(self.T)]

    def out_width(self) -> int:
        return sum(self.O[t] for t in range(self.T))

    def out_blocks_tower(self) -> list[tuple[int, int, int]]:
        """[(dst_col, width, recv_f element offset)] tower-grouped output."""
        out, col, off = [], 0, 0
        for t in range(self.T):
            out.append((col, self.O[t], off))
            col += self.O[t]
            off += self.B * self.O[t]
        return out

    # ------------------------------------------------------- flat step c ----
    def c_send_splits(self, r: int) -> list[int]:
        return [self.B * self.SW[r]] * self.G

    def c_recv_splits(self, r: int) -> list[int]:
        return [self.B * self.SW[o] for o in range(self.G)]

    def c_recv_offset(self, owner: int, k: int) -> int:
        return sum(self.B * self.SW[o] for o in range(owner)) + self.B * self.pre[owner][k]

    def c_blocks(self) -> list[FeatureBlock]:
        return self._feature_blocks(self.features, self.c_recv_offset)

    def flat_width(self) -> int:
        return sum(self.dims[f] for f in self.features)

    # ------------------------------------------------------------ layout ----
    def tower_layout_blocks(self, tm_kinds: dict) -> list[tuple[str, int, int]]:
        """exchange.py:451-460: ("tower", t, O_t) for TM towers, else features."""
        blocks = []
        for t in range(self.T):
            if tm_kinds.get(t, "passthrough") != "passthrough":
                blocks.append(("tower", t, self.O[t]))
            else:
                blocks.extend(("feature", f, self.dims[f]) for f in self.tower_features[t])
        return blocks

    # ------------------------------------------------------------ bytes ----
    def bytes_per_rank(self, elem_bytes: int) -> dict:
        """Wire bytes each rank SENDS to other ranks per step (the roofline's
        exchange bytes; self messages are free), worst rank."""
        out = {}
        B, G, T, W = self.B, self.G, self.T, self.W
        flat = max(sum(B * self.SW[r] for p in range(G) if p != r) for r in range(G)) if G else 0
        out["c"] = flat * elem_bytes
        if self.feature_towers is not None:
            d = max(sum(T * B * self.SW[r] for m in self.group_of(r) if m != r) for r in range(G))
            f = max((T - 1) * B * self.O[self.tower_of(r)] for r in range(G))
            out["d"], out["f"] = d * elem_bytes, f * elem_bytes
        return out
