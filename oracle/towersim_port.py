"""numpy restatement of the reference SPTT forward path -- TEST INFRASTRUCTURE ONLY.

Every function cites the reference location it restates (paths relative to
/root/reference/pkg/src/towersim/).  Inputs are KJT-form arrays rather than the
reference's nested Python lists:

* ``lengths``  int array (G, F, B): bag length of (rank, feature-position, bag)
* ``values``   int array: all indices, concatenated in (rank, feature, bag) order
* ``features`` sorted feature ids; feature f reads table f (embedding.py:3-5)
* ``tables``   {table_id: ndarray (rows, dim)} in float64 or float32
* ``shards``   list of (table_id, rank, scheme, (r0, r1), (c0, c1)) in shard-id order

Outputs are float64 like the reference's (embedding.py:72).  Pooling sums run
sequentially in bag order in the table dtype, which is what
``values[list(bag)].sum(axis=0)`` (embedding.py:84) does (pinned by
tests/golden/lookup_order.npz).
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np

__all__ = [
    "OTopo",
    "split_ranges",
    "place_shards",
    "class_order",
    "class_members",
    "peer_order",
    "link_class",
    "uniform_tables",
    "integer_tables",
    "make_bags",
    "kjt_offsets",
    "pool",
    "route_step_a",
    "baseline_forward",
    "tower_forward",
    "realign_cols",
    "init_tm_weights",
    "tm_forward",
    "tm_output_width",
    "tm_flops",
    "bf16_round",
    "byte_totals",
]


# --------------------------------------------------------------------------- #
# topology  (topology.py)
# --------------------------------------------------------------------------- #
@dataclass(frozen=True)
class OTopo:
    """ClusterTopology + TowerLayout in one (topology.py:21-103)."""

    num_hosts: int
    ranks_per_host: int
    hosts_per_tower: int = 1

    @property
    def G(self) -> int:  # topology.py:49-51
        return self.num_hosts * self.ranks_per_host

    @property
    def W(self) -> int:  # group_width, topology.py:91-93
        return self.ranks_per_host * self.hosts_per_tower

    @property
    def T(self) -> int:  # validate_for, topology.py:78-89
        assert self.G % self.W == 0
        return self.G // self.W

    def tower_of_rank(self, r: int) -> int:  # topology.py:95-97
        return r // self.W

    def tower_ranks(self, t: int) -> list[int]:  # topology.py:99-103
        return list(range(t * self.W, (t + 1) * self.W))


def class_order(topo: OTopo) -> list[int]:
    """topology.py:125-137 -- key (g % W, g // W); the order SPTT routes by."""
    return sorted(range(topo.G), key=lambda g: (g % topo.W, g // topo.W))


def class_members(c: int, topo: OTopo) -> list[int]:
    """topology.py:140-145."""
    return [t * topo.W + c for t in range(topo.T)]


def peer_order(topo: OTopo) -> list[int]:
    """topology.py:113-122 -- the paper's literal order (NOT used for routing)."""
    return sorted(range(topo.G), key=lambda g: (g % topo.T, g // topo.ranks_per_host, g))


def link_class(src: int, dst: int, topo: OTopo) -> str:
    """topology.py:148-156."""
    if src == dst:
        return "self"
    if src // topo.ranks_per_host == dst // topo.ranks_per_host:
        return "intra_host"
    return "cross_host"


# --------------------------------------------------------------------------- #
# placement  (embedding.py:88-212)
# --------------------------------------------------------------------------- #
def split_ranges(total: int, parts: int) -> list[tuple[int, int]]:
    """embedding.py:88-103 -- first total % parts ranges take one extra."""
    if parts < 1 or parts > total:
        raise ValueError(f"cannot split {total} into {parts} parts")
    base, extra = divmod(total, parts)
    out, start = [], 0
    for i in range(parts):
        stop = start + base + (1 if i < extra else 0)
        out.append((start, stop))
        start = stop
    return out


def place_shards(table_shapes: dict, plan: dict, topo: OTopo) -> list:
    """embedding.py:174-212 -- round-robin with one cursor per tower, tables by id.

    table_shapes: {tid: (rows, dim)}; plan: {tid: (scheme, num_shards, tower)}.
    """
    cursors = {t: 0 for t in range(topo.T)}
    shards = []
    for tid in sorted(table_shapes):
        rows, dim = table_shapes[tid]
        scheme, count, tower = plan[tid]
        ranks = topo.tower_ranks(tower)
        if scheme == "table_wise":
            pieces = [((0, rows), (0, dim))]
        elif scheme == "column_wise":
            pieces = [((0, rows), cr) for cr in split_ranges(dim, count)]
        else:
            pieces = [(rr, (0, dim)) for rr in split_ranges(rows, count)]
        for rr, cr in pieces:
            rank = ranks[cursors[tower] % len(ranks)]
            cursors[tower] += 1
            shards.append((tid, rank, scheme, rr, cr))
    return shards


# --------------------------------------------------------------------------- #
# inputs  (embedding.py:46-61, 259-295)
# --------------------------------------------------------------------------- #
def uniform_tables(table_shapes: dict, seed: int, dtype=np.float64) -> dict:
    """embedding.py:58-60 -- uniform(-1, 1) from default_rng([seed, table_id])."""
    out = {}
    for tid, (rows, dim) in table_shapes.items():
        rng = np.random.default_rng([seed, tid])
        out[tid] = rng.uniform(-1.0, 1.0, size=(rows, dim)).astype(dtype)
    return out


def integer_tables(table_shapes: dict) -> dict:
    """embedding.py:54-57 -- value(t, r, c) = t*1e6 + r*1e3 + c (float64)."""
    out = {}
    for tid, (rows, dim) in table_shapes.items():
        r = np.arange(rows, dtype=np.float64)[:, None]
        c = np.arange(dim, dtype=np.float64)[None, :]
        out[tid] = tid * 1_000_000.0 + r * 1_000.0 + c
    return out


def make_bags(G: int, table_rows: dict, local_batch: int, hotness: dict, seed: int):
    """embedding.py:259-295 restated to KJT arrays (same rng call sequence).

    Returns (lengths (G, F, B) int32, values int64, pooling {feat: none|sum}).
    """
    rng = np.random.default_rng(seed)
    feats = sorted(table_rows)
    lengths = np.zeros((G, len(feats), local_batch), dtype=np.int32)
    vals = []
    for r in range(G):
        for fi, f in enumerate(feats):
            spec = hotness[f]
            for b in range(local_batch):
                n = 1 if spec == 1 else int(rng.integers(spec[0], spec[1] + 1))
                lengths[r, fi, b] = n
                vals.append(rng.integers(0, table_rows[f], size=n))
    pooling = {f: ("none" if hotness[f] == 1 else "sum") for f in feats}
    values = np.concatenate(vals).astype(np.int64) if vals else np.zeros(0, np.int64)
    return lengths, values, pooling


def kjt_offsets(lengths: np.ndarray) -> np.ndarray:
    """Exclusive prefix sum over the flattened (rank, feature, bag) lengths."""
    flat = np.asarray(lengths, dtype=np.int64).reshape(-1)
    return np.concatenate([[0], np.cumsum(flat)])


def bf16_round(x: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even to bfloat16, returned as float32 (for bf16 paths)."""
    a = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    rounded = (a + 0x7FFF + ((a >> 16) & 1)) & 0xFFFF0000
    return rounded.astype(np.uint32).view(np.float32)


# --------------------------------------------------------------------------- #
# pooled lookup  (embedding.py:64-85, exchange.py:130-146)
# --------------------------------------------------------------------------- #
def pool(values: np.ndarray, lens: np.ndarray, idx: np.ndarray, mode: str,
         acc_dtype=None) -> np.ndarray:
    """Per-bag row select / bag-order sequential sum / mean; empty bag -> 0.

    embedding.py:64-85.  ``mean`` is NOT in the reference (it raises
    DomainError, embedding.py:69-70); here it is sum / len with empty -> 0
    (TorchRec convention) -- parity unpinned.
    """
    lens = np.asarray(lens, dtype=np.int64)
    idx = np.asarray(idx, dtype=np.int64)
    n = lens.shape[0]
    dt = acc_dtype or values.dtype
    out = np.zeros((n, values.shape[1]), dtype=dt)
    if mode == "none":
        if np.any(lens != 1):
            raise ValueError("pooling=none requires bags of length 1")
    if n == 0:
        return out.astype(np.float64)
    if idx.size and (idx.min() < 0 or idx.max() >= values.shape[0]):
        raise IndexError("index out of range")
    starts = np.concatenate([[0], np.cumsum(lens)[:-1]])
    for k in range(int(lens.max(initial=0))):
        sel = lens > k
        out[sel] += values[idx[starts[sel] + k]].astype(dt)
    if mode == "mean":
        nz = lens > 0
        out[nz] = out[nz] / lens[nz, None].astype(dt)
    return out.astype(np.float64)


def _feature_pos(features: Sequence[int]) -> dict:
    return {f: i for i, f in enumerate(features)}


def _bags_of(lengths, values, offsets, rank: int, fpos: int):
    """(lens, idx) of rank's bags for the feature at position fpos."""
    G, F, B = lengths.shape
    base = (rank * F + fpos) * B
    lens = lengths[rank, fpos]
    start, stop = offsets[base], offsets[base + B]
    return lens, values[start:stop]


def _shard_pool(tables, shard, lens, idx, mode):
    """exchange.py:130-146 -- row-wise filters to [r0, r1) and sum-pools."""
    tid, _, scheme, (r0, r1), (c0, c1) = shard
    vals = tables[tid][r0:r1, c0:c1]
    if scheme == "row_wise":
        keep = (idx >= r0) & (idx < r1)
        # per-bag filtered lengths, order preserved
        bag_id = np.repeat(np.arange(len(lens)), lens)
        new_lens = np.bincount(bag_id[keep], minlength=len(lens))
        return pool(vals, new_lens, idx[keep] - r0, "sum"), float(keep.sum() * (c1 - c0))
    return pool(vals, lens, idx, mode), float(np.sum(lens) * (c1 - c0))


def _combine(pieces: list) -> np.ndarray:
    """exchange.py:112-127 -- column shards concat by col range; row shards sum (fp64)."""
    schemes = {p[0][2] for p in pieces}
    if schemes == {"row_wise"}:
        ordered = sorted(pieces, key=lambda p: p[0][3])
        total = ordered[0][1].astype(np.float64).copy()
        for _, mat in ordered[1:]:
            total += mat
        return total
    if "row_wise" in schemes:
        raise ValueError("a table mixes row-wise and column-wise shards")
    ordered = sorted(pieces, key=lambda p: p[0][4])
    return np.concatenate([m for _, m in ordered], axis=1)


# --------------------------------------------------------------------------- #
# step a routing  (exchange.py:162-179)
# --------------------------------------------------------------------------- #
def route_step_a(lengths, values, features, shards, G: int):
    """Per (src, owner): [(sid, lens, idx)] -- the full bag list goes to every
    shard owner of the table (exchange.py:172-178), shards in sid order."""
    offsets = kjt_offsets(lengths)
    fp = _feature_pos(features)
    live = [(sid, s) for sid, s in enumerate(shards) if s[0] in fp]
    out = {}
    for src in range(G):
        for owner in range(G):
            bundle = []
            for sid, s in live:
                if s[1] != owner:
                    continue
                lens, idx = _bags_of(lengths, values, offsets, src, fp[s[0]])
                bundle.append((sid, lens.copy(), idx.copy()))
            out[(src, owner)] = bundle
    return out


def _wire(bytes_map: dict, label: str, src: int, dst: int, n: int):
    bytes_map.setdefault(label, []).append((src, dst, n))


def byte_totals(entries, topo: OTopo):
    """simnet.py:67-77 -- (intra_host, cross_host); self messages never count."""
    intra = cross = 0
    for s, d, n in entries:
        lc = link_class(s, d, topo)
        if lc == "intra_host":
            intra += n
        elif lc == "cross_host":
            cross += n
    return intra, cross


def _lookup_all(lengths, values, features, pooling, tables, shards, G, order):
    """Steps a+b (exchange.py:149-197): blocks[owner][sid] = list of (B, w) in ``order``."""
    routed = route_step_a(lengths, values, features, shards, G)
    wire = {}
    for (src, owner), bundle in routed.items():
        _wire(wire, "a", src, owner, 4 * int(sum(len(i) for _, _, i in bundle)))
    blocks, flops = {}, {o: 0.0 for o in range(G)}
    for owner in range(G):
        per = {sid: [] for sid, s in enumerate(shards) if s[1] == owner and s[0] in pooling}
        for src in order:
            for sid, lens, idx in routed[(src, owner)]:
                mat, fl = _shard_pool(tables, shards[sid], lens, idx, pooling[shards[sid][0]])
                per[sid].append(mat)
                flops[owner] += fl
        blocks[owner] = per
    return blocks, flops, wire


# --------------------------------------------------------------------------- #
# flat baseline  (exchange.py:200-241)
# --------------------------------------------------------------------------- #
def baseline_forward(lengths, values, features, pooling, tables, shards, topo: OTopo):
    """Returns (outputs {rank: (B, sum N)}, layout [(feature, f, N)], wire)."""
    G = topo.G
    blocks, flops, wire = _lookup_all(lengths, values, features, pooling, tables, shards,
                                      G, list(range(G)))
    outputs = {}
    for owner in range(G):
        for dest in range(G):
            n = sum(m[dest].size for m in blocks[owner].values())
            _wire(wire, "c", owner, dest, 4 * n)
    for rank in range(G):
        pieces = {f: [] for f in features}
        for owner in range(G):
            for sid, mats in blocks[owner].items():
                pieces[shards[sid][0]].append((shards[sid], mats[rank]))
        outputs[rank] = np.concatenate([_combine(pieces[f]) for f in features], axis=1)
    layout = [("feature", f, tables[f].shape[1]) for f in features]
    return outputs, layout, wire, {"b": max(flops.values())}


# --------------------------------------------------------------------------- #
# SPTT  (exchange.py:275-462)
# --------------------------------------------------------------------------- #
def tower_forward(lengths, values, features, pooling, tables, shards, assignment: dict,
                  topo: OTopo, tm_cfgs: Optional[dict] = None, tm_weights: Optional[dict] = None,
                  rowwise_rs: bool = False):
    """SPTT a-f.  tm_cfgs {tower: cfg dict or None}; tm_weights {tower: weights}.

    Destination blocks are permuted into CLASS order (exchange.py:319-321) --
    not the paper's peer order.  Output columns are tower-grouped
    (exchange.py:451-460).  swap_bc / omit_permute do not change results
    (exchange.py:324-344), so they are not modelled.
    """
    G, W, T = topo.G, topo.W, topo.T
    tm_cfgs = tm_cfgs or {}
    tm_weights = tm_weights or {}
    dest_seq = [t * W + c for c in range(W) for t in range(T)]
    dest_pos = {r: i for i, r in enumerate(dest_seq)}
    blocks, flops_b, wire = _lookup_all(lengths, values, features, pooling, tables, shards,
                                        G, list(range(G)))
    B = lengths.shape[2]
    by_tower = {t: [f for f in sorted(assignment) if assignment[f] == t and f in pooling]
                for t in range(T)}
    rs_tables = set()
    if rowwise_rs:
        rs_tables = {f for f in features
                     if any(s[2] == "row_wise" for s in shards if s[0] == f)}

    def stacked(owner, sid, cls):  # exchange.py:361-365
        mats = [blocks[owner][sid][dest_pos[p]] for p in class_members(cls, topo)]
        return np.concatenate(mats, axis=0)

    # permute to class order (exchange.py:338-343)
    blocks = {o: {sid: [m[p] for p in dest_seq] for sid, m in per.items()}
              for o, per in blocks.items()}
    dest_pos = {r: i for i, r in enumerate(dest_seq)}

    assembled = {r: {} for r in range(G)}
    for tower in range(T):
        group = topo.tower_ranks(tower)
        feats = by_tower[tower]
        # step d all-to-all (exchange.py:367-378)
        recv = {m: [] for m in group}
        for owner in group:
            for cls, member in enumerate(group):
                bundle = [(sid, stacked(owner, sid, cls)) for sid in blocks[owner]
                          if shards[sid][0] not in rs_tables]
                _wire(wire, "d", owner, member, 4 * sum(m.size for _, m in bundle))
                recv[member].append(bundle)
        # row-wise reduce-scatter (exchange.py:380-395)
        rs_res = {}
        for f in feats:
            if f not in rs_tables:
                continue
            contrib = {}
            for sid, s in enumerate(shards):
                if s[0] != f:
                    continue
                parts = contrib.setdefault(s[1], [None] * W)
                for cls in range(W):
                    piece = stacked(s[1], sid, cls)
                    parts[cls] = piece if parts[cls] is None else parts[cls] + piece
            out = {}
            for j, dst in enumerate(group):
                total = None
                for src in group:
                    if src not in contrib:
                        continue
                    _wire(wire, "d", src, dst, 4 * contrib[src][j].size)
                    total = contrib[src][j].astype(np.float64).copy() if total is None \
                        else total + contrib[src][j]
                out[dst] = total
            rs_res[f] = out
        for member in group:  # exchange.py:397-408
            for f in feats:
                if f in rs_tables:
                    assembled[member][f] = rs_res[f][member]
                else:
                    pieces = [(shards[sid], m) for bundle in recv[member]
                              for sid, m in bundle if shards[sid][0] == f]
                    assembled[member][f] = _combine(pieces)

    # step e (exchange.py:410-437)
    dest_blocks, tm_work, widths = {}, {r: 0.0 for r in range(G)}, {}
    for tower in range(T):
        feats = by_tower[tower]
        cfg = tm_cfgs.get(tower)
        if cfg is not None:
            dims = {tables[f].shape[1] for f in feats}
            if len(dims) > 1:
                raise ValueError("tower mixes embedding dims")
            in_dim = dims.pop() if dims else 1
            widths[tower] = tm_output_width(cfg, len(feats), in_dim)
        else:
            widths[tower] = sum(tables[f].shape[1] for f in feats)
    for rank in range(G):
        tower = topo.tower_of_rank(rank)
        feats = by_tower[tower]
        cfg = tm_cfgs.get(tower)
        per = []
        for j in range(T):
            mats = [assembled[rank][f][j * B:(j + 1) * B] for f in feats]
            if cfg is not None:
                x = np.stack(mats, axis=1) if mats else np.zeros((B, 0, 1))
                per.append(tm_forward(x, cfg, tm_weights[tower]))
                in_dim = x.shape[2]
                tm_work[rank] += tm_flops(cfg, len(feats), in_dim, B)
            elif mats:
                per.append(np.concatenate(mats, axis=1))
            else:
                per.append(np.zeros((B, 0)))
        dest_blocks[rank] = per

    # step f (exchange.py:439-449)
    outputs = {}
    for cls in range(W):
        group = class_members(cls, topo)
        for dst_i, dst in enumerate(group):
            recv = []
            for src in group:
                blk = dest_blocks[src][dst_i]
                _wire(wire, "f", src, dst, 4 * blk.size)
                recv.append(blk)
            outputs[dst] = np.concatenate(recv, axis=1)

    layout = []
    for tower in range(T):
        if tm_cfgs.get(tower) is not None:
            layout.append(("tower", tower, widths[tower]))
        else:
            layout.extend(("feature", f, tables[f].shape[1]) for f in by_tower[tower])
    flops = {"b": max(flops_b.values()), "e": max(tm_work.values())}
    return outputs, layout, wire, flops


def realign_cols(layout, target: Sequence[int]) -> np.ndarray:
    """exchange.py:465-486 as a column gather index; tower blocks are refused."""
    if any(k != "feature" for k, _, _ in layout):
        raise ValueError("layout contains compressed tower blocks")
    starts, col = {}, 0
    widths = {}
    for _, ident, w in layout:
        starts[ident] = col
        widths[ident] = w
        col += w
    if sorted(target) != sorted(widths):
        raise ValueError("target features differ from layout features")
    return np.concatenate([np.arange(starts[f], starts[f] + widths[f]) for f in target]) \
        if target else np.zeros(0, np.int64)


# --------------------------------------------------------------------------- #
# tower modules  (towermod.py)
# --------------------------------------------------------------------------- #
def _uniform(rng, shape, fan_in):
    """towermod.py:69-71."""
    bound = 1.0 / np.sqrt(max(fan_in, 1))
    return rng.uniform(-bound, bound, size=shape)


def init_tm_weights(cfg: dict, num_features: int, in_dim: int, salt: int = 0):
    """towermod.py:74-99 -- same seeding and draw order.  cfg keys: kind, out_dim,
    per_feature_outputs, flat_outputs, cross_layers, seed."""
    rng = np.random.default_rng([cfg["seed"], salt, num_features, in_dim])
    kind = cfg["kind"]
    if kind == "passthrough":
        return None
    D = cfg["out_dim"]
    if kind == "dlrm":
        c, p = cfg["per_feature_outputs"], cfg["flat_outputs"]
        flat_in = num_features * in_dim
        return {
            "w_flat": _uniform(rng, (p * D, flat_in), flat_in),
            "b_flat": _uniform(rng, (p * D,), flat_in),
            "w_feat": _uniform(rng, (c * D, in_dim), in_dim),
            "b_feat": _uniform(rng, (c * D,), in_dim),
        }
    m = num_features * in_dim
    cross = [(_uniform(rng, (m, m), m), _uniform(rng, (m,), m))
             for _ in range(cfg["cross_layers"])]
    return {
        "cross": cross,
        "w_proj": _uniform(rng, (num_features * D, m), m),
        "b_proj": _uniform(rng, (num_features * D,), m),
    }


def tm_output_width(cfg: dict, num_features: int, in_dim: int) -> int:
    """towermod.py:102-107."""
    if cfg["kind"] == "passthrough":
        return num_features * in_dim
    if cfg["kind"] == "dlrm":
        return cfg["out_dim"] * (cfg["per_feature_outputs"] * num_features + cfg["flat_outputs"])
    return num_features * cfg["out_dim"]


def tm_forward(embs: np.ndarray, cfg: dict, w) -> np.ndarray:
    """towermod.py:110-166 (dlrm: [flat proj | per-feature proj]; dcn: cross + proj)."""
    B, F, N = embs.shape
    if cfg["kind"] == "passthrough":
        return embs.reshape(B, -1)
    if cfg["kind"] == "dlrm":
        flat = embs.reshape(B, F * N)
        o1 = flat @ w["w_flat"].T + w["b_flat"]
        o2 = (embs @ w["w_feat"].T + w["b_feat"]).reshape(B, -1)
        return np.concatenate([o1, o2], axis=1)
    x0 = embs.reshape(B, F * N)
    xl = x0
    for cw, cb in w["cross"]:
        xl = x0 * (xl @ cw.T + cb) + xl  # towermod.py:132-139
    return xl @ w["w_proj"].T + w["b_proj"]


def tm_flops(cfg: dict, num_features: int, in_dim: int, batch: int) -> float:
    """towermod.py:194-206."""
    if cfg["kind"] == "passthrough" or num_features == 0:
        return 0.0
    if cfg["kind"] == "dlrm":
        flat = num_features * in_dim
        return 2.0 * batch * (flat * cfg["flat_outputs"] * cfg["out_dim"]
                              + num_features * in_dim * cfg["per_feature_outputs"] * cfg["out_dim"])
    m = num_features * in_dim
    per_layer = 2.0 * batch * m * m + 3.0 * batch * m
    return cfg["cross_layers"] * per_layer + 2.0 * batch * m * num_features * cfg["out_dim"]
