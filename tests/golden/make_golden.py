"""Generate golden fixtures by running the REAL reference (`towersim`) here.

Test infrastructure only.  This script imports the read-only reference from
/root/reference/pkg/src (it exists only in the build container, never on the GPU
box) and freezes its outputs into small .npz/.json fixtures under tests/golden/.
The oracle (oracle/towersim_port.py) is pinned against these fixtures by
tests/test_oracle_golden.py, and the GPU parity tests reuse the same fixtures.

Regenerate with:  python tests/golden/make_golden.py
"""

from __future__ import annotations

import copy
import itertools
import json
import os
import sys

import numpy as np

REF_SRC = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REF_SRC)

import towersim  # noqa: E402
from towersim import exchange as ts_exchange  # noqa: E402
from towersim import simnet as ts_simnet  # noqa: E402
from towersim.cli import RunContext, load_config, random_config  # noqa: E402
from towersim.embedding import (  # noqa: E402
    EmbeddingTable,
    SparseBatch,
    TablePlan,
    init_table_deterministic,
    lookup,
    make_batch,
    shard_tables,
)
from towersim.exchange import ExchangeOptions, TowerPlan, baseline_exchange, realign, tower_exchange  # noqa: E402
from towersim.topology import ClusterTopology, TowerLayout, class_order, peer_order  # noqa: E402
from towersim.towermod import (  # noqa: E402
    TMConfig,
    init_tm_weights,
    tm_flops,
    tm_forward,
    tm_output_width,
    tm_weight_jvp,
)

FLAG_COMBOS = list(itertools.product([False, True], repeat=3))


# --------------------------------------------------------------------------- #
# helpers: batch <-> KJT arrays, trace -> byte table, layout -> list
# --------------------------------------------------------------------------- #
def batch_to_kjt(batch: SparseBatch):
    """lengths (G, F, B) int32 and values flat int64 in (rank, feature, bag) order."""
    feats = batch.features
    G, B = batch.num_ranks, batch.local_batch
    lengths = np.zeros((G, len(feats), B), dtype=np.int32)
    vals = []
    for r in range(G):
        for fi, f in enumerate(feats):
            for b, bag in enumerate(batch.bags[r][f]):
                lengths[r, fi, b] = len(bag)
                vals.extend(bag)
    return lengths, np.asarray(vals, dtype=np.int64)


def trace_table(trace) -> dict:
    out = {}
    for label in trace.labels():
        intra, cross = trace.byte_totals(label)
        out[label] = [int(intra), int(cross)]
        out[label + "_sent"] = {str(k): int(v) for k, v in trace.sent_by_rank(label).items()}
    return out


def layout_list(layout) -> list:
    return [[k, int(i), int(w)] for k, i, w in layout.blocks]


def placement_list(placement) -> list:
    return [
        [s.table_id, s.rank, s.scheme, list(s.row_range), list(s.col_range)]
        for s in placement.shards
    ]


def capture_step_a(fn, *args, **kwargs):
    """Run fn while recording every step-a payload (src, owner, [(sid, bags)])."""
    captured = []
    real = ts_exchange.all_to_all

    def spy(group, sends, label, trace):
        if label == "a":
            for src in group:
                for j, dst in enumerate(group):
                    captured.append(
                        (src, dst, [(t.tag, [list(b) for b in t.data]) for t in sends[src][j]])
                    )
        return real(group, sends, label, trace)

    ts_exchange.all_to_all = spy
    try:
        res = fn(*args, **kwargs)
    finally:
        ts_exchange.all_to_all = real
    return res, captured


# --------------------------------------------------------------------------- #
# 1. the acceptance sweep (tests/test_acceptance.py:46-81): seed 2024, flags
# --------------------------------------------------------------------------- #
def gen_acceptance(n_configs: int = 60, real_values: bool = False):
    """``real_values``: the same configs with U(-1, 1) float64 tables (the
    reference's own non-integer mode) instead of integer-valued ones, so sums
    of row-wise partials exercise the reference's summation order bit for bit."""
    rng = np.random.default_rng(2024)
    meta, arrays = [], {}
    for i in range(n_configs):
        cfg = random_config(rng)
        if real_values:
            cfg["tables"]["integer_values"] = False
        swap, omit, rs = FLAG_COMBOS[i % len(FLAG_COMBOS)]
        cfg["exchange"] = {"swap_bc": swap, "omit_permute": omit, "rowwise_reducescatter": rs}
        ctx = RunContext(cfg)
        base = ctx.run_baseline()
        tower = ctx.run_tower()
        target = [ident for _, ident, _ in base.layout.blocks]
        realigned = realign(tower, target)
        lengths, values = batch_to_kjt(ctx.batch)
        G = ctx.topo.world_size
        arrays[f"c{i}_lengths"] = lengths
        arrays[f"c{i}_values"] = values
        arrays[f"c{i}_base"] = np.stack([base.outputs[r] for r in range(G)])
        arrays[f"c{i}_tower"] = np.stack([tower.outputs[r] for r in range(G)])
        arrays[f"c{i}_realigned"] = np.stack([realigned.outputs[r] for r in range(G)])
        meta.append(
            {
                "index": i,
                "cfg": cfg,
                "world": G,
                "num_hosts": ctx.topo.num_hosts,
                "ranks_per_host": ctx.topo.ranks_per_host,
                "num_towers": ctx.layout.num_towers,
                "hosts_per_tower": ctx.layout.hosts_per_tower,
                "assignment": {str(k): int(v) for k, v in ctx.assignment.items()},
                "pooling": {str(k): v for k, v in ctx.batch.pooling.items()},
                "local_batch": ctx.batch.local_batch,
                "placement": placement_list(ctx.placement),
                "table_seed": int(cfg["seed"]) * 1_000_003 + 1,
                "base_layout": layout_list(base.layout),
                "tower_layout": layout_list(tower.layout),
                "base_trace": trace_table(base.trace),
                "tower_trace": trace_table(tower.trace),
                "flops": {k: float(v) for k, v in tower.flops.items()},
                "base_flops": {k: float(v) for k, v in base.flops.items()},
            }
        )
    return meta, arrays


# --------------------------------------------------------------------------- #
# 1b. full-size C1: 2 x 4, F = 26, N = 64, B = 512 / rank, 100k
# rows, float64 U(-1, 1) tables; single- and multi-hot.  The outputs are ~55 MB
# per case, so the fixture keeps per-rank SHA-256 digests of the exact float64
# bytes (plus the batch digest and a few rows) -- bit-exact checks at full size.
# --------------------------------------------------------------------------- #
def _sha(a: np.ndarray) -> str:
    import hashlib

    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def gen_c1_full():
    out = {}
    topo = ClusterTopology(2, 4)
    layout = TowerLayout(2)
    tables = {t: init_table_deterministic(t, 100_000, 64, seed=0) for t in range(26)}
    assignment = {t: (0 if t < 13 else 1) for t in range(26)}
    placement = shard_tables(tables, {t: TablePlan("table_wise", 1, assignment[t]) for t in tables}, topo, layout)
    tp = TowerPlan(layout, assignment)
    for name, hot in (("single_hot", 1), ("multi_hot", (10, 30))):
        batch = make_batch(topo, tables, 512, {t: hot for t in tables}, seed=1)
        tower = tower_exchange(batch, placement, tp, topo)
        base = baseline_exchange(batch, placement, topo)
        lengths, values = batch_to_kjt(batch)
        out[name] = {
            "hot": hot if hot == 1 else list(hot),
            "lengths_sha": _sha(lengths.astype(np.int32)),
            "values_sha": _sha(values.astype(np.int64)),
            "nnz": int(values.size),
            "tower_sha": {str(r): _sha(tower.outputs[r]) for r in range(8)},
            "base_sha": {str(r): _sha(base.outputs[r]) for r in range(8)},
            "tower_rows0_3": {str(r): tower.outputs[r][:4].tolist() for r in (0, 5)},
            "tower_layout": layout_list(tower.layout),
            "tower_trace": trace_table(tower.trace),
            "base_trace": trace_table(base.trace),
        }
    return out


# --------------------------------------------------------------------------- #
# 2. Appendix-A worked 2x4 example with step-a capture
# --------------------------------------------------------------------------- #
def gen_worked_2x4():
    topo = ClusterTopology(2, 4)
    layout = TowerLayout(2)
    tables = {t: init_table_deterministic(t, 8, 2, integer=True) for t in range(6)}
    assignment = {0: 0, 1: 0, 2: 0, 3: 1, 4: 1, 5: 1}
    plan = {t: TablePlan("table_wise", 1, assignment[t]) for t in tables}
    placement = shard_tables(tables, plan, topo, layout)
    batch = make_batch(topo, tables, 1, {t: 1 for t in tables}, seed=1)
    tp = TowerPlan(layout, assignment)
    tower, cap = capture_step_a(tower_exchange, batch, placement, tp, topo, ExchangeOptions())
    base = baseline_exchange(batch, placement, topo)
    lengths, values = batch_to_kjt(batch)
    meta = {
        "placement": placement_list(placement),
        "class_order": list(class_order(topo, layout)),
        "peer_order": list(peer_order(topo, layout)),
        "assignment": {str(k): v for k, v in assignment.items()},
        "step_a": [[s, d, [[int(sid), bags] for sid, bags in bundle]] for s, d, bundle in cap],
        "tower_layout": layout_list(tower.layout),
        "tower_trace": trace_table(tower.trace),
        "base_trace": trace_table(base.trace),
    }
    arrays = {
        "lengths": lengths,
        "values": values,
        "tower": np.stack([tower.outputs[r] for r in range(8)]),
        "base": np.stack([base.outputs[r] for r in range(8)]),
    }
    return meta, arrays


# --------------------------------------------------------------------------- #
# 3. float32 tables (bit-exact fp32 pooling) at a reduced C1 shape, all schemes
# --------------------------------------------------------------------------- #
def fp32_tables(num, rows, dim, seed):
    out = {}
    for t in range(num):
        rng = np.random.default_rng([seed, t])
        out[t] = EmbeddingTable(t, rows, dim, rng.uniform(-1, 1, (rows, dim)).astype(np.float32))
    return out


def _compact(x: np.ndarray) -> np.ndarray:
    """Store as float32 when that is lossless (fp32-table sums are fp32-exact)."""
    x32 = x.astype(np.float32)
    return x32 if np.array_equal(x32.astype(np.float64), x) else x


def gen_fp32_c1(scheme: str, shards: int, hot, local_batch=16, rows=1000, dim=32, tm=None,
                keep_base=False):
    topo = ClusterTopology(2, 4)
    layout = TowerLayout(2)
    tables = fp32_tables(26, rows, dim, seed=0)
    assignment = {t: (0 if t < 13 else 1) for t in range(26)}
    plan = {
        t: TablePlan(scheme, 1 if scheme == "table_wise" else shards, assignment[t])
        for t in tables
    }
    placement = shard_tables(tables, plan, topo, layout)
    batch = make_batch(topo, tables, local_batch, {t: hot for t in tables}, seed=1)
    tp = TowerPlan(layout, assignment)
    opts = ExchangeOptions(tower_modules=tm)
    tower = tower_exchange(batch, placement, tp, topo, opts)
    base = baseline_exchange(batch, placement, topo)
    lengths, values = batch_to_kjt(batch)
    meta = {
        "scheme": scheme,
        "shards": shards,
        "hot": hot,
        "local_batch": local_batch,
        "rows": rows,
        "dim": dim,
        "placement": placement_list(placement),
        "pooling": {str(k): v for k, v in batch.pooling.items()},
        "tower_layout": layout_list(tower.layout),
        "tower_trace": trace_table(tower.trace),
        "base_trace": trace_table(base.trace),
        "flops": {k: float(v) for k, v in tower.flops.items()},
    }
    arrays = {
        "lengths": lengths,
        "values": values,
        "tower": _compact(np.stack([tower.outputs[r] for r in range(8)])),
    }
    if keep_base:
        arrays["base"] = _compact(np.stack([base.outputs[r] for r in range(8)]))
    if tm is not None:
        meta["tm"] = {
            "kind": tm.kind,
            "out_dim": tm.out_dim,
            "per_feature_outputs": tm.per_feature_outputs,
            "flat_outputs": tm.flat_outputs,
            "cross_layers": tm.cross_layers,
            "seed": tm.seed,
        }
    return meta, arrays


# --------------------------------------------------------------------------- #
# 4. lookup sum-order pin: long bags on an fp32 table
# --------------------------------------------------------------------------- #
def gen_lookup_order():
    rng = np.random.default_rng(7)
    table = rng.uniform(-1, 1, (1024, 32)).astype(np.float32)
    lens = rng.integers(0, 201, size=64)
    bags = [[int(i) for i in rng.integers(0, 1024, size=int(n))] for n in lens]
    out = lookup(table, bags, "sum")
    offsets = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    values = np.asarray([i for b in bags for i in b], dtype=np.int64)
    return {"table": table, "offsets": offsets, "values": values, "out": out}


# --------------------------------------------------------------------------- #
# 5. tower-module numerics: forward, width, flops, weight JVP (backward pin)
# --------------------------------------------------------------------------- #
TM_CASES = [
    ("dlrm", dict(out_dim=4, per_feature_outputs=1, flat_outputs=0), 3, 8),
    ("dlrm", dict(out_dim=3, per_feature_outputs=2, flat_outputs=1), 4, 6),
    ("dlrm", dict(out_dim=16, per_feature_outputs=1, flat_outputs=2), 5, 32),
    ("dcn", dict(out_dim=4, cross_layers=1), 2, 8),
    ("dcn", dict(out_dim=3, cross_layers=2), 3, 4),
    ("dcn", dict(out_dim=8, cross_layers=3), 4, 16),
]


def gen_tm():
    meta, arrays = [], {}
    rng = np.random.default_rng(31)
    for i, (kind, kw, F, N) in enumerate(TM_CASES):
        cfg = TMConfig(kind=kind, seed=i, **kw)
        salt = 5 + i
        w = init_tm_weights(cfg, F, N, salt=salt)
        d = init_tm_weights(cfg, F, N, salt=salt + 100)
        embs = rng.normal(size=(7, F, N))
        out = tm_forward(embs, cfg, w)
        jvp = tm_weight_jvp(embs, cfg, w, d)
        arrays[f"t{i}_embs"] = embs
        arrays[f"t{i}_out"] = out
        arrays[f"t{i}_jvp"] = jvp
        if kind == "dlrm":
            for name in ("w_flat", "b_flat", "w_feat", "b_feat"):
                arrays[f"t{i}_w_{name}"] = getattr(w, name)
                arrays[f"t{i}_d_{name}"] = getattr(d, name)
        else:
            for l, ((cw, cb), (dw, db)) in enumerate(zip(w.cross, d.cross)):
                arrays[f"t{i}_w_cross{l}_w"] = cw
                arrays[f"t{i}_w_cross{l}_b"] = cb
                arrays[f"t{i}_d_cross{l}_w"] = dw
                arrays[f"t{i}_d_cross{l}_b"] = db
            arrays[f"t{i}_w_w_proj"] = w.w_proj
            arrays[f"t{i}_w_b_proj"] = w.b_proj
            arrays[f"t{i}_d_w_proj"] = d.w_proj
            arrays[f"t{i}_d_b_proj"] = d.b_proj
        meta.append(
            {
                "index": i,
                "kind": kind,
                "kw": kw,
                "seed": i,
                "salt": salt,
                "F": F,
                "N": N,
                "width": tm_output_width(cfg, F, N),
                "flops_b7": tm_flops(cfg, F, N, 7),
            }
        )
    return meta, arrays


def main():
    meta = {}
    acc_meta, acc_arr = gen_acceptance()
    meta["acceptance"] = acc_meta
    np.savez_compressed(os.path.join(HERE, "acceptance.npz"), **acc_arr)

    # 200 configs of the acceptance sweep with real-valued tables
    ar_meta, ar_arr = gen_acceptance(200, real_values=True)
    meta["acceptance_real"] = ar_meta
    np.savez_compressed(os.path.join(HERE, "acceptance_real.npz"), **ar_arr)

    meta["c1_full"] = gen_c1_full()

    w_meta, w_arr = gen_worked_2x4()
    meta["worked_2x4"] = w_meta
    np.savez_compressed(os.path.join(HERE, "worked_2x4.npz"), **w_arr)

    fp32 = {}
    cases = [
        ("tw_single", "table_wise", 1, 1, None),
        ("tw_multi", "table_wise", 1, (10, 30), None),
        ("cw_multi", "column_wise", 2, (0, 6), None),
        ("rw_multi", "row_wise", 3, (0, 6), None),
        ("tw_dlrm", "table_wise", 1, (1, 4), TMConfig(kind="dlrm", out_dim=8, seed=3)),
        ("tw_dcn", "table_wise", 1, (1, 4), TMConfig(kind="dcn", out_dim=8, cross_layers=2, seed=3)),
    ]
    fp32_meta = {}
    for name, scheme, shards, hot, tm in cases:
        m, a = gen_fp32_c1(scheme, shards, hot, tm=tm, dim=16 if tm is not None else 32,
                           local_batch=8 if tm is not None else 16,
                           keep_base=(name == "tw_single"))
        fp32_meta[name] = m
        for k, v in a.items():
            fp32[f"{name}_{k}"] = v
    meta["fp32_c1"] = fp32_meta
    np.savez_compressed(os.path.join(HERE, "fp32_c1.npz"), **fp32)

    np.savez_compressed(os.path.join(HERE, "lookup_order.npz"), **gen_lookup_order())

    tm_meta, tm_arr = gen_tm()
    meta["tm"] = tm_meta
    np.savez_compressed(os.path.join(HERE, "tm.npz"), **tm_arr)

    meta["generator"] = {
        "reference": "towersim " + towersim.__version__ + " from /root/reference/pkg/src",
        "numpy": np.__version__,
    }
    with open(os.path.join(HERE, "golden.json"), "w", encoding="utf-8") as fh:
        json.dump(meta, fh, indent=1, sort_keys=True)
    print("wrote golden fixtures to", HERE)


if __name__ == "__main__":
    main()
