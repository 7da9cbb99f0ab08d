"""Pin the numpy oracle against fixtures produced by the real reference.

CPU only.  If these pass, the oracle reproduces towersim bit for bit on the
reference's own acceptance configs (tests/test_acceptance.py:46-81 in the
reference), the Appendix-A worked example, fp32 tables at a reduced C1 shape,
long-bag pooling order and the tower-module numerics.
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import acceptance_case, fp32_case, golden_meta, golden_npz, tm_case
from oracle import (
    OTopo,
    baseline_forward,
    byte_totals,
    class_order,
    init_tm_weights,
    peer_order,
    place_shards,
    pool,
    realign_cols,
    route_step_a,
    tm_backward,
    tm_flops,
    tm_forward,
    tm_output_width,
    tower_forward,
)

N_ACC = len(golden_meta()["acceptance"])
N_ACC_REAL = len(golden_meta()["acceptance_real"])


def _tm_cfg_from(m):
    t = m["cfg"]["tm"]
    if t["kind"] == "passthrough":
        return None
    return {"kind": t["kind"], "out_dim": t["out_dim"], "per_feature_outputs": t["per_feature_outputs"],
            "flat_outputs": t["flat_outputs"], "cross_layers": t["cross_layers"], "seed": t["seed"]}


@pytest.mark.parametrize("key,i", [("acceptance", i) for i in range(N_ACC)] +
                         [("acceptance_real", i) for i in range(N_ACC_REAL)])
def test_acceptance_config_bit_exact(key, i):
    """Integer-valued tables (60 configs) and the 200-config sweep with
    real-valued float64 tables, where every sum -- bag order, row-range order,
    the reduce-scatter's per-owner then group order -- must match bit for bit."""
    c = acceptance_case(i, key)
    topo = c["topo"]
    base, blayout, bwire, bflops = baseline_forward(
        c["lengths"], c["values"], c["features"], c["pooling"], c["tables"], c["shards"], topo)
    tower, tlayout, twire, tflops = tower_forward(
        c["lengths"], c["values"], c["features"], c["pooling"], c["tables"], c["shards"],
        c["assignment"], topo, rowwise_rs=c["exchange"]["rowwise_reducescatter"])
    for r in range(topo.G):
        assert np.array_equal(base[r], c["base"][r])
        assert np.array_equal(tower[r], c["tower"][r])
    cols = realign_cols(tlayout, [f for _, f, _ in blayout])
    for r in range(topo.G):
        assert np.array_equal(tower[r][:, cols], c["realigned"][r])
    m = c["meta"]
    assert [list(x) for x in tlayout] == m["tower_layout"]
    assert [list(x) for x in blayout] == m["base_layout"]
    for label, entries in bwire.items():
        assert list(byte_totals(entries, topo)) == m["base_trace"][label]
    for label, entries in twire.items():
        assert list(byte_totals(entries, topo)) == m["tower_trace"][label], label
    assert tflops["b"] == m["flops"]["b"]


def test_acceptance_placement_matches():
    for i in range(N_ACC):
        c = acceptance_case(i)
        m = c["meta"]
        t = m["cfg"]["tables"]
        shapes = {tid: (int(t["rows"]), int(t["dim"])) for tid in range(int(t["count"]))}
        scheme = t["sharding"]
        W = c["topo"].W
        plan = {}
        for tid in shapes:
            count = 1 if scheme == "table_wise" else min(
                int(t["shards_per_table"]), shapes[tid][1] if scheme == "column_wise" else shapes[tid][0], W)
            plan[tid] = (scheme, count, c["assignment"][tid])
        assert place_shards(shapes, plan, c["topo"]) == c["shards"]


def test_worked_2x4_example():
    m = golden_meta()["worked_2x4"]
    arr = golden_npz("worked_2x4")
    topo = OTopo(2, 4)
    assert class_order(topo) == m["class_order"] == [0, 4, 1, 5, 2, 6, 3, 7]
    assert peer_order(topo) == m["peer_order"] == [0, 2, 4, 6, 1, 3, 5, 7]
    from oracle import integer_tables

    tables = integer_tables({t: (8, 2) for t in range(6)})
    shards = [(a, b, c, tuple(d), tuple(e)) for a, b, c, d, e in m["placement"]]
    assert {s[0]: s[1] for s in shards} == {0: 0, 1: 1, 2: 2, 3: 4, 4: 5, 5: 6}
    assignment = {int(k): v for k, v in m["assignment"].items()}
    routed = route_step_a(arr["lengths"], arr["values"], list(range(6)), shards, 8)
    for src, dst, bundle in m["step_a"]:
        mine = routed[(src, dst)]
        assert [sid for sid, _, _ in mine] == [sid for sid, _ in bundle]
        for (sid, lens, idx), (_, bags) in zip(mine, bundle):
            assert list(lens) == [len(b) for b in bags]
            assert list(idx) == [i for b in bags for i in b]
    pooling = {f: "none" for f in range(6)}
    tower, layout, _, _ = tower_forward(arr["lengths"], arr["values"], list(range(6)), pooling,
                                        tables, shards, assignment, topo)
    for r in range(8):
        assert np.array_equal(tower[r], arr["tower"][r])
    # rank 5's output
    assert list(arr["tower"][5][0]) == [0, 1, 1003000, 1003001, 2007000, 2007001, 3001000,
                                        3001001, 4003000, 4003001, 5003000, 5003001]


@pytest.mark.parametrize("name", ["tw_single", "tw_multi", "cw_multi", "rw_multi", "tw_dlrm", "tw_dcn"])
def test_fp32_reduced_c1(name):
    c = fp32_case(name)
    m = c["meta"]
    tm_cfgs, tm_w = None, None
    if "tm" in m:
        cfg = dict(m["tm"])
        dims = m["dim"]
        tm_cfgs = {t: cfg for t in range(2)}
        tm_w = {t: init_tm_weights(cfg, 13, dims, salt=t) for t in range(2)}
    tower, layout, wire, flops = tower_forward(
        c["lengths"], c["values"], c["features"], c["pooling"], c["tables"], c["shards"],
        c["assignment"], c["topo"], tm_cfgs, tm_w)
    for r in range(8):
        if "tm" in m:
            np.testing.assert_allclose(tower[r], c["tower"][r], rtol=1e-12, atol=1e-12)
        else:
            assert np.array_equal(tower[r], c["tower"][r])
    assert [list(x) for x in layout] == m["tower_layout"]
    if "base" in c:
        base, _, _, _ = baseline_forward(c["lengths"], c["values"], c["features"], c["pooling"],
                                         c["tables"], c["shards"], c["topo"])
        for r in range(8):
            assert np.array_equal(base[r], c["base"][r])


def test_lookup_sequential_bag_order_fp32():
    g = golden_npz("lookup_order")
    lens = np.diff(g["offsets"])
    out = pool(g["table"], lens, g["values"], "sum")
    assert np.array_equal(out, g["out"])
    # pairwise / reordered summation would NOT match: sanity that the pin bites
    alt = np.zeros_like(out)
    for b in range(len(lens)):
        rows = g["table"][g["values"][g["offsets"][b]:g["offsets"][b + 1]]].astype(np.float64)
        alt[b] = rows.sum(axis=0).astype(np.float32)
    assert not np.array_equal(alt, out)


@pytest.mark.parametrize("i", range(len(golden_meta()["tm"])))
def test_tm_forward_width_flops(i):
    cfg, w, d, embs, out, jvp, m = tm_case(i)
    w2 = init_tm_weights(cfg, m["F"], m["N"], salt=m["salt"])
    if cfg["kind"] == "dlrm":
        for k in w:
            assert np.array_equal(w2[k], w[k])
    else:
        for (a, b), (c2, d2) in zip(w["cross"], w2["cross"]):
            assert np.array_equal(a, c2) and np.array_equal(b, d2)
        assert np.array_equal(w2["w_proj"], w["w_proj"])
    mine = tm_forward(embs, cfg, w)
    np.testing.assert_allclose(mine, out, rtol=1e-13, atol=1e-13)
    assert tm_output_width(cfg, m["F"], m["N"]) == m["width"]
    assert tm_flops(cfg, m["F"], m["N"], 7) == m["flops_b7"]


def _inner(dw, d, kind):
    if kind == "dlrm":
        return sum(float(np.sum(dw[k] * d[k])) for k in ("w_flat", "b_flat", "w_feat", "b_feat"))
    s = float(np.sum(dw["w_proj"] * d["w_proj"]) + np.sum(dw["b_proj"] * d["b_proj"]))
    for (gw, gb), (dw_, db_) in zip(dw["cross"], d["cross"]):
        s += float(np.sum(gw * dw_) + np.sum(gb * db_))
    return s


@pytest.mark.parametrize("i", range(len(golden_meta()["tm"])))
def test_tm_weight_grads_adjoint_of_reference_jvp(i):
    """<g, J d> (reference tm_weight_jvp) == <J^T g, d> (oracle backward)."""
    cfg, w, d, embs, out, jvp, m = tm_case(i)
    rng = np.random.default_rng(100 + i)
    g = rng.normal(size=out.shape)
    _, dw = tm_backward(embs, cfg, w, g)
    lhs = float(np.sum(g * jvp))
    rhs = _inner(dw, d, cfg["kind"])
    assert abs(lhs - rhs) <= 1e-10 * max(1.0, abs(lhs))


@pytest.mark.parametrize("i", range(len(golden_meta()["tm"])))
def test_tm_input_grads_finite_difference(i):
    cfg, w, d, embs, out, jvp, m = tm_case(i)
    rng = np.random.default_rng(200 + i)
    g = rng.normal(size=out.shape)
    dx, _ = tm_backward(embs, cfg, w, g)
    v = rng.normal(size=embs.shape)
    eps = 1e-6
    fd = (np.sum(g * tm_forward(embs + eps * v, cfg, w))
          - np.sum(g * tm_forward(embs - eps * v, cfg, w))) / (2 * eps)
    assert abs(fd - np.sum(dx * v)) <= 1e-6 * max(1.0, abs(fd))


def test_acceptance_real_sweep_covers_rowwise_reducescatter():
    """The real-valued sweep reaches the orders that integer tables cannot
    distinguish: row-wise shards with and without the reduce-scatter form."""
    ms = golden_meta()["acceptance_real"]
    rw = [m for m in ms if m["cfg"]["tables"]["sharding"] == "row_wise"]
    assert any(m["cfg"]["exchange"]["rowwise_reducescatter"] for m in rw)
    assert any(not m["cfg"]["exchange"]["rowwise_reducescatter"] for m in rw)
    assert not any(m["cfg"]["tables"]["integer_values"] for m in ms)


@pytest.mark.parametrize("multi", [False, True])
def test_c1_full_size_oracle_digests(multi):
    """Full-size C1 (2 x 4, F = 26, N = 64, B = 512, 100k rows): the oracle's
    float64 outputs hash to the reference's (SHA-256 of the exact bytes)."""
    import paper_2403_00877_b200 as TS
    from conftest import c1_full_inputs, sha256
    from oracle import OTopo

    m = golden_meta()["c1_full"]["multi_hot" if multi else "single_hot"]
    topo, placement, batch, plan, tables = c1_full_inputs(TS, multi)
    G, F, B = 8, 26, 512
    lengths = np.zeros((G, F, B), dtype=np.int32)
    vals = []
    for r in range(G):
        for f in range(F):
            for b, bag in enumerate(batch.bags[r][f]):
                lengths[r, f, b] = len(bag)
                vals.extend(bag)
    values = np.asarray(vals, dtype=np.int64)
    assert sha256(lengths) == m["lengths_sha"] and sha256(values) == m["values_sha"]
    shards = [(s.table_id, s.rank, s.scheme, s.row_range, s.col_range) for s in placement.shards]
    tvals = {t: tables[t].values for t in tables}
    pooling = dict(batch.pooling)
    tower, tlayout, twire, _ = tower_forward(lengths, values, list(range(F)), pooling, tvals, shards,
                                             {t: (0 if t < 13 else 1) for t in range(F)}, OTopo(2, 4))
    base, _, _, _ = baseline_forward(lengths, values, list(range(F)), pooling, tvals, shards, OTopo(2, 4))
    for r in range(G):
        assert sha256(tower[r]) == m["tower_sha"][str(r)], r
        assert sha256(base[r]) == m["base_sha"][str(r)], r
    for label, entries in twire.items():
        assert list(byte_totals(entries, OTopo(2, 4))) == m["tower_trace"][label], label
