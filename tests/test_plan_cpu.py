"""CPU tests of the host-side routing plan and reference-mirror logic (no GPU).

The numpy emulation (tests/plan_emulation.py) moves data exactly as the plan
says; its outputs must equal the oracle's (and so the reference's) on every
golden acceptance config.  Plus unit checks of topology / placement / byte
accounting against the reference's own KATs.
"""

from __future__ import annotations

import numpy as np
import pytest

import paper_2403_00877_b200 as P
from conftest import acceptance_case, fp32_case, golden_meta
from paper_2403_00877_b200.plan import ExchangePlan
from plan_emulation import emulate_flat, emulate_sptt

N_ACC = len(golden_meta()["acceptance"])


def _plan(c, sptt=True):
    topo = P.ClusterTopology(c["topo"].num_hosts, c["topo"].ranks_per_host)
    layout = P.TowerLayout(c["topo"].T, c["topo"].hosts_per_tower)
    shards = [P.Shard(a, b, s, tuple(r), tuple(cc)) for a, b, s, r, cc in c["shards"]]
    dims = {f: c["tables"][f].shape[1] for f in c["features"]}
    if sptt:
        return ExchangePlan(topo, layout, shards, c["features"], dims, c["pooling"], c["lengths"].shape[2],
                            feature_towers=c["assignment"])
    return ExchangePlan(topo, P.TowerLayout(1, topo.num_hosts), shards, c["features"], dims, c["pooling"],
                        c["lengths"].shape[2])


@pytest.mark.parametrize("i", range(N_ACC))
def test_plan_emulation_reproduces_reference(i):
    c = acceptance_case(i)
    plan = _plan(c)
    out = emulate_sptt(plan, c["tables"], c["lengths"], c["values"])
    for r in range(plan.G):
        assert np.array_equal(out[r], c["tower"][r])
    flat = emulate_flat(_plan(c, sptt=False), c["tables"], c["lengths"], c["values"])
    for r in range(plan.G):
        assert np.array_equal(flat[r], c["base"][r])
    # layout blocks match the reference (pass-through)
    assert [list(b) for b in plan.tower_layout_blocks({})] == c["meta"]["tower_layout"]


@pytest.mark.parametrize("name", ["cw_multi", "rw_multi", "tw_single"])
def test_plan_emulation_fp32_cases(name):
    c = fp32_case(name)
    plan = _plan(c)
    out = emulate_sptt(plan, c["tables"], c["lengths"], c["values"])
    for r in range(8):
        np.testing.assert_allclose(out[r], c["tower"][r], rtol=1e-7, atol=1e-7)


def test_wire_bytes_formulas_c1():
    """SURVEY §0 fact 7 at C1 (2x4, F=26, N=64, B=512, fp32): flat c 7/8*BFNs,
    SPTT d 3/4*BFNs per rank."""
    topo = P.ClusterTopology(2, 4)
    layout = P.TowerLayout(2)
    feats = list(range(26))
    assignment = {f: (0 if f < 13 else 1) for f in feats}
    tables = {f: P.EmbeddingTable(f, 8, 64, np.zeros((8, 64))) for f in feats}
    placement = P.shard_tables(tables, {f: P.TablePlan("table_wise", 1, assignment[f]) for f in feats}, topo,
                               layout)
    plan = ExchangePlan(topo, layout, placement.shards, feats, {f: 64 for f in feats}, {f: "none" for f in feats},
                        512, feature_towers=assignment)
    B, F, N, s = 512, 26, 64, 4
    # per-rank maxima (shards are dealt unevenly: 4/3/3/3 tables per rank)
    assert plan.bytes_per_rank(s)["f"] == (2 - 1) * B * 13 * N * s
    # totals over all ranks equal the reference trace totals
    tot_d = sum(sum(plan.T * B * plan.SW[r] for m in plan.group_of(r) if m != r) for r in range(8)) * s
    assert tot_d == 20_447_232
    flat = ExchangePlan(topo, P.TowerLayout(1, 2), placement.shards, feats, {f: 64 for f in feats},
                        {f: "none" for f in feats}, 512)
    tot_c = sum(sum(B * flat.SW[r] for p in range(8) if p != r) for r in range(8)) * s
    assert tot_c == 10_223_616 + 13_631_488
    tot_f = sum((plan.T - 1) * B * plan.O[plan.tower_of(r)] for r in range(8)) * s
    assert tot_f == 13_631_488


def test_topology_kats():
    topo = P.ClusterTopology(2, 4)
    layout = P.TowerLayout(2)
    assert P.class_order(topo, layout) == (0, 4, 1, 5, 2, 6, 3, 7)
    assert P.peer_order(topo, layout) == (0, 2, 4, 6, 1, 3, 5, 7)
    assert P.peer_order(P.ClusterTopology(2, 2), P.TowerLayout(2)) == (0, 2, 1, 3)
    assert P.class_members(1, topo, layout) == [1, 5]
    assert P.link_class(0, 1, P.ClusterTopology(2, 2)) == "intra_host"
    assert P.link_class(0, 2, P.ClusterTopology(2, 2)) == "cross_host"
    assert P.peers(5, P.ClusterTopology(2, 4)) == {1, 5}
    with pytest.raises(P.DomainError):
        P.TowerLayout(3).validate_for(topo)


def test_placement_kats():
    assert P.split_ranges(10, 3) == [(0, 4), (4, 7), (7, 10)]
    with pytest.raises(P.DomainError):
        P.split_ranges(2, 3)
    topo = P.ClusterTopology(2, 4)
    layout = P.TowerLayout(2)
    tables = {t: P.init_table_deterministic(t, 8, 2, integer=True) for t in range(6)}
    assignment = {0: 0, 1: 0, 2: 0, 3: 1, 4: 1, 5: 1}
    pl = P.shard_tables(tables, {t: P.TablePlan("table_wise", 1, assignment[t]) for t in range(6)}, topo, layout)
    assert {s.table_id: s.rank for s in pl.shards} == {0: 0, 1: 1, 2: 2, 3: 4, 4: 5, 5: 6}
    with pytest.raises(P.PlanError):
        P.shard_tables(tables, {0: P.TablePlan("table_wise", 1, 5)}, topo, layout)
    t0 = P.init_table_deterministic(0, 4, 4, integer=True)
    assert t0.values[1, 2] == 1002.0


def test_plan_errors_match_reference():
    topo = P.ClusterTopology(2, 2)
    layout = P.TowerLayout(2)
    tables = {t: P.init_table_deterministic(t, 8, 3, integer=True) for t in range(4)}
    assignment = {t: t // 2 for t in range(4)}
    pl = P.shard_tables(tables, {t: P.TablePlan("table_wise", 1, assignment[t]) for t in range(4)}, topo, layout)
    with pytest.raises(P.PlanError):
        ExchangePlan(topo, layout, pl.shards, [0, 1, 2, 3], {t: 3 for t in range(4)}, {t: "none" for t in range(4)},
                     2, feature_towers={**assignment, 0: 1})
    with pytest.raises(P.PlanError):
        ExchangePlan(topo, layout, pl.shards, [0, 1, 2, 3], {t: 3 for t in range(4)}, {t: "none" for t in range(4)},
                     2, feature_towers={k: v for k, v in assignment.items() if k != 0})


def test_tm_host_math_matches_reference_formulas():
    cfg = P.TMConfig(kind="dlrm", out_dim=64)
    assert P.tm_output_width(cfg, 4, 128) == 256
    sizes = P.balanced_group_sizes(26, 8)
    ratios = [P.compression_ratio([P.tm_output_width(P.TMConfig(kind="dlrm", out_dim=d), s, 128) for s in sizes],
                                  sizes, 128) for d in (64, 32, 16, 8)]
    assert ratios == [2.0, 4.0, 8.0, 16.0]
    assert P.interaction_pairs(8, 4, 0.5) == (28.0, 10.0)
    with pytest.raises(P.DomainError):
        P.TMConfig(kind="mlp")


def test_library_exports_every_header_symbol():
    """The C ABI library loads (no GPU needed) and exports every function
    declared in include/dmt.h."""
    import os
    import re

    from paper_2403_00877_b200 import _lib

    if not os.path.exists(_lib.LIB_PATH):  # fresh checkout: build it (nvcc cross-compiles)
        from paper_2403_00877_b200.build import build

        build()
    lib = _lib.load_library(require_cuda=False)
    hdr = open(os.path.join(os.path.dirname(os.path.dirname(__file__)), "include", "dmt.h")).read()
    names = set(re.findall(r"^(?:int|int64_t|size_t|const char\*)\s+(dmt_\w+)\(", hdr, flags=re.M))
    assert len(names) >= 20
    for n in names:
        assert hasattr(lib, n), n
    assert set(_lib.EXPORTED) <= names | {"dmt_version"}
    assert lib.dmt_version().startswith(b"libdmt")


def test_product_refuses_cpu_fallback(monkeypatch):
    import torch

    from paper_2403_00877_b200 import _lib

    monkeypatch.setattr(torch.cuda, "is_available", lambda: False)
    with pytest.raises(P.TowersimError):
        _lib.lib()


@pytest.mark.parametrize("i", range(N_ACC))
def test_plan_trace_matches_reference_trace(i):
    """costmodel.plan_trace (host-side bytes from the plan, no run) equals the
    reference's recorded sent_by_rank per step at its 4 B/element wire format:
    step a, c (flat), d (all-to-all form), f (pass-through towers)."""
    from paper_2403_00877_b200 import costmodel as cm

    c = acceptance_case(i)
    m = c["meta"]
    lengths = c["lengths"]  # (G, F, B)
    nnz = {r: [int(lengths[r, j].sum()) for j in range(lengths.shape[1])] for r in range(lengths.shape[0])}
    tower = cm.plan_trace(_plan(c), nnz, 4, "sptt")
    flat = cm.plan_trace(_plan(c, sptt=False), nnz, 4, "flat")
    rs = m["cfg"]["exchange"]["rowwise_reducescatter"]
    has_tm = float(m["flops"].get("e", 0.0)) > 0
    want_t, want_b = m["tower_trace"], m["base_trace"]

    def sent(tr, label):
        return {str(k): v for k, v in tr.sent_by_rank(label).items()}

    assert sent(flat, "a") == want_b["a_sent"] and sent(flat, "c") == want_b["c_sent"]
    assert sent(tower, "a") == want_t["a_sent"]
    if not rs:
        assert sent(tower, "d") == want_t["d_sent"]
    if not has_tm:
        assert sent(tower, "f") == want_t["f_sent"]


def test_powerlaw_lengths_c5():
    """C5 pooling factors: seeded, in [1, 200], mean ~ 20, heavy tail."""
    from paper_2403_00877_b200.sptt import powerlaw_lengths

    a = powerlaw_lengths(512, 4096, seed=3)
    b = powerlaw_lengths(512, 4096, seed=3)
    assert np.array_equal(a, b) and a.dtype == np.int32 and a.shape == (512, 4096)
    assert a.min() >= 1 and a.max() <= 200
    assert 15.0 < a.mean() < 22.0
    assert (a >= 100).mean() > 0.005  # heavy tail present
