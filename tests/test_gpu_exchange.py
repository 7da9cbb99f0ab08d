"""GPU parity of the reference-compatible exchange API (tower_exchange,
baseline_exchange, realign) against the reference's own golden outputs."""

from __future__ import annotations

import numpy as np
import pytest

from conftest import acceptance_case, fp32_case, golden_meta

pytestmark = pytest.mark.gpu

N_ACC = len(golden_meta()["acceptance"])
N_ACC_REAL = len(golden_meta()["acceptance_real"])


def _api_inputs(c, dtype=None):
    """Reference-typed objects (our package) from a golden case."""
    import paper_2403_00877_b200 as P

    m = c["meta"]
    topo = P.ClusterTopology(c["topo"].num_hosts, c["topo"].ranks_per_host)
    layout = P.TowerLayout(c["topo"].T, c["topo"].hosts_per_tower)
    tables = {t: P.EmbeddingTable(t, v.shape[0], v.shape[1], v) for t, v in c["tables"].items()}
    shards = [P.Shard(a, b, s, tuple(r), tuple(cc)) for a, b, s, r, cc in c["shards"]]
    placement = P.ShardedEmbedding(tables, shards)
    G, F, B = c["lengths"].shape
    offs = np.concatenate([[0], np.cumsum(c["lengths"].reshape(-1))])
    bags = []
    for r in range(G):
        per = {}
        for fi, f in enumerate(c["features"]):
            base = (r * F + fi) * B
            per[f] = [[int(x) for x in c["values"][offs[base + b]:offs[base + b + 1]]] for b in range(B)]
        bags.append(per)
    batch = P.SparseBatch(bags, B, dict(c["pooling"]))
    plan = P.TowerPlan(layout, dict(c["assignment"]))
    return P, topo, layout, placement, batch, plan


@pytest.mark.parametrize("key,i", [("acceptance", i) for i in range(N_ACC)] +
                         [("acceptance_real", i) for i in range(N_ACC_REAL)])
def test_acceptance_configs_bit_exact(key, i):
    """The reference's acceptance sweep through the GPU API: 60 configs with
    integer tables and 200 with real-valued float64 tables (bag-order lookup
    sums, row-range and reduce-scatter combine orders all bit-exact)."""
    c = acceptance_case(i, key)
    P, topo, layout, placement, batch, plan = _api_inputs(c)
    ex = c["exchange"]
    opts = P.ExchangeOptions(swap_bc=ex["swap_bc"], omit_permute=ex["omit_permute"],
                             rowwise_reducescatter=ex["rowwise_reducescatter"])
    base = P.baseline_exchange(batch, placement, topo)
    tower = P.tower_exchange(batch, placement, plan, topo, opts)
    m = c["meta"]
    for r in range(topo.world_size):
        assert np.array_equal(base.outputs[r], c["base"][r]), r
        assert np.array_equal(tower.outputs[r], c["tower"][r]), r
    assert [list(b) for b in tower.layout.blocks] == m["tower_layout"]
    assert [list(b) for b in base.layout.blocks] == m["base_layout"]
    re = P.realign(tower, [f for _, f, _ in base.layout.blocks])
    for r in range(topo.world_size):
        assert np.array_equal(re.outputs[r], c["realigned"][r])
    for label in ("a", "c"):
        assert list(base.trace.byte_totals(label)) == m["base_trace"][label], label
    for label in ("a", "d", "f"):
        assert list(tower.trace.byte_totals(label)) == m["tower_trace"][label], label


@pytest.mark.parametrize("name", ["tw_single", "tw_multi", "cw_multi", "rw_multi"])
def test_fp32_tables_reduced_c1(name):
    c = fp32_case(name)
    P, topo, layout, placement, batch, plan = _api_inputs(c)
    tower = P.tower_exchange(batch, placement, plan, topo)
    for r in range(8):
        if name == "rw_multi":  # fp64 partial sums rounded to fp32 once
            np.testing.assert_allclose(tower.outputs[r], c["tower"][r], rtol=1e-6, atol=1e-6)
        else:
            assert np.array_equal(tower.outputs[r], c["tower"][r])
    if "base" in c:
        base = P.baseline_exchange(batch, placement, topo)
        for r in range(8):
            assert np.array_equal(base.outputs[r], c["base"][r])


@pytest.mark.parametrize("name", ["tw_dlrm", "tw_dcn"])
def test_fp32_tables_with_tower_modules(name):
    c = fp32_case(name)
    P, topo, layout, placement, batch, plan = _api_inputs(c)
    t = c["meta"]["tm"]
    cfg = P.TMConfig(kind=t["kind"], out_dim=t["out_dim"], per_feature_outputs=t["per_feature_outputs"],
                     flat_outputs=t["flat_outputs"], cross_layers=t["cross_layers"], seed=t["seed"])
    tower = P.tower_exchange(batch, placement, plan, topo, P.ExchangeOptions(tower_modules=cfg))
    assert [list(b) for b in tower.layout.blocks] == c["meta"]["tower_layout"]
    for r in range(8):
        np.testing.assert_allclose(tower.outputs[r], c["tower"][r], rtol=1e-5, atol=1e-5)


def test_tm_forward_golden():
    import paper_2403_00877_b200 as P
    from conftest import tm_case

    for i in range(len(golden_meta()["tm"])):
        cfg, w, d, embs, out, jvp, m = tm_case(i)
        tc = P.TMConfig(kind=cfg["kind"], out_dim=cfg["out_dim"], per_feature_outputs=cfg["per_feature_outputs"],
                        flat_outputs=cfg["flat_outputs"], cross_layers=cfg["cross_layers"], seed=cfg["seed"])
        weights = P.init_tm_weights(tc, m["F"], m["N"], salt=m["salt"])
        got = P.tm_forward(embs, tc, weights)
        np.testing.assert_allclose(got, out, rtol=1e-5, atol=1e-5)


@pytest.mark.parametrize("multi", [False, True])
def test_c1_full_size_bit_exact(multi):
    """Full-size C1 (2 towers x 4, 26 x 100k x 64 float64 tables, B = 512 per
    rank, single- and multi-hot) through tower_exchange / baseline_exchange on
    the GPU: SHA-256 of every rank's exact float64 output equals the
    reference's, and so do the step-a/d/f byte totals."""
    import paper_2403_00877_b200 as P
    from conftest import c1_full_inputs, sha256

    m = golden_meta()["c1_full"]["multi_hot" if multi else "single_hot"]
    topo, placement, batch, plan, _ = c1_full_inputs(P, multi)
    tower = P.tower_exchange(batch, placement, plan, topo)
    base = P.baseline_exchange(batch, placement, topo)
    for r in range(8):
        assert sha256(tower.outputs[r]) == m["tower_sha"][str(r)], r
        assert sha256(base.outputs[r]) == m["base_sha"][str(r)], r
    for r in ("0", "5"):
        assert np.array_equal(tower.outputs[int(r)][:4], np.asarray(m["tower_rows0_3"][r]))
    assert [list(b) for b in tower.layout.blocks] == m["tower_layout"]
    for label in ("a", "d", "f"):
        assert list(tower.trace.byte_totals(label)) == m["tower_trace"][label], label
