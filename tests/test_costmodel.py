"""Cost model (costmodel.py) vs the REAL reference's numbers on the traces of
the 60 acceptance configs (tests/golden/costmodel.json, made by
make_costmodel_golden.py), plus the calibration fit.  CPU only."""

from __future__ import annotations

import json
import math
import os

import pytest

from paper_2403_00877_b200 import costmodel as cm
from paper_2403_00877_b200.errors import DomainError, ReportError
from paper_2403_00877_b200.simnet import CommTrace
from paper_2403_00877_b200.topology import ClusterTopology, TowerLayout

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = json.load(open(os.path.join(HERE, "golden", "costmodel.json")))
ACC = json.load(open(os.path.join(HERE, "golden", "golden.json")))["acceptance"]


def _params(name):
    kw = dict(GOLD["params"][name])
    if "efficiency" in kw:
        kw["efficiency"] = {int(k): v for k, v in kw["efficiency"].items()}
    return cm.CostParams(**kw)


def _trace(topo, table):
    """Rebuild a trace with the reference's per-label sent_by_rank totals."""
    tr = CommTrace(topo)
    for label in [k for k in table if not k.endswith("_sent")]:
        sent = table.get(label + "_sent", {})
        if not sent:
            tr.record(label, 0, 0, 0)
        for src, nb in sent.items():
            tr.record(label, int(src), int(src), int(nb))
    return tr


def _close(a, b):
    return math.isclose(a, b, rel_tol=1e-12, abs_tol=1e-30)


@pytest.mark.parametrize("i", range(60))
def test_pipeline_cost_matches_reference(i):
    meta, gold = ACC[i], GOLD["configs"][i]
    topo = ClusterTopology(meta["num_hosts"], meta["ranks_per_host"])
    layout = TowerLayout(meta["num_towers"], meta["hosts_per_tower"])
    kinds = {"d": "reducescatter"} if gold["rowwise_reducescatter"] else None
    for name, want in gold["costs"].items():
        p = _params(name)
        cb = cm.pipeline_cost(_trace(topo, meta["base_trace"]), topo, p, flops=meta["base_flops"])
        ct = cm.pipeline_cost(_trace(topo, meta["tower_trace"]), topo, p, layout=layout, flops=meta["flops"],
                              step_kinds=kinds)
        for got, w in ((cb, want["base"]), (ct, want["tower"])):
            assert list(got.per_step) == list(w["per_step"])
            for k in w["per_step"]:
                assert _close(got.per_step[k], w["per_step"][k]), (name, k)
            assert _close(got.exposed_comm, w["exposed"]) and _close(got.compute, w["compute"])
        rep = cm.speedup_report(cb, ct)
        for k, v in want["speedup"].items():
            assert _close(rep[k], v), k


def test_closed_forms_and_validation():
    p = cm.CostParams(efficiency={1: 1.0}, alpha_out=1e-5, beta_out=1e9)
    assert cm.collective_latency("alltoall", 1, 1e9, "cross", p) == 0.0
    assert math.isclose(cm.collective_latency("alltoall", 2, 1000.0, "cross", p), 1e-5 + 500.0 / 1e9)
    assert cm.efficiency_at({1: 1.0, 8: 1.0, 16: 0.8}, 12) == 1.0
    assert cm.efficiency_at({4: 0.5}, 2) == 0.5
    t = cm.default_efficiency()
    assert t[8] == 1.0 and math.isclose(t[16], 0.8)
    with pytest.raises(DomainError):
        cm.CostParams(efficiency={1: 0.5, 2: 0.9})
    with pytest.raises(DomainError):
        cm.CostParams(beta_up=0)
    with pytest.raises(DomainError):
        cm.collective_latency("gather", 2, 1.0, "intra", p)
    topo = ClusterTopology(1, 2)
    tr = CommTrace(topo)
    tr.record("f", 0, 1, 8)
    with pytest.raises(ReportError):
        cm.pipeline_cost(tr, topo, cm.CostParams())
    with pytest.raises(DomainError):
        cm.speedup_report(cm.CostBreakdown({}, 0.0, 0.0), cm.CostBreakdown({}, 1.0, 0.0))


def test_calibrate_recovers_alpha_beta_efficiency():
    truth = cm.CostParams(alpha_up=7e-6, beta_up=600e9, efficiency={1: 1.0, 2: 1.0, 4: 0.9, 8: 0.7})
    samples = []
    for w in (2, 4, 8):
        for s in (1 << 20, 8 << 20, 64 << 20, 256 << 20):
            samples.append(cm.Sample(w, float(s), cm.INTRA, cm.collective_latency("alltoall", w, s, "intra", truth)))
    fit = cm.calibrate(samples)
    assert math.isclose(fit.alpha_up, 7e-6, rel_tol=1e-6)
    assert math.isclose(fit.beta_up, 600e9, rel_tol=1e-6)
    for w, e in truth.efficiency.items():
        assert math.isclose(cm.efficiency_at(fit.efficiency, w), e, rel_tol=1e-6)
    # scale-out untouched without samples
    assert fit.beta_out == cm.CostParams().beta_out
