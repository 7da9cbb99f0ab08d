"""Shared fixtures.  `-m gpu` tests need a B200; everything else runs on CPU."""

from __future__ import annotations

import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a) device")


def pytest_collection_modifyitems(config, items):
    try:
        import torch

        has_gpu = torch.cuda.is_available()
    except Exception:  # pragma: no cover
        has_gpu = False
    if has_gpu:
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


_cache: dict = {}


def golden_meta() -> dict:
    if "meta" not in _cache:
        with open(os.path.join(GOLDEN, "golden.json"), encoding="utf-8") as fh:
            _cache["meta"] = json.load(fh)
    return _cache["meta"]


def golden_npz(name: str):
    if name not in _cache:
        _cache[name] = dict(np.load(os.path.join(GOLDEN, name + ".npz")))
    return _cache[name]


def acceptance_case(i: int, key: str = "acceptance"):
    """Rebuild the inputs of acceptance config i (tests/golden/make_golden.py);
    key "acceptance_real" = the 200-config sweep with real-valued tables."""
    from oracle import OTopo, integer_tables, uniform_tables

    m = golden_meta()[key][i]
    arr = golden_npz(key)
    cfg = m["cfg"]
    t = cfg["tables"]
    shapes = {tid: (int(t["rows"]), int(t["dim"])) for tid in range(int(t["count"]))}
    if t["integer_values"]:
        tables = integer_tables(shapes)
    else:
        tables = uniform_tables(shapes, m["table_seed"])
    topo = OTopo(m["num_hosts"], m["ranks_per_host"], m["hosts_per_tower"])
    shards = [(a, b, c, tuple(d), tuple(e)) for a, b, c, d, e in m["placement"]]
    features = sorted(int(k) for k in m["pooling"])
    pooling = {int(k): v for k, v in m["pooling"].items()}
    assignment = {int(k): v for k, v in m["assignment"].items()}
    return dict(
        meta=m,
        topo=topo,
        tables=tables,
        shards=shards,
        features=features,
        pooling=pooling,
        assignment=assignment,
        lengths=arr[f"c{i}_lengths"],
        values=arr[f"c{i}_values"],
        base=arr[f"c{i}_base"],
        tower=arr[f"c{i}_tower"],
        realigned=arr[f"c{i}_realigned"],
        exchange=cfg["exchange"],
    )


def c1_full_inputs(TS, multi_hot: bool):
    """Full-size C1 through a towersim-compatible API module ``TS`` (this
    package): 2 x 4, 26 float64 U(-1, 1) tables x 100k x 64 (seed 0), B = 512,
    batch seed 1 (tests/golden/make_golden.gen_c1_full)."""
    topo = TS.ClusterTopology(2, 4)
    layout = TS.TowerLayout(2)
    tables = {t: TS.init_table_deterministic(t, 100_000, 64, seed=0) for t in range(26)}
    assignment = {t: (0 if t < 13 else 1) for t in range(26)}
    placement = TS.shard_tables(tables, {t: TS.TablePlan("table_wise", 1, assignment[t]) for t in tables}, topo,
                                layout)
    hot = (10, 30) if multi_hot else 1
    batch = TS.make_batch(topo, tables, 512, {t: hot for t in tables}, seed=1)
    return topo, placement, batch, TS.TowerPlan(layout, assignment), tables


def sha256(a) -> str:
    import hashlib

    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def fp32_case(name: str):
    """Rebuild inputs of a reduced-C1 float32-table case (make_golden.gen_fp32_c1)."""
    from oracle import OTopo, uniform_tables

    m = golden_meta()["fp32_c1"][name]
    arr = golden_npz("fp32_c1")
    shapes = {tid: (m["rows"], m["dim"]) for tid in range(26)}
    tables = uniform_tables(shapes, 0, dtype=np.float32)
    topo = OTopo(2, 4, 1)
    shards = [(a, b, c, tuple(d), tuple(e)) for a, b, c, d, e in m["placement"]]
    features = list(range(26))
    pooling = {int(k): v for k, v in m["pooling"].items()}
    assignment = {t: (0 if t < 13 else 1) for t in range(26)}
    out = dict(
        meta=m,
        topo=topo,
        tables=tables,
        shards=shards,
        features=features,
        pooling=pooling,
        assignment=assignment,
        lengths=arr[f"{name}_lengths"],
        values=arr[f"{name}_values"],
        tower=arr[f"{name}_tower"].astype(np.float64),
    )
    if f"{name}_base" in arr:
        out["base"] = arr[f"{name}_base"].astype(np.float64)
    return out


def tm_case(i: int):
    """(cfg dict, weights, direction, embs, out, jvp, meta) of golden TM case i."""
    m = golden_meta()["tm"][i]
    arr = golden_npz("tm")
    cfg = {"kind": m["kind"], "out_dim": 64, "per_feature_outputs": 1, "flat_outputs": 0,
           "cross_layers": 3, "seed": m["seed"]}
    cfg.update(m["kw"])

    def weights(prefix):
        if m["kind"] == "dlrm":
            return {k: arr[f"t{i}_{prefix}_{k}"] for k in ("w_flat", "b_flat", "w_feat", "b_feat")}
        cross = []
        layer = 0
        while f"t{i}_{prefix}_cross{layer}_w" in arr:
            cross.append((arr[f"t{i}_{prefix}_cross{layer}_w"], arr[f"t{i}_{prefix}_cross{layer}_b"]))
            layer += 1
        return {"cross": cross, "w_proj": arr[f"t{i}_{prefix}_w_proj"],
                "b_proj": arr[f"t{i}_{prefix}_b_proj"]}

    return cfg, weights("w"), weights("d"), arr[f"t{i}_embs"], arr[f"t{i}_out"], \
        arr[f"t{i}_jvp"], m


@pytest.fixture
def rng():
    return np.random.default_rng(12345)


def max_rel_err(got, want) -> float:
    """max |got - want| / max |want| (max-norm relative error), float64."""
    got = np.asarray(got, dtype=np.float64)
    want = np.asarray(want, dtype=np.float64)
    den = float(np.abs(want).max()) if want.size else 0.0
    return float(np.abs(got - want).max()) / max(den, 1e-300) if want.size else 0.0


def oracle_tm_weights(tm) -> dict:
    """A device TowerModule's *current* weights (as stored: bf16-rounded for a
    bf16 module) in the oracle's dict layout, so the oracle evaluates exactly
    the model the device holds."""
    w = tm.host_weights()
    if tm.cfg.kind == "dlrm":
        return {"w_flat": w.w_flat, "b_flat": w.b_flat, "w_feat": w.w_feat, "b_feat": w.b_feat}
    return {"cross": [tuple(c) for c in w.cross], "w_proj": w.w_proj, "b_proj": w.b_proj}


def oracle_tm_cfg(cfg) -> dict:
    return {"kind": cfg.kind, "out_dim": cfg.out_dim, "per_feature_outputs": cfg.per_feature_outputs,
            "flat_outputs": cfg.flat_outputs, "cross_layers": cfg.cross_layers, "seed": cfg.seed}
