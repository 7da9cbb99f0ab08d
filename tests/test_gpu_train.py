"""GPU parity of the backward path: fused embedding-bag backward + optimizers,
tower-module backward, and a full SPTT train step (loopback ranks) against the
oracle's restatement (oracle/backward.py)."""

from __future__ import annotations

import numpy as np
import pytest
import torch

from conftest import max_rel_err, oracle_tm_weights

pytestmark = pytest.mark.gpu

import oracle  # noqa: E402


def dev():
    return torch.device("cuda")


def _bwd_case(rng, rows, width, nbags, maxlen, mode, hot=False):
    lens = np.ones(nbags, np.int64) if mode == "none" else rng.integers(0, maxlen + 1, size=nbags)
    if hot:  # power-law-ish: many repeats of a few rows
        idx = (rng.zipf(1.3, size=int(lens.sum())) - 1) % rows
    else:
        idx = rng.integers(0, rows, size=int(lens.sum()))
    g = rng.normal(size=(nbags, width)).astype(np.float32)
    return lens, idx, g


@pytest.mark.parametrize("opt", ["sgd", "adagrad"])
@pytest.mark.parametrize("mode", ["sum", "mean", "none"])
@pytest.mark.parametrize("hot", [False, True])
@pytest.mark.parametrize("width", [4, 64, 128, 200])
@pytest.mark.parametrize("dt", ["fp32", "bf16"])
def test_embedding_backward_fused_optimizer(opt, mode, hot, width, dt):
    from paper_2403_00877_b200 import _lib as L
    from paper_2403_00877_b200 import kernels as K

    rng = np.random.default_rng(width + (7 if hot else 0))
    rows = 500
    table = rng.uniform(-1, 1, (rows, width)).astype(np.float32)
    lens, idx, g = _bwd_case(rng, rows, width, 300, 12, mode, hot)
    tdt = torch.bfloat16 if dt == "bf16" else torch.float32
    W = torch.from_numpy(table.copy()).to(dev()).to(tdt)
    G = torch.from_numpy(g).to(dev()).to(tdt)
    if dt == "bf16":  # the oracle starts from the same bf16-rounded table / gradients
        table = W.float().cpu().numpy()
        g = G.float().cpu().numpy()
    state = torch.full((rows,), 0.1, dtype=torch.float32, device=dev())
    offs = K.lengths_to_offsets(torch.from_numpy(lens.astype(np.int32)).to(dev()))
    I = torch.from_numpy(idx.astype(np.int32)).to(dev())
    seg = K.Segment(weights=W, out=G, out_offset=0, out_ld=width, bag_begin=0, nbags=len(lens),
                    pooling=L.POOL_CODE[mode], state=state if opt == "adagrad" else None)
    ws = K.pooled_lookup_bwd_workspace(int(lens.sum()), rows, len(lens), dev())
    K.pooled_lookup_bwd(K.SegmentTable([seg], dev()), offs, I, int(lens.sum()), rows,
                        L.OPT_ROWWISE_ADAGRAD if opt == "adagrad" else L.OPT_SGD, 0.05, 1e-8, ws)
    uniq, grads = oracle.embedding_row_grads(rows, lens, idx, g.astype(np.float64), mode)
    if opt == "sgd":
        want = oracle.apply_sgd(table, uniq, grads, 0.05)
    else:
        want, want_s = oracle.apply_rowwise_adagrad(table, np.full(rows, 0.1), uniq, grads, 0.05, 1e-8)
        np.testing.assert_allclose(state.double().cpu().numpy(), want_s, rtol=1e-5, atol=1e-6)
    tol = 1e-2 if dt == "bf16" else 1e-5  # north-star tolerance per dtype
    np.testing.assert_allclose(W.double().cpu().numpy(), want, rtol=tol, atol=tol)


def test_embedding_backward_is_deterministic():
    from paper_2403_00877_b200 import _lib as L
    from paper_2403_00877_b200 import kernels as K

    rng = np.random.default_rng(1)
    rows, width = 64, 128
    lens, idx, g = _bwd_case(rng, rows, width, 4000, 30, "sum", hot=True)
    outs = []
    for _ in range(3):
        W = torch.zeros((rows, width), dtype=torch.float32, device=dev())
        offs = K.lengths_to_offsets(torch.from_numpy(lens.astype(np.int32)).to(dev()))
        seg = K.Segment(weights=W, out=torch.from_numpy(g).to(dev()), out_offset=0, out_ld=width, bag_begin=0,
                        nbags=len(lens), pooling=L.POOL_SUM)
        ws = K.pooled_lookup_bwd_workspace(int(lens.sum()), rows, len(lens), dev())
        K.pooled_lookup_bwd(K.SegmentTable([seg], dev()), offs, torch.from_numpy(idx.astype(np.int32)).to(dev()),
                            int(lens.sum()), rows, L.OPT_SGD, 1.0, 0.0, ws)
        outs.append(W.cpu().numpy())
    assert np.array_equal(outs[0], outs[1]) and np.array_equal(outs[1], outs[2])


_MANY_SHARDS = r"""
import sys, numpy as np, torch
sys.path.insert(0, {root!r})
from paper_2403_00877_b200 import _lib as L
from paper_2403_00877_b200 import kernels as K

def run(dt, opt, big=False):
    rng = np.random.default_rng(5)
    dev = torch.device("cuda")
    # 40 shards of very different sizes (1 .. 3000 rows) in one key space, so
    # several shard boundaries share a bucket of the apply's shard table;
    # 14-bit keys = 2 radix passes, big (a 300k-row shard added) 19 bits = 3
    sizes = [1, 2, 3, 7, 1, 3000, 5, 1, 1, 64, 900, 2, 2, 2, 17, 1, 1200, 33, 1, 8] * 2
    if big:
        sizes[7] = 300000
    width, nbags = 128, 700
    tdt = torch.bfloat16 if dt == "bf16" else torch.float32
    tables, segs, lens_all, idx_all, g_all = [], [], [], [], []
    G = torch.empty(len(sizes) * nbags * width, device=dev, dtype=tdt)
    kb = 0
    for t, rows in enumerate(sizes):
        lens = rng.integers(0, 9, size=nbags)
        idx = (rng.zipf(1.5, size=int(lens.sum())) - 1) % rows
        W = torch.from_numpy(rng.uniform(-1, 1, (rows, width)).astype(np.float32)).to(dev).to(tdt)
        g = torch.from_numpy(rng.normal(size=(nbags, width)).astype(np.float32)).to(dev).to(tdt)
        G[t * nbags * width:(t + 1) * nbags * width] = g.reshape(-1)
        st = torch.full((rows,), 0.1, dtype=torch.float32, device=dev)
        segs.append(K.Segment(weights=W, out=G, out_offset=t * nbags * width, out_ld=width, bag_begin=t * nbags,
                              nbags=nbags, pooling=L.POOL_SUM, key_base=kb, state=st if opt else None))
        tables.append((W.clone(), st.clone(), W, st, rows))
        lens_all.append(lens); idx_all.append(idx); g_all.append(g.float().cpu().numpy())
        kb += rows
    lens = np.concatenate(lens_all)
    offs = K.lengths_to_offsets(torch.from_numpy(lens.astype(np.int32)).to(dev))
    I = torch.from_numpy(np.concatenate(idx_all).astype(np.int32)).to(dev)
    nnz = int(lens.sum())
    ws = K.pooled_lookup_bwd_workspace(nnz, kb, len(lens), dev)
    K.pooled_lookup_bwd(K.SegmentTable(segs, dev), offs, I, nnz, kb,
                        L.OPT_ROWWISE_ADAGRAD if opt else L.OPT_SGD, 0.05, 1e-8, ws)
    torch.cuda.synchronize()
    return tables, lens_all, idx_all, g_all

if __name__ == "__main__":
    out = {{}}
    for dt in ("bf16", "fp32"):
        for opt in (0, 1):
            for big in (0, 1):
                tables, *_ = run(dt, opt, bool(big))
                for t, (W0, S0, W, S, rows) in enumerate(tables):
                    out[f"{{dt}}_{{opt}}_{{big}}_{{t}}"] = W.float().cpu().numpy()
                    out[f"{{dt}}_{{opt}}_{{big}}_{{t}}_s"] = S.cpu().numpy()
    np.savez(sys.argv[1], **out)
"""


def _many_shards_module(tmp_path):
    import importlib.util
    import os

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    path = tmp_path / "many_shards.py"
    path.write_text(_MANY_SHARDS.format(root=root))
    spec = importlib.util.spec_from_file_location("many_shards", path)
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod, path


@pytest.mark.parametrize("big", [False, True])
@pytest.mark.parametrize("opt", [0, 1])
@pytest.mark.parametrize("dt", ["bf16", "fp32"])
def test_embedding_backward_many_shards(dt, opt, big, tmp_path):
    """40 shards of 1..3000 rows in one key space: the apply's shard table
    (bucket of the key -> shard of its first key, then a forward walk) must
    resolve every key to its own shard."""
    mod, _ = _many_shards_module(tmp_path)
    tables, lens_all, idx_all, g_all = mod.run(dt, opt, big)
    # fp32: the 1-row shards sum ~2,800 N(0, 1) gradient rows in fp32 (the
    # oracle in fp64): 2e-5 absolute after lr 0.05, hence atol 5e-5
    rtol, atol = (1e-2, 1e-2) if dt == "bf16" else (1e-5, 5e-5)
    for (W0, S0, W, S, rows), lens, idx, g in zip(tables, lens_all, idx_all, g_all):
        table = W0.float().cpu().numpy().astype(np.float64)
        uniq, grads = oracle.embedding_row_grads(rows, lens, idx, g.astype(np.float64), "sum")
        if opt:
            want, want_s = oracle.apply_rowwise_adagrad(table, S0.double().cpu().numpy(), uniq, grads, 0.05, 1e-8)
            np.testing.assert_allclose(S.double().cpu().numpy(), want_s, rtol=1e-5, atol=1e-6)
        else:
            want = oracle.apply_sgd(table, uniq, grads, 0.05)
        np.testing.assert_allclose(W.double().cpu().numpy(), want, rtol=rtol, atol=atol)


def test_embedding_backward_apply_variants_agree(tmp_path):
    """Every apply variant (DMT_BWD_VARIANT) and both sorts (DMT_BWD_SORT: the
    hand-written radix sort, CUB) -- read once per process, so one subprocess
    each -- sum a run's rows in the same order: bit-identical tables and
    optimizer state."""
    import os
    import subprocess
    import sys

    _, path = _many_shards_module(tmp_path)
    res = {}
    for v in ("7", "cub", "0", "1", "2", "4", "5", "6"):
        out = tmp_path / f"v{v}.npz"
        env = dict(os.environ)
        if v == "cub":
            env["DMT_BWD_SORT"] = "cub"
        else:
            env["DMT_BWD_VARIANT"] = v
        subprocess.run([sys.executable, str(path), str(out)], env=env, check=True, timeout=600)
        res[v] = np.load(out)
    for v, r in res.items():
        for k in r.files:
            if k.split("_")[1] == "0" or v == "cub":  # same summation order -> identical bits
                assert np.array_equal(r[k], res["7"][k]), (v, k)
            else:  # row-wise Adagrad: the squared-norm reduction tree differs between kernels
                np.testing.assert_allclose(r[k], res["7"][k], rtol=2e-6, atol=1e-7, err_msg=f"{v} {k}")


def _tm_objects(kind, F, N, dt, seed=0, layers=3):
    import paper_2403_00877_b200 as P

    if kind == "dlrm":
        cfg = P.TMConfig(kind="dlrm", out_dim=16, per_feature_outputs=2, flat_outputs=1, seed=seed)
        ocfg = {"kind": "dlrm", "out_dim": 16, "per_feature_outputs": 2, "flat_outputs": 1, "cross_layers": 3,
                "seed": seed}
    else:
        cfg = P.TMConfig(kind="dcn", out_dim=16, cross_layers=layers, seed=seed)
        ocfg = {"kind": "dcn", "out_dim": 16, "per_feature_outputs": 1, "flat_outputs": 0, "cross_layers": layers,
                "seed": seed}
    w = P.init_tm_weights(cfg, F, N, salt=1)
    ow = oracle.init_tm_weights(ocfg, F, N, salt=1)
    return P.TowerModule(cfg, F, N, w, dtype=dt), ocfg, ow


# DCN variants: 3 layers / width 192 = pair-sum final epilogue + fused bias
# column sums; width 48 = pair sum on the unaligned epilogue path with separate
# column sums; 5 layers = the fp32 dx0-accumulator form (more than 4 pairs).
# "side" (the default) computes dx0 and the bias gradients on a side stream.
@pytest.mark.parametrize("kind,F,N,layers", [("dlrm", 6, 32, 3), ("dcn", 6, 32, 3), ("dcn", 3, 16, 3),
                                             ("dcn", 6, 32, 5), ("dcn", 4, 32, 1)])
@pytest.mark.parametrize("dt", [torch.float32, torch.bfloat16])
@pytest.mark.parametrize("form", ["side", "accumulate", "pairs"])
def test_tower_module_backward_vs_oracle(kind, F, N, layers, dt, form, monkeypatch):
    import paper_2403_00877_b200 as P

    if kind == "dlrm" and form == "pairs":
        pytest.skip("DCN-only variant")
    monkeypatch.setattr(P.TowerModule, "dcn_bwd_form", form)
    rows = 300
    tm, ocfg, _ = _tm_objects(kind, F, N, dt, layers=layers)
    ow = oracle_tm_weights(tm)  # the weights the device holds (bf16-rounded for bf16)
    rng = np.random.default_rng(4)
    x = rng.normal(size=(rows, F, N)) * 0.5
    if dt == torch.bfloat16:
        x = oracle.bf16_round(x.astype(np.float32)).astype(np.float64)
    xt = torch.from_numpy(x.reshape(rows, F * N)).to(dev(), dt)
    y = tm.forward(xt, save=True)
    want_y = oracle.tm_forward(x, ocfg, ow)
    tol = 1e-5 if dt == torch.float32 else 1e-2  # north-star tolerances (max-norm relative)
    assert max_rel_err(y.double().cpu().numpy(), want_y) <= tol
    g = rng.normal(size=want_y.shape)
    if dt == torch.bfloat16:
        g = oracle.bf16_round(g.astype(np.float32)).astype(np.float64)
    dx = tm.backward(torch.from_numpy(g).to(dev(), dt))
    want_dx, want_dw = oracle.tm_backward(x, ocfg, ow, g)
    assert max_rel_err(dx.double().cpu().numpy().reshape(rows, F, N), want_dx) <= tol
    if kind == "dlrm":
        pairs = [(k, want_dw[k]) for k in ("w_flat", "b_flat", "w_feat", "b_feat")]
    else:
        pairs = [("w_proj", want_dw["w_proj"]), ("b_proj", want_dw["b_proj"])]
        for i, (gw, gb) in enumerate(want_dw["cross"]):
            pairs += [(f"w{i}", gw), (f"b{i}", gb)]
    for k, want in pairs:
        got = tm.grads[k].double().cpu().numpy()
        assert max_rel_err(got, want) <= tol, (k, max_rel_err(got, want))


def _assert_sgd_rows(got, before, want, tol=1e-5, what=""):
    """Table rows after an optimizer step: the update (got - before) equals the
    oracle's (want - before) to ``tol`` max-norm relative; untouched rows are
    bit-identical.  fp32 tables: the stored value's own rounding (2^-24
    relative) is allowed on top."""
    d_want = want - before
    scale = max(np.abs(d_want).max(), 1e-300)
    err = np.abs(got - want)
    bound = tol * scale + 2.0 ** -23 * np.abs(want)
    assert (err <= bound).all(), (what, float((err / scale).max()))
    untouched = d_want == 0
    assert np.array_equal(got[untouched], before[untouched]), what


@pytest.mark.parametrize("hosts,rph,kind,scheme,opt", [
    (2, 2, "dlrm", "table_wise", "sgd"), (2, 4, "dcn", "table_wise", "sgd"), (4, 2, "dcn", "table_wise", "sgd"),
    (1, 1, "dcn", "table_wise", "sgd"), (2, 2, "dcn", "column_wise", "sgd"), (2, 2, "dcn", "row_wise", "sgd"),
    (2, 2, "dlrm", "table_wise", "adagrad"), (2, 4, "dcn", "column_wise", "adagrad"),
    # one-rank towers (W = 1): lookup -> X and dX -> embedding backward in place
    (2, 1, "dcn", "column_wise", "sgd"), (4, 1, "dlrm", "table_wise", "adagrad"), (2, 1, "dcn", "row_wise", "sgd")])
def test_sptt_train_step_loopback_vs_oracle(hosts, rph, kind, scheme, opt):
    """Full step on G simulated ranks: outputs, then every table row after the
    optimizer (SGD or row-wise Adagrad), for table/column/row-wise shards."""
    import paper_2403_00877_b200 as P
    from paper_2403_00877_b200.fabric import LoopbackFabric
    from paper_2403_00877_b200.pipeline import KJT
    from paper_2403_00877_b200.sptt import SPTT, build_world

    F, rows, N, B = 8, 60, 16, 5
    topo, layout, placement, assignment = build_world(hosts, rph, 1, F, rows, N, seed=2, scheme=scheme,
                                                      shards_per_table=2)
    G, T = topo.world_size, layout.num_towers
    # mean pooling is undefined over row-wise partial pools (the reference sums them)
    pooling = {f: ("mean" if f % 3 == 0 and scheme != "row_wise" else "sum") for f in range(F)}
    if kind == "dlrm":
        cfg = P.TMConfig(kind="dlrm", out_dim=8, per_feature_outputs=1, flat_outputs=1, seed=1)
    else:
        cfg = P.TMConfig(kind="dcn", out_dim=8, cross_layers=2, seed=1)
    ocfg = {"kind": cfg.kind, "out_dim": 8, "per_feature_outputs": cfg.per_feature_outputs,
            "flat_outputs": cfg.flat_outputs, "cross_layers": cfg.cross_layers, "seed": 1}
    before = {t: placement.tables[t].values.astype(np.float64).copy() for t in range(F)}
    lr = 0.05
    model = SPTT(topo, layout, placement, assignment, pooling, B, LoopbackFabric(G, dev()), tm=cfg,
                 dtype=torch.float32, lr=lr, optimizer=opt, eps=1e-6)
    rng = np.random.default_rng(11)
    lens = rng.integers(0, 5, size=(G, F, B)).astype(np.int32)
    vals = rng.integers(0, rows, size=int(lens.sum())).astype(np.int64)
    offs = np.concatenate([[0], np.cumsum(lens.reshape(-1))])
    kjts = {}
    for r in range(G):
        seg = vals[offs[r * F * B]:offs[(r + 1) * F * B]]
        kjts[r] = KJT(torch.from_numpy(lens[r].reshape(-1)).to(dev()), torch.from_numpy(seg.astype(np.int32)).to(dev()),
                      [int(lens[r, f].sum()) for f in range(F)], B)
    O = model.plan.out_width()
    grads = {r: torch.from_numpy(rng.normal(size=(B, O)).astype(np.float32)).to(dev()) for r in range(G)}
    outs = model.train_step(kjts, grads)
    torch.cuda.synchronize()
    # the direct-X path is taken exactly for one-rank towers without row-wise shards
    assert bool(model.engine.direct_x) == (rph == 1 and scheme != "row_wise")

    shards = [(s.table_id, s.rank, s.scheme, s.row_range, s.col_range) for s in placement.shards]
    flat, _, _, _ = oracle.baseline_forward(lens, vals, list(range(F)), pooling, before, shards,
                                            oracle.OTopo(hosts, rph))
    by_tower = {t: [f for f in range(F) if assignment[f] == t] for t in range(T)}
    tw = {t: oracle.init_tm_weights(ocfg, len(by_tower[t]), N, salt=t) for t in range(T)}
    grad_rows = {t: np.zeros_like(before[t]) for t in range(F)}
    for r in range(G):
        g_r = grads[r].double().cpu().numpy()
        col = 0
        for t in range(T):
            fs = by_tower[t]
            x = flat[r][:, fs[0] * N:(fs[-1] + 1) * N].reshape(B, len(fs), N)
            ow_ = oracle.tm_output_width(ocfg, len(fs), N)
            y = oracle.tm_forward(x, ocfg, tw[t])
            np.testing.assert_allclose(outs[r][:, col:col + ow_].double().cpu().numpy(), y, rtol=1e-5, atol=1e-5)
            dx, _ = oracle.tm_backward(x, ocfg, tw[t], g_r[:, col:col + ow_])
            col += ow_
            for i, f in enumerate(fs):
                base = (r * F + f) * B
                for b in range(B):
                    n = offs[base + b + 1] - offs[base + b]
                    for k in range(offs[base + b], offs[base + b + 1]):
                        scale = 1.0 / n if pooling[f] == "mean" else 1.0
                        grad_rows[f][vals[k]] += scale * dx[b, i]
    expect = {}
    for f in range(F):
        touched = np.unique(vals[np.concatenate([np.arange(offs[(r * F + f) * B], offs[(r * F + f + 1) * B])
                                                 for r in range(G)])])
        if opt == "sgd":
            expect[f] = oracle.apply_sgd(before[f], touched, grad_rows[f][touched], lr)
        else:
            expect[f], _ = oracle.apply_rowwise_adagrad(before[f], np.zeros(rows), touched,
                                                        grad_rows[f][touched], lr, 1e-6)
    for sid, sh in enumerate(placement.shards):
        got = model.engine.weights[sid].double().cpu().numpy()
        (r0, r1), (c0, c1) = sh.row_range, sh.col_range
        want = expect[sh.table_id][r0:r1, c0:c1]
        if opt == "adagrad" and sh.scheme == "column_wise":
            # row-wise Adagrad on a column shard normalises by that shard's own
            # squared-gradient mean (one accumulator per shard row), so compare
            # against the shard-local rule
            gsh = grad_rows[sh.table_id][:, c0:c1]
            tch = np.unique(np.nonzero(np.any(gsh != 0, axis=1))[0])
            want, _ = oracle.apply_rowwise_adagrad(before[sh.table_id][:, c0:c1], np.zeros(rows), tch, gsh[tch],
                                                   lr, 1e-6)
        _assert_sgd_rows(got, before[sh.table_id][r0:r1, c0:c1], want, what=f"shard {sid}")


@pytest.mark.parametrize("dt", [torch.float32, torch.bfloat16])
def test_dcn_fused_sgd_matches_unfused(dt):
    """W -= lr * dW inside the dW GEMM epilogue == explicit grads + SGD."""
    F, N, rows, lr = 4, 32, 256, 0.05
    tm_a, _, _ = _tm_objects("dcn", F, N, dt, seed=3)
    tm_b, _, _ = _tm_objects("dcn", F, N, dt, seed=3)
    rng = np.random.default_rng(8)
    x = torch.from_numpy(rng.normal(size=(rows, F * N)) * 0.5).to(dev(), dt)
    g = torch.from_numpy(rng.normal(size=(rows, tm_a.width))).to(dev(), dt)
    tm_a.forward(x, save=True)
    dxa = tm_a.backward(g)
    tm_a.sgd_step(lr)
    tm_b.forward(x, save=True)
    dxb = tm_b.backward(g, fused_lr=lr)
    tm_b.sgd_step(lr)  # biases only
    tol = 1e-5 if dt == torch.float32 else 2e-2
    assert torch.allclose(dxa.double(), dxb.double(), rtol=tol, atol=tol)
    for k in tm_a.w:
        assert torch.allclose(tm_a.w[k].double(), tm_b.w[k].double(), rtol=tol, atol=tol), k


@pytest.mark.parametrize("hosts,rph,top_kind", [(2, 2, "dcn"), (1, 2, "dlrm"), (2, 1, "dcn")])
def test_full_model_bce_step_loopback_vs_oracle(hosts, rph, top_kind):
    """DCN + SPTT model with a loss: SPTT (DCN tower modules) -> top head
    (crossnet + one-logit projection, or a one-logit linear) -> BCE on labels.
    Loss, top weights after SGD and every embedding row after SGD vs the
    oracle's flat-model restatement (fp32, rtol 1e-4)."""
    import paper_2403_00877_b200 as P
    from paper_2403_00877_b200.fabric import LoopbackFabric
    from paper_2403_00877_b200.pipeline import KJT
    from paper_2403_00877_b200.sptt import SPTT, build_world

    F, rows, N, B = 6, 50, 16, 4
    topo, layout, placement, assignment = build_world(hosts, rph, 1, F, rows, N, seed=3)
    G, T = topo.world_size, layout.num_towers
    pooling = {f: "sum" for f in range(F)}
    cfg = P.TMConfig(kind="dcn", out_dim=4, cross_layers=2, seed=1)
    ocfg = {"kind": "dcn", "out_dim": 4, "per_feature_outputs": 1, "flat_outputs": 0, "cross_layers": 2, "seed": 1}
    if top_kind == "dcn":
        top = P.TMConfig(kind="dcn", out_dim=1, cross_layers=2, seed=7)
        otop = {"kind": "dcn", "out_dim": 1, "per_feature_outputs": 1, "flat_outputs": 0, "cross_layers": 2,
                "seed": 7}
    else:
        top = P.TMConfig(kind="dlrm", out_dim=1, per_feature_outputs=1, flat_outputs=0, seed=7)
        otop = {"kind": "dlrm", "out_dim": 1, "per_feature_outputs": 1, "flat_outputs": 0, "cross_layers": 3,
                "seed": 7}
    before = {t: placement.tables[t].values.astype(np.float64).copy() for t in range(F)}
    lr = 0.1
    model = SPTT(topo, layout, placement, assignment, pooling, B, LoopbackFabric(G, dev()), tm=cfg,
                 dtype=torch.float32, lr=lr, top=top)
    rng = np.random.default_rng(5)
    lens = rng.integers(1, 4, size=(G, F, B)).astype(np.int32)
    vals = rng.integers(0, rows, size=int(lens.sum())).astype(np.int64)
    offs = np.concatenate([[0], np.cumsum(lens.reshape(-1))])
    kjts, labels = {}, {}
    yl = rng.integers(0, 2, size=(G, B)).astype(np.float32)
    for r in range(G):
        seg = vals[offs[r * F * B]:offs[(r + 1) * F * B]]
        kjts[r] = KJT(torch.from_numpy(lens[r].reshape(-1)).to(dev()), torch.from_numpy(seg.astype(np.int32)).to(dev()),
                      [int(lens[r, f].sum()) for f in range(F)], B)
        labels[r] = torch.from_numpy(yl[r]).to(dev())
    top_w0 = model.top.host_weights()
    losses = model.train_step_bce(kjts, labels)
    torch.cuda.synchronize()

    shards = [(s.table_id, s.rank, s.scheme, s.row_range, s.col_range) for s in placement.shards]
    flat, _, _, _ = oracle.baseline_forward(lens, vals, list(range(F)), pooling, before, shards,
                                            oracle.OTopo(hosts, rph))
    by_tower = {t: [f for f in range(F) if assignment[f] == t] for t in range(T)}
    tw = {t: oracle.init_tm_weights(ocfg, len(by_tower[t]), N, salt=t) for t in range(T)}
    O = model.plan.out_width()
    otw = oracle.init_tm_weights(otop, 1, O, salt=1_000_003)
    key = "w_proj" if top_kind == "dcn" else "w_feat"
    np.testing.assert_allclose(getattr(top_w0, key), otw[key], rtol=1e-6)
    grad_rows = {t: np.zeros_like(before[t]) for t in range(F)}
    scale = 1.0 / (G * B)
    top_grad_sum = None
    for r in range(G):
        col, ys, xs = 0, [], {}
        for t in range(T):
            fs = by_tower[t]
            xs[t] = flat[r][:, fs[0] * N:(fs[-1] + 1) * N].reshape(B, len(fs), N)
            ys.append(oracle.tm_forward(xs[t], ocfg, tw[t]))
        y = np.concatenate(ys, axis=1)
        z = oracle.tm_forward(y.reshape(B, 1, O), otop, otw)
        loss, dz = oracle.bce_with_logits(z, yl[r].reshape(B, 1), scale)
        assert abs(float(losses[r].item()) - loss) <= 1e-5 * max(1.0, abs(loss))
        gy, gw = oracle.tm_backward(y.reshape(B, 1, O), otop, otw, dz)
        gy = gy.reshape(B, O)
        top_grad_sum = gw[key] if top_grad_sum is None else top_grad_sum + gw[key]
        for t in range(T):
            fs = by_tower[t]
            ow_ = oracle.tm_output_width(ocfg, len(fs), N)
            dx, _ = oracle.tm_backward(xs[t], ocfg, tw[t], gy[:, col:col + ow_])
            col += ow_
            for i, f in enumerate(fs):
                base = (r * F + f) * B
                for b in range(B):
                    for k in range(offs[base + b], offs[base + b + 1]):
                        grad_rows[f][vals[k]] += dx[b, i]
    wt = model.top.host_weights()
    got_leaf = getattr(wt, key)
    want_leaf = otw[key] - lr * top_grad_sum
    assert max_rel_err(got_leaf - getattr(top_w0, key), want_leaf - otw[key]) <= 1e-5
    for sid, sh in enumerate(placement.shards):
        f = sh.table_id
        touched = np.unique(vals[np.concatenate([np.arange(offs[(r * F + f) * B], offs[(r * F + f + 1) * B])
                                                 for r in range(G)])])
        want = oracle.apply_sgd(before[f], touched, grad_rows[f][touched], lr)
        got = model.engine.weights[sid].double().cpu().numpy()
        (r0, r1), (c0, c1) = sh.row_range, sh.col_range
        _assert_sgd_rows(got, before[f][r0:r1, c0:c1], want[r0:r1, c0:c1], what=f"shard {sid}")


@pytest.mark.parametrize("scheme", ["table_wise", "row_wise"])
def test_train_api_check_indices(scheme):
    """SPTT(check_indices=True) raises TableLookupError for an index outside
    its table -- also for row-wise tables, where every shard filters the index
    (embedding.py:74-77); off by default (no host sync)."""
    import paper_2403_00877_b200 as P
    from paper_2403_00877_b200.fabric import LoopbackFabric
    from paper_2403_00877_b200.pipeline import KJT
    from paper_2403_00877_b200.sptt import SPTT, build_world

    F, rows, N, B = 4, 30, 8, 3
    topo, layout, placement, assignment = build_world(2, 2, 1, F, rows, N, seed=1, scheme=scheme,
                                                      shards_per_table=2)
    G = topo.world_size
    pooling = {f: "sum" for f in range(F)}
    kjts = {}
    for r in range(G):
        lens = np.full(F * B, 2, dtype=np.int32)
        vals = np.random.default_rng(r).integers(0, rows, size=2 * F * B).astype(np.int32)
        if r == 1:
            vals[5] = rows + 7  # out of range for its table
        kjts[r] = KJT(torch.from_numpy(lens).to(dev()), torch.from_numpy(vals).to(dev()), [2 * B] * F, B)
    ok = SPTT(topo, layout, placement, assignment, pooling, B, LoopbackFabric(G, dev()), dtype=torch.float32)
    ok.forward(kjts, save=False)  # unchecked: no error, no sync
    chk = SPTT(topo, layout, placement, assignment, pooling, B, LoopbackFabric(G, dev()), dtype=torch.float32,
               check_indices=True)
    with pytest.raises(P.TableLookupError):
        chk.forward(kjts, save=False)


def _ragged_world(hosts, rph, seed=3):
    from paper_2403_00877_b200.pipeline import KJT
    from paper_2403_00877_b200.sptt import build_world, powerlaw_lengths

    F, rows, N, B = 6, 80, 16, 32
    topo, layout, placement, assignment = build_world(hosts, rph, 1, F, rows, N, seed=seed)
    G = topo.world_size
    batches = []
    for i in range(4):
        kj = {}
        for r in range(G):
            lens = powerlaw_lengths(F, B, 1000 * i + r, mean=6.0, cap=40)
            vals = np.random.default_rng(7 * i + r).integers(0, rows, size=int(lens.sum())).astype(np.int32)
            kj[r] = KJT(torch.from_numpy(lens.reshape(-1)).to(dev()), torch.from_numpy(vals).to(dev()),
                        [int(x) for x in lens.sum(axis=1)], B)
        batches.append(kj)
    cap = [max(b[r].nnz_per_feature[f] for b in batches for r in range(G)) + 5 for f in range(F)]
    return topo, layout, placement, assignment, batches, cap, F, B


@pytest.mark.parametrize("hosts,rph", [(1, 1), (2, 2), (4, 1)])
def test_capacity_padded_ragged_steps_match_exact_counts(hosts, rph):
    """C5-style ragged batches: the capacity-padded step a (static splits, no
    count exchange) gives the same outputs and table updates, bit for bit, as
    the exact-count path; CUDA-graph replays of it equal eager steps bitwise."""
    import paper_2403_00877_b200 as P
    from paper_2403_00877_b200.fabric import LoopbackFabric
    from paper_2403_00877_b200.pipeline import KJT
    from paper_2403_00877_b200.sptt import SPTT

    cfg = P.TMConfig(kind="dcn", out_dim=4, cross_layers=2, seed=1)

    def model():
        topo, layout, placement, assignment, batches, cap, F, B = _ragged_world(hosts, rph)
        m = SPTT(topo, layout, placement, assignment, {f: "sum" for f in range(F)}, B,
                 LoopbackFabric(topo.world_size, dev()), tm=cfg, dtype=torch.float32, lr=0.5, dense_lr=1e-3)
        return m, batches, cap, B

    exact, batches, cap, B = model()
    padded, _, _, _ = model()
    padded.set_capacity(cap)
    G = len(batches[0])
    g = {r: torch.full((B, exact.out_width), 0.01, device=dev()) for r in range(G)}
    for bt in batches:
        oe = exact.train_step(bt, g)
        op = padded.train_step(bt, g)
        for r in range(G):
            assert torch.equal(oe[r], op[r])
    assert not padded.engine.capacity_overflowed()
    for sid, w in exact.engine.weights.items():
        assert torch.equal(w, padded.engine.weights[sid])
    # graph replay of the padded step == eager padded steps
    graph, _, _, _ = model()
    graph.set_capacity(cap)
    eager, _, _, _ = model()
    eager.set_capacity(cap)
    st = {r: KJT(batches[0][r].lengths.clone(), torch.zeros(sum(cap), dtype=torch.int32, device=dev()),
                 batches[0][r].nnz_per_feature, B) for r in range(G)}
    for r in range(G):
        st[r].values[: batches[0][r].values.numel()].copy_(batches[0][r].values)
    replay, outs = graph.capture(st, g, warmup=2)
    for _ in range(2):
        eager.train_step(batches[0], g)
    for i in (1, 2, 3):
        for r in range(G):
            st[r].lengths.copy_(batches[i][r].lengths)
            st[r].values[: batches[i][r].values.numel()].copy_(batches[i][r].values)
        replay()
        oe = eager.train_step(batches[i], g)
        torch.cuda.synchronize()
        for r in range(G):
            assert torch.equal(outs[r], oe[r]), (i, r)
    for sid, w in eager.engine.weights.items():
        assert torch.equal(w, graph.engine.weights[sid])
    # a feature over its capacity raises the device flag
    small, _, _, _ = model()
    small.set_capacity([1] * len(cap))
    small.forward(batches[0], save=False)
    assert small.engine.capacity_overflowed()


def test_capacity_padded_step_a_device_byte_counters():
    """With a capacity-padded step a the host only knows capacities; the
    CommTrace step-a bytes come from device counters (dmt_kjt_slot_offsets)
    and equal the exact-count path's trace (the reference's payload_nbytes)."""
    import paper_2403_00877_b200 as P
    from paper_2403_00877_b200.fabric import LoopbackFabric
    from paper_2403_00877_b200.sptt import SPTT

    topo, layout, placement, assignment, batches, cap, F, B = _ragged_world(2, 2)
    G = topo.world_size
    traces = []
    for padded in (False, True):
        tr = P.CommTrace(topo)
        m = SPTT(topo, layout, placement, assignment, {f: "sum" for f in range(F)}, B, LoopbackFabric(G, dev()),
                 dtype=torch.float32, trace=tr)
        if padded:
            m.set_capacity(cap)
        m.forward(batches[1], save=False)
        traces.append(tr)
    for label in ("a", "d", "f"):
        assert traces[0].byte_totals(label) == traces[1].byte_totals(label), label
    assert traces[0].sent_by_rank("a") == traces[1].sent_by_rank("a")
