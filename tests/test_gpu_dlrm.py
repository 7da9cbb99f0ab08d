"""The C3 model: DLRM (bottom MLP, pairwise dot interaction, top MLP, BCE)
around SPTT, on the GPU vs the float64 restatement in oracle/dlrm.py
(the reference has no dense model -- parity unpinned,
north-star tolerances: fp32 1e-5 / bf16 1e-2, max-norm relative)."""

from __future__ import annotations

import numpy as np
import pytest
import torch

from conftest import max_rel_err

pytestmark = pytest.mark.gpu

import oracle  # noqa: E402

TOL = {torch.float32: 1e-5, torch.bfloat16: 1e-2}


def dev():
    return torch.device("cuda")


@pytest.mark.parametrize("dt", [torch.float32, torch.bfloat16])
@pytest.mark.parametrize("B,F,D", [(300, 26, 64), (7, 3, 8), (64, 13, 128), (5, 0, 16)])
def test_dot_interaction_vs_oracle(dt, B, F, D):
    from paper_2403_00877_b200 import kernels as K

    rng = np.random.default_rng(B + F + D)
    dense = torch.from_numpy(rng.normal(size=(B, D))).to(dev(), dt)
    sparse = torch.from_numpy(rng.normal(size=(B, max(F, 1) * D))).to(dev(), dt)[:, :F * D] if F else \
        torch.zeros((B, D), device=dev(), dtype=dt)
    z = K.dot_interaction_fwd(dense, sparse, F)
    dn, sp = dense.double().cpu().numpy(), sparse.double().cpu().numpy()
    want = oracle.interaction_forward(dn, sp[:, :F * D], F)
    assert z.shape == want.shape
    assert max_rel_err(z.double().cpu().numpy(), want) <= TOL[dt]
    gz = torch.from_numpy(rng.normal(size=want.shape)).to(dev(), dt)
    dd, ds = K.dot_interaction_bwd(gz, dense, sparse, F)
    wd, ws = oracle.interaction_backward(gz.double().cpu().numpy(), dn, sp[:, :F * D], F)
    assert max_rel_err(dd.double().cpu().numpy(), wd) <= TOL[dt]
    if F:
        assert max_rel_err(ds.double().cpu().numpy(), ws) <= TOL[dt]


@pytest.mark.parametrize("dt", [torch.float32, torch.bfloat16])
def test_relu_epilogues_vs_fp64(dt):
    """EPI_BIAS_RELU (forward) and EPI_RELU_BWD (dX masked by the previous
    layer's ReLU output) vs float64."""
    from paper_2403_00877_b200 import _lib as L
    from paper_2403_00877_b200 import kernels as K

    g = torch.Generator(device="cuda").manual_seed(3)
    m, n, k = 1000, 512, 416
    x = torch.randn(m, k, device="cuda", generator=g).to(dt)
    w = (torch.randn(n, k, device="cuda", generator=g) / k ** 0.5).to(dt)
    b = torch.randn(n, device="cuda", generator=g)
    y = torch.empty(m, n, device="cuda", dtype=dt)
    K.gemm(x, w, y, bias=b, epilogue=L.EPI_BIAS_RELU)
    want = torch.clamp(x.double() @ w.double().T + b.double(), min=0)
    mag = x.double().abs() @ w.double().abs().T + b.double().abs()
    assert ((y.double() - want).abs() <= TOL[dt] * mag).all()
    dz = torch.randn(m, n, device="cuda", generator=g).to(dt)
    mask_src = torch.randn(m, k, device="cuda", generator=g).to(dt)
    dx = torch.empty(m, k, device="cuda", dtype=dt)
    K.gemm(dz, w, dx, trans_b=True, epilogue=L.EPI_RELU_BWD, x0=mask_src)
    want = (dz.double() @ w.double()) * (mask_src.double() > 0)
    mag = dz.double().abs() @ w.double().abs()
    assert ((dx.double() - want).abs() <= TOL[dt] * mag).all()
    assert (dx[mask_src <= 0] == 0).all()


@pytest.mark.parametrize("dt", [torch.float32, torch.bfloat16])
def test_mlp_forward_backward_vs_oracle(dt):
    from paper_2403_00877_b200.dlrm import MLP

    rng = np.random.default_rng(5)
    B, widths = 384, [13, 512, 256, 64]
    mlp = MLP(widths, True, dt, dev(), seed=9)
    x = torch.from_numpy(rng.normal(size=(B, 13))).to(dev(), dt)
    layers = mlp.host_weights()
    y = mlp.forward(x)
    want, xs = oracle.mlp_forward(x.double().cpu().numpy(), layers, True)
    assert max_rel_err(y.double().cpu().numpy(), want) <= TOL[dt]
    dy = torch.from_numpy(rng.normal(size=(B, 64))).to(dev(), dt)
    # the backward is checked on the activations the device saved: a ReLU
    # pre-activation within rounding of 0 may take the other branch in bf16
    dev_xs = [t.double().cpu().numpy() for t in mlp._saved]
    dx = mlp.backward(dy, need_dx=True)
    wdx, wg = oracle.mlp_backward(dev_xs, layers, True, dy.double().cpu().numpy())
    assert max_rel_err(dx.double().cpu().numpy(), wdx) <= TOL[dt]
    for l, (gw, gb) in enumerate(wg):
        assert max_rel_err(mlp.grads[f"w{l}"].double().cpu().numpy(), gw) <= TOL[dt], l
        assert max_rel_err(mlp.grads[f"b{l}"].double().cpu().numpy(), gb) <= TOL[dt], l


@pytest.mark.parametrize("hosts,rph", [(2, 2), (1, 1), (2, 1)])
def test_dlrm_train_step_loopback_vs_oracle(hosts, rph):
    """Full C3-style step on simulated ranks (fp32): loss, every dense-arch
    weight after the world-all-reduced SGD, and every embedding row after SGD
    vs the float64 restatement (SPTT forward -> oracle DLRM step -> DLRM tower
    module backward -> embedding SGD)."""
    import paper_2403_00877_b200 as P
    from paper_2403_00877_b200.dlrm import DLRM
    from paper_2403_00877_b200.fabric import LoopbackFabric
    from paper_2403_00877_b200.pipeline import KJT
    from paper_2403_00877_b200.sptt import SPTT, build_world

    F, rows, N, B, D, d_in = 6, 40, 16, 4, 8, 5
    topo, layout, placement, assignment = build_world(hosts, rph, 1, F, rows, N, seed=6)
    G, T = topo.world_size, layout.num_towers
    pooling = {f: "sum" for f in range(F)}
    cfg = P.TMConfig(kind="dlrm", out_dim=D, per_feature_outputs=1, flat_outputs=0, seed=2)
    ocfg = {"kind": "dlrm", "out_dim": D, "per_feature_outputs": 1, "flat_outputs": 0, "cross_layers": 3, "seed": 2}
    before = {t: placement.tables[t].values.astype(np.float64).copy() for t in range(F)}
    lr, dlr = 0.5, 0.05
    sptt = SPTT(topo, layout, placement, assignment, pooling, B, LoopbackFabric(G, dev()), tm=cfg,
                dtype=torch.float32, lr=lr, dense_lr=dlr)
    model = DLRM(sptt, d_in, bottom=(16,), top=(32, 16), seed=4)
    bot0, top0 = model.bottom.host_weights(), model.top.host_weights()
    rng = np.random.default_rng(8)
    lens = rng.integers(1, 4, size=(G, F, B)).astype(np.int32)
    vals = rng.integers(0, rows, size=int(lens.sum())).astype(np.int64)
    offs = np.concatenate([[0], np.cumsum(lens.reshape(-1))])
    dx = rng.normal(size=(G, B, d_in)).astype(np.float32)
    yl = rng.integers(0, 2, size=(G, B)).astype(np.float32)
    kjts, dense_x, labels = {}, {}, {}
    for r in range(G):
        seg = vals[offs[r * F * B]:offs[(r + 1) * F * B]]
        kjts[r] = KJT(torch.from_numpy(lens[r].reshape(-1)).to(dev()), torch.from_numpy(seg.astype(np.int32)).to(dev()),
                      [int(lens[r, f].sum()) for f in range(F)], B)
        dense_x[r] = torch.from_numpy(dx[r]).to(dev())
        labels[r] = torch.from_numpy(yl[r]).to(dev())
    losses = model.train_step(kjts, dense_x, labels)
    torch.cuda.synchronize()

    shards = [(s.table_id, s.rank, s.scheme, s.row_range, s.col_range) for s in placement.shards]
    flat, _, _, _ = oracle.baseline_forward(lens, vals, list(range(F)), pooling, before, shards,
                                            oracle.OTopo(hosts, rph))
    by_tower = {t: [f for f in range(F) if assignment[f] == t] for t in range(T)}
    tw = {t: oracle.init_tm_weights(ocfg, len(by_tower[t]), N, salt=t) for t in range(T)}
    scale = 1.0 / (G * B)
    grad_rows = {t: np.zeros_like(before[t]) for t in range(F)}
    bot_acc = top_acc = None
    for r in range(G):
        xs, embs = {}, []
        for t in range(T):
            fs = by_tower[t]
            xs[t] = flat[r][:, fs[0] * N:(fs[-1] + 1) * N].reshape(B, len(fs), N)
            embs.append(oracle.tm_forward(xs[t], ocfg, tw[t]))
        emb = np.concatenate(embs, axis=1)
        loss, demb, bg, tg = oracle.dlrm_step(dx[r].astype(np.float64), emb, yl[r], bot0, top0, F, scale)
        assert abs(float(losses[r].item()) - loss) <= 1e-5 * max(1.0, abs(loss))
        bot_acc = bg if bot_acc is None else [(a + c, b + d) for (a, b), (c, d) in zip(bot_acc, bg)]
        top_acc = tg if top_acc is None else [(a + c, b + d) for (a, b), (c, d) in zip(top_acc, tg)]
        col = 0
        for t in range(T):
            fs = by_tower[t]
            ow = oracle.tm_output_width(ocfg, len(fs), N)
            dxt, _ = oracle.tm_backward(xs[t], ocfg, tw[t], demb[:, col:col + ow])
            col += ow
            for i, f in enumerate(fs):
                base = (r * F + f) * B
                for b in range(B):
                    for k in range(offs[base + b], offs[base + b + 1]):
                        grad_rows[f][vals[k]] += dxt[b, i]
    def check_sgd(got, w, g):  # update within 1e-5 (max-norm) + the fp32 storage rounding
        want = w - dlr * g
        bound = 1e-5 * np.abs(dlr * g).max() + 2.0 ** -24 * np.abs(want)
        assert (np.abs(got - want) <= bound).all(), float((np.abs(got - want) - bound).max())

    for got, w0, acc in ((model.bottom.host_weights(), bot0, bot_acc), (model.top.host_weights(), top0, top_acc)):
        for (gw, gb), (w, b), (aw, ab) in zip(got, w0, acc):
            check_sgd(gw, w, aw)
            check_sgd(gb, b, ab)
    for sid, sh in enumerate(placement.shards):
        f = sh.table_id
        touched = np.unique(vals[np.concatenate([np.arange(offs[(r * F + f) * B], offs[(r * F + f + 1) * B])
                                                 for r in range(G)])])
        want = oracle.apply_sgd(before[f], touched, grad_rows[f][touched], lr)
        got = sptt.engine.weights[sid].double().cpu().numpy()
        (r0, r1), (c0, c1) = sh.row_range, sh.col_range
        d_want = want[r0:r1, c0:c1] - before[f][r0:r1, c0:c1]
        assert np.abs(got - want[r0:r1, c0:c1]).max() <= 1e-5 * np.abs(d_want).max() + 2 ** -23 * np.abs(want).max()
