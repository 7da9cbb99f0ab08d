"""Parity at the benchmarked configuration (BASELINE configs[1], C2).

The bench times the DCN tower module at full C2 size -- 8192 x 3328 x 3328
GEMMs (BN 256, ~5.6 persistent waves) at N=1 and 16384 x 1664 x 1664 (BN 192)
for the T=2 tower shape at N>1 -- and replays the whole train step from a CUDA
graph.  These tests check exactly those launches and that replay:

* every GEMM launch of one DCN step (crossnet fwd with the CROSS epilogue,
  projection, the DCN_BWD / DCN_FINAL backward epilogues, dW, and the fused
  SGD epilogue W -= lr * dW) at both shapes against float64 torch, with the
  element-wise error bound  |got - want| <= tol * (|A| |B|^T [+ epilogue
  magnitudes])  -- tol = 1e-2 (bf16) / 1e-5 (fp32, 3xTF32), the north star's;
* the tower module forward + backward at full C2 size against the oracle
  (oracle.tm_forward / oracle.tm_backward, float64 numpy) on the weights the
  device holds, max-norm relative error <= 1e-2 (bf16) / 1e-5 (fp32);
* CUDA-graph replays of the full train step against eager steps, bitwise, on
  a C2-scale slice (26 tables x 100k rows x 128, B = 8192, L = 20, DCN TM),
  and the first step against the oracle (pooled lookup -> TM -> backward ->
  embedding SGD), for bf16 and fp32 tables.
"""

from __future__ import annotations

import numpy as np
import pytest
import torch

from conftest import max_rel_err, oracle_tm_cfg, oracle_tm_weights

pytestmark = pytest.mark.gpu

import oracle  # noqa: E402

# rows, M = F * N (crossnet width), P = F * D (projection width)
SHAPES = {"n1_t1": (8192, 26 * 128, 26 * 64), "t2_tower": (16384, 13 * 128, 13 * 64)}
TOL = {torch.bfloat16: 1e-2, torch.float32: 1e-5}
DTS = [torch.bfloat16, torch.float32]
DT_IDS = ["bf16", "fp32"]


def dev():
    return torch.device("cuda")


def _mats(seed, *shapes, scale=1.0, dt=torch.float32):
    g = torch.Generator(device="cuda").manual_seed(seed)
    return [(torch.randn(*s, device="cuda", generator=g) * scale).to(dt) for s in shapes]


def _w(seed, rows, cols, dt):
    g = torch.Generator(device="cuda").manual_seed(seed)
    bound = 1.0 / cols ** 0.5
    return ((torch.rand(rows, cols, device="cuda", generator=g) * 2 - 1) * bound).to(dt)


def _check(got, want, bound, what):
    err = (got.double() - want).abs()
    bad = err > bound
    if bool(bad.any()):
        i = int(torch.argmax((err - bound).flatten()))
        raise AssertionError(f"{what}: {int(bad.sum())} elements over the bound; worst at {i}: err "
                             f"{float(err.flatten()[i]):.3e} bound {float(bound.flatten()[i]):.3e}")


def _absmm(a, b):
    return a.double().abs() @ b.double().abs().T


@pytest.mark.parametrize("dt", DTS, ids=DT_IDS)
@pytest.mark.parametrize("shape", list(SHAPES), ids=list(SHAPES))
def test_c2_gemm_crossnet_and_projection_forward(shape, dt):
    """u = xl W^T + b, x' = x0 * u + xl (CROSS epilogue) and y = x Wp^T + bp."""
    from paper_2403_00877_b200 import _lib as L
    from paper_2403_00877_b200 import kernels as K

    rows, M, P = SHAPES[shape]
    tol = TOL[dt]
    x0, xl = _mats(1, (rows, M), (rows, M), scale=0.5, dt=dt)
    W, Wp = _w(2, M, M, dt), _w(3, P, M, dt)
    b, bp = _mats(4, (M,), (P,), scale=0.1)
    out = torch.empty(rows, M, device="cuda", dtype=dt)
    u = torch.empty(rows, M, device="cuda", dtype=dt)
    K.gemm(xl, W, out, bias=b, epilogue=L.EPI_CROSS, x0=x0, xl=xl, aux=u)
    y = torch.empty(rows, P, device="cuda", dtype=dt)
    K.gemm(out, Wp, y, bias=bp, epilogue=L.EPI_BIAS)
    torch.cuda.synchronize()
    mag = _absmm(xl, W) + b.double().abs()
    uu = xl.double() @ W.double().T + b.double()
    _check(u, uu, tol * mag, "u")
    _check(out, x0.double() * uu + xl.double(), tol * (x0.double().abs() * mag + xl.double().abs()), "x_next")
    del mag, uu
    _check(y, out.double() @ Wp.double().T + bp.double(), tol * (_absmm(out, Wp) + bp.double().abs()), "y")


@pytest.mark.parametrize("dt", DTS, ids=DT_IDS)
@pytest.mark.parametrize("shape", list(SHAPES), ids=list(SHAPES))
def test_c2_gemm_dcn_backward_epilogues(shape, dt):
    """The three dX-side launches of the DCN backward (towermod._dcn_bwd):
    DCN_BWD from gy (dx0 written), DCN_BWD of a middle layer (C = g, dx0
    accumulated) and DCN_FINAL (dX = gu W0 + g + dx0)."""
    from paper_2403_00877_b200 import _lib as L
    from paper_2403_00877_b200 import kernels as K

    rows, M, P = SHAPES[shape]
    tol = TOL[dt]
    gy, = _mats(5, (rows, P), dt=dt)
    x0, u1, u0 = _mats(6, (rows, M), (rows, M), (rows, M), scale=0.5, dt=dt)
    Wp, W1, W0 = _w(7, P, M, dt), _w(8, M, M, dt), _w(9, M, M, dt)
    g = torch.empty(rows, M, device="cuda", dtype=dt)
    gu = [torch.empty(rows, M, device="cuda", dtype=dt) for _ in range(2)]
    dx0 = torch.empty(rows, M, device="cuda", dtype=torch.float32)
    # layer L: g = gy Wp ; gu = g * x0 ; dx0 = g * u
    K.gemm(gy, Wp, g, trans_b=True, epilogue=L.EPI_DCN_BWD, x0=x0, xl=u1, aux=gu[1], aux2=dx0, aux2_accum=False)
    torch.cuda.synchronize()
    mag = gy.double().abs() @ Wp.double().abs()
    want_g = gy.double() @ Wp.double()
    _check(g, want_g, tol * mag, "g_L")
    # gu and dx0 are formed from the fp32 accumulator (before g is rounded)
    x0d, u1d, u0d = x0.double(), u1.double(), u0.double()
    _check(gu[1], want_g * x0d, tol * mag * x0d.abs(), "gu_L")
    _check(dx0, want_g * u1d, tol * mag * u1d.abs(), "dx0_L")
    want_dx0 = want_g * u1d
    dx0_mag = mag * u1d.abs()
    g_prev, gu_prev = g.clone(), gu[1].clone()
    del want_g
    # middle layer: g' = gu W1 + g ; gu' = g' * x0 ; dx0 += g' * u0
    K.gemm(gu[1], W1, g, trans_b=True, epilogue=L.EPI_DCN_BWD, c=g, beta=1.0, x0=x0, xl=u0, aux=gu[0], aux2=dx0,
           aux2_accum=True)
    torch.cuda.synchronize()
    mag = gu_prev.double().abs() @ W1.double().abs() + g_prev.double().abs()
    want_g = gu_prev.double() @ W1.double() + g_prev.double()
    _check(g, want_g, tol * mag, "g_mid")
    _check(gu[0], want_g * x0d, tol * mag * x0d.abs(), "gu_mid")
    want_dx0 += want_g * u0d
    _check(dx0, want_dx0, tol * (dx0_mag + mag * u0d.abs()), "dx0_mid")
    del mag, want_g, dx0_mag
    # final layer: dX = gu W0 + g + dx0
    dx = torch.empty(rows, M, device="cuda", dtype=dt)
    K.gemm(gu[0], W0, dx, trans_b=True, epilogue=L.EPI_DCN_FINAL, c=g, beta=1.0, aux2=dx0)
    torch.cuda.synchronize()
    want = gu[0].double() @ W0.double() + g.double() + dx0.double()
    mag = gu[0].double().abs() @ W0.double().abs() + g.double().abs() + dx0.double().abs()
    _check(dx, want, tol * mag, "dX")


@pytest.mark.parametrize("dt", DTS, ids=DT_IDS)
@pytest.mark.parametrize("shape", list(SHAPES), ids=list(SHAPES))
def test_c2_gemm_weight_grads_and_fused_sgd(shape, dt):
    """dW = gu^T x (fp32 out, K = rows: the long-K launches), dWp = gy^T xL,
    and the fused SGD epilogue W -= lr * gu^T x (SCALE_ACC + ACC, the W = 1
    bench path) into a weight in the compute dtype."""
    from paper_2403_00877_b200 import _lib as L
    from paper_2403_00877_b200 import kernels as K

    rows, M, P = SHAPES[shape]
    tol = TOL[dt]
    gu, x = _mats(10, (rows, M), (rows, M), scale=0.5, dt=dt)
    gy, = _mats(11, (rows, P), dt=dt)
    dW = torch.empty(M, M, device="cuda", dtype=torch.float32)
    K.gemm(gu, x, dW, trans_a=True, trans_b=True)
    torch.cuda.synchronize()
    _check(dW, gu.double().T @ x.double(), tol * (gu.double().abs().T @ x.double().abs()), "dW")
    del dW
    dWp = torch.empty(P, M, device="cuda", dtype=torch.float32)
    K.gemm(gy, x, dWp, trans_a=True, trans_b=True)
    torch.cuda.synchronize()
    _check(dWp, gy.double().T @ x.double(), tol * (gy.double().abs().T @ x.double().abs()), "dWp")
    del dWp
    lr = 1e-3
    W = _w(12, M, M, dt)
    W0 = W.double().clone()
    K.gemm(gu, x, W, trans_a=True, trans_b=True, epilogue=L.EPI_ACC, beta=1.0, alpha=-lr)
    torch.cuda.synchronize()
    want = W0 - lr * (gu.double().T @ x.double())
    ulp = 2.0 ** -8 if dt == torch.bfloat16 else 2.0 ** -23  # rounding of the stored weight
    _check(W, want, ulp * want.abs() + tol * lr * (gu.double().abs().T @ x.double().abs()), "W fused SGD")


def _tower_module(dt, F, N, D=64, layers=3, seed=0):
    import paper_2403_00877_b200 as P

    cfg = P.TMConfig(kind="dcn", out_dim=D, cross_layers=layers, seed=seed)
    return P.TowerModule(cfg, F, N, P.init_tm_weights(cfg, F, N, salt=0), dtype=dt), cfg


@pytest.mark.parametrize("dt", DTS, ids=DT_IDS)
@pytest.mark.parametrize("shape", list(SHAPES), ids=list(SHAPES))
def test_c2_tower_module_fwd_bwd_vs_oracle(shape, dt):
    """Full-size DCN tower module (3 cross layers + projection, D = 64) forward
    and backward vs the oracle on the device's own (dtype-rounded) weights:
    Y, dX and every weight / bias gradient within the north-star tolerance
    (max-norm relative)."""
    rows, M, P = SHAPES[shape]
    F, N = M // 128, 128
    tm, cfg = _tower_module(dt, F, N)
    ocfg, ow = oracle_tm_cfg(cfg), oracle_tm_weights(tm)
    rng = np.random.default_rng(3)
    # pooled-sum-like activations: 20 rows of U(-1, 1)
    x = (rng.uniform(-1, 1, size=(rows, M)) * np.sqrt(20.0 / 3.0)).astype(np.float32)
    xt = torch.from_numpy(x).to(dev()).to(dt)
    x = xt.double().cpu().numpy()
    gy = (rng.normal(size=(rows, P)) * 1e-3).astype(np.float32)
    gyt = torch.from_numpy(gy).to(dev()).to(dt)
    gy = gyt.double().cpu().numpy()
    y = tm.forward(xt, save=True)
    dx = tm.backward(gyt)
    torch.cuda.synchronize()
    tol = TOL[dt]
    xo = x.reshape(rows, F, N)
    want_y = oracle.tm_forward(xo, ocfg, ow)
    assert max_rel_err(y.double().cpu().numpy(), want_y) <= tol, "Y"
    want_dx, want_dw = oracle.tm_backward(xo, ocfg, ow, gy)
    errs = {"dX": max_rel_err(dx.double().cpu().numpy().reshape(rows, F, N), want_dx)}
    pairs = [("w_proj", want_dw["w_proj"]), ("b_proj", want_dw["b_proj"])]
    for i, (gw, gb) in enumerate(want_dw["cross"]):
        pairs += [(f"w{i}", gw), (f"b{i}", gb)]
    for k, want in pairs:
        errs[k] = max_rel_err(tm.grads[k].double().cpu().numpy(), want)
    bad = {k: v for k, v in errs.items() if v > tol}
    assert not bad, (bad, errs)


@pytest.mark.parametrize("dt", DTS, ids=DT_IDS)
def test_c2_tower_module_fused_sgd_vs_oracle(dt):
    """The N=1 bench path: dW GEMM epilogues update W in place (fused_lr),
    biases by dmt_sgd_dense -- against oracle W - lr * dW."""
    rows, M, P = SHAPES["n1_t1"]
    F, N = 26, 128
    tm, cfg = _tower_module(dt, F, N, seed=4)
    ocfg, ow = oracle_tm_cfg(cfg), oracle_tm_weights(tm)
    rng = np.random.default_rng(5)
    xt = torch.from_numpy((rng.uniform(-1, 1, size=(rows, M)) * 2.5).astype(np.float32)).to(dev()).to(dt)
    gyt = torch.from_numpy((rng.normal(size=(rows, P)) * 1e-2).astype(np.float32)).to(dev()).to(dt)
    x, gy = xt.double().cpu().numpy().reshape(rows, F, N), gyt.double().cpu().numpy()
    lr = 0.05
    tm.forward(xt, save=True)
    tm.backward(gyt, fused_lr=lr)
    tm.sgd_step(lr)  # biases (the fused epilogue updated the matrices)
    torch.cuda.synchronize()
    _, want_dw = oracle.tm_backward(x, ocfg, ow, gy)
    got = oracle_tm_weights(tm)
    ulp = 2.0 ** -8 if dt == torch.bfloat16 else 2.0 ** -23
    tol = TOL[dt]
    names = [("w_proj", ow["w_proj"], want_dw["w_proj"], got["w_proj"])]
    for i in range(cfg.cross_layers):
        names.append((f"w{i}", ow["cross"][i][0], want_dw["cross"][i][0], got["cross"][i][0]))
        names.append((f"b{i}", ow["cross"][i][1], want_dw["cross"][i][1], got["cross"][i][1]))
    for name, w0, dw, w1 in names:
        want = w0 - lr * dw
        err = np.abs(w1 - want)
        bound = ulp * np.abs(want) + tol * lr * np.abs(dw).max()
        assert (err <= bound).all(), (name, float((err - bound).max()))


# --------------------------------------------------------------------------- #
# the timed path: CUDA-graph replay of the full train step
# --------------------------------------------------------------------------- #
C2S = dict(F=26, rows=100_000, N=128, B=8192, L=20, D=64, layers=3)


def _c2_slice_model(dt, lr, dense_lr=1e-4):
    import paper_2403_00877_b200 as P
    from paper_2403_00877_b200.fabric import LoopbackFabric
    from paper_2403_00877_b200.sptt import SPTT, device_world

    c = C2S
    topo, layout, placement, assignment = device_world(1, 1, 1, c["F"], c["rows"], c["N"], dt, [0], seed=0,
                                                       device=dev())
    cfg = P.TMConfig(kind="dcn", out_dim=c["D"], cross_layers=c["layers"], per_feature_outputs=1, flat_outputs=0,
                     seed=0)
    model = SPTT(topo, layout, placement, assignment, {f: "sum" for f in range(c["F"])}, c["B"],
                 LoopbackFabric(1, dev()), tm=cfg, dtype=dt, device=dev(), lr=lr, dense_lr=dense_lr)
    model.engine.uniform_nnz = True  # the captured step's step-a path, eager too
    return model, cfg


def _batches(n, dt, width):
    from paper_2403_00877_b200.sptt import random_kjt

    c = C2S
    gen = torch.Generator(device="cuda").manual_seed(77)
    kj = [random_kjt(c["F"], c["B"], c["rows"], c["L"], gen, dev()) for _ in range(n)]
    gy = [(torch.randn(c["B"], width, generator=gen, device="cuda") * 1e-3).to(dt) for _ in range(n)]
    return kj, gy


@pytest.mark.parametrize("dt", DTS, ids=DT_IDS)
def test_c2_slice_graph_replay_bitwise_equals_eager_and_oracle(dt):
    """SPTT.capture -> replay (the bench's timed path) vs eager train steps,
    bitwise: outputs of 3 replays, then every table shard and TM weight.  The
    first eager step is also checked against the oracle (C2 slice, L = 20,
    B = 8192): outputs and the SGD-updated table rows."""
    from paper_2403_00877_b200.pipeline import KJT

    # sparse lr 1 (table updates ~1e-2, far above the fp32 storage ulp) and
    # dense lr 1e-4: a dW GEMM sums 8192 rows, so a shared lr large enough to
    # move the tables measurably would move the DCN weights by many times
    # their own size and the model would reach inf within 3 steps
    lr = 1.0
    c = C2S
    eager, cfg = _c2_slice_model(dt, lr)
    kj, gy = _batches(4, dt, eager.out_width)
    tables0 = {sid: w.double().cpu().numpy() for sid, w in eager.engine.weights.items()}
    tm0 = oracle_tm_weights(eager.tms[0])

    # ---- eager step 1 vs the oracle --------------------------------------
    outs = eager.train_step({0: kj[0]}, {0: gy[0]})
    torch.cuda.synchronize()
    y1 = outs[0].double().cpu().numpy()
    tol = TOL[dt]
    lens = np.full(c["B"], c["L"], dtype=np.int64)
    vals = kj[0].values.cpu().numpy().astype(np.int64).reshape(c["F"], c["B"] * c["L"])
    sid_of = {eager.placement.shards[s].table_id: s for s in eager.engine.weights}
    x = np.stack([oracle.pool(tables0[sid_of[f]], lens, vals[f], "sum", acc_dtype=np.float64)
                  for f in range(c["F"])], axis=1)  # (B, F, N)
    if dt == torch.bfloat16:  # the device pools in fp32 and stores the TM input in bf16
        x = oracle.bf16_round(x.astype(np.float32)).astype(np.float64)
    ocfg = oracle_tm_cfg(cfg)
    want_y = oracle.tm_forward(x, ocfg, tm0)
    assert max_rel_err(y1, want_y) <= tol, ("outputs", max_rel_err(y1, want_y))
    dx, _ = oracle.tm_backward(x, ocfg, tm0, gy[0].double().cpu().numpy())
    ulp = 2.0 ** -8 if dt == torch.bfloat16 else 2.0 ** -23
    for f in range(c["F"]):
        sid = sid_of[f]
        uniq, g = oracle.embedding_row_grads(c["rows"], lens, vals[f], dx[:, f, :])
        want = oracle.apply_sgd(tables0[sid], uniq, g, lr)
        got = eager.engine.weights[sid].double().cpu().numpy()
        delta = np.abs(lr * g).max()
        bound = ulp * np.abs(want) + tol * delta
        err = np.abs(got - want)
        assert (err <= bound).all(), (f, float((err - bound).max()), delta)
        untouched = np.setdiff1d(np.arange(c["rows"]), uniq)
        assert np.array_equal(got[untouched], tables0[sid][untouched])

    # ---- graph replay vs eager, bitwise -----------------------------------
    graph, _ = _c2_slice_model(dt, lr)
    # bring both to the same state: the graph model's capture() runs 2 eager
    # warm-up steps on the static batch (kj[0]) -- give eager the second one
    eager.train_step({0: kj[0]}, {0: gy[0]})
    st = {0: KJT(kj[0].lengths.clone(), kj[0].values.clone(), kj[0].nnz_per_feature, c["B"])}
    g_static = {0: gy[0].clone()}
    replay, g_outs = graph.capture(st, g_static, warmup=2)
    for i in (1, 2, 3):
        st[0].lengths.copy_(kj[i].lengths)
        st[0].values.copy_(kj[i].values)
        g_static[0].copy_(gy[i])
        replay()
        e_out = eager.train_step({0: kj[i]}, {0: gy[i]})
        torch.cuda.synchronize()
        assert torch.equal(g_outs[0], e_out[0]), f"replay {i}: outputs differ from the eager step"
    for sid, w in eager.engine.weights.items():
        assert torch.equal(graph.engine.weights[sid], w), f"shard {sid} differs after 3 replays"
    for k, w in eager.tms[0].w.items():
        assert torch.equal(graph.tms[0].w[k], w), f"TM weight {k} differs after 3 replays"
