"""Bisect the graph-vs-eager mismatch: single GEMM, tower module forward, full forward."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import torch
from paper_2403_00877_b200 import _lib as L, kernels as K
import paper_2403_00877_b200 as P

dt = torch.bfloat16
dev = torch.device("cuda")
g = torch.Generator(device="cuda").manual_seed(0)


def graphed(fn):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fn()
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr):
        out = fn()
    return gr, out


# C: single CROSS gemm
rows, M = 8192, 3328
x0 = torch.randn(rows, M, device=dev, generator=g).to(dt)
W = (torch.randn(M, M, device=dev, generator=g) / M ** 0.5).to(dt)
b = torch.randn(M, device=dev, generator=g)
o_e = torch.empty(rows, M, device=dev, dtype=dt)
K.gemm(x0, W, o_e, bias=b, epilogue=L.EPI_CROSS, x0=x0, xl=x0)


def f1():
    o = torch.empty(rows, M, device=dev, dtype=dt)
    K.gemm(x0, W, o, bias=b, epilogue=L.EPI_CROSS, x0=x0, xl=x0)
    return o


gr, o_g = graphed(f1)
gr.replay()
torch.cuda.synchronize()
print("C single cross gemm graph==eager:", torch.equal(o_g, o_e), flush=True)

# B: tower module forward
cfg = P.TMConfig(kind="dcn", out_dim=64, cross_layers=3, seed=0)
tm = P.TowerModule(cfg, 26, 128, P.init_tm_weights(cfg, 26, 128), dtype=dt)
X = (torch.rand(rows, M, device=dev, generator=g) * 5 - 2.5).to(dt)
Y = torch.empty(rows, 26 * 64, device=dev, dtype=dt)
ye = tm.forward(X, save=True).clone()
gr, _ = graphed(lambda: tm.forward(X, save=True, out=Y))
gr.replay()
torch.cuda.synchronize()
print("B tm forward graph==eager:", torch.equal(Y, ye), flush=True)
# B2: tm forward + backward (no SGD)
gy = (torch.randn(rows, 26 * 64, device=dev, generator=g) * 0.05).to(dt)
tm.forward(X, save=True)
dxe = tm.backward(gy).clone()
ge = {k: v.clone() for k, v in tm.grads.items()}


def fb():
    tm.forward(X, save=True, out=Y)
    return tm.backward(gy)


gr, dxg = graphed(fb)
gr.replay()
torch.cuda.synchronize()
print("B2 tm fwd+bwd graph==eager: dX", torch.equal(dxg, dxe), "grads",
      {k: torch.equal(tm.grads[k], ge[k]) for k in ge}, flush=True)
# B3: fused sgd: two identical modules
tmA = P.TowerModule(cfg, 26, 128, P.init_tm_weights(cfg, 26, 128), dtype=dt)
tmB = P.TowerModule(cfg, 26, 128, P.init_tm_weights(cfg, 26, 128), dtype=dt)


def fbs(t):
    t.forward(X, save=True, out=Y)
    t.backward(gy, fused_lr=0.05)
    t.sgd_step(0.05)


fbs(tmA); fbs(tmA); fbs(tmA)  # 3 eager
gr, _ = graphed(lambda: fbs(tmB))  # 1 eager warmup inside graphed
gr.replay(); gr.replay()
torch.cuda.synchronize()
print("B3 tm fused-sgd 3 steps graph==eager:", {k: torch.equal(tmA.w[k], tmB.w[k]) for k in tmA.w}, flush=True)

# A: full engine forward only
from test_gpu_c2_parity import _c2_slice_model, _batches
from paper_2403_00877_b200.pipeline import KJT
m, _ = _c2_slice_model(dt, 0.05)
kj, gys = _batches(2, dt, m.out_width)
st = {0: KJT(kj[0].lengths.clone(), kj[0].values.clone(), kj[0].nnz_per_feature, 8192)}
oe = m.engine.forward({0: kj[0]}, save=True)[0].clone()
gr, og = graphed(lambda: m.engine.forward(st, save=True))
gr.replay()
torch.cuda.synchronize()
print("A engine forward graph==eager:", torch.equal(og[0], oe), flush=True)
