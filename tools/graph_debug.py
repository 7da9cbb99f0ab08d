"""Graph replay vs eager on the C2 slice: find the first diverging state."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import torch
from test_gpu_c2_parity import _c2_slice_model, _batches, C2S
from paper_2403_00877_b200.pipeline import KJT

dt = torch.float32 if "fp32" in sys.argv else torch.bfloat16
c = C2S
eager, _ = _c2_slice_model(dt, 0.05)
graph, _ = _c2_slice_model(dt, 0.05)
kj, gy = _batches(4, dt, eager.out_width)


def cmp(tag):
    torch.cuda.synchronize()
    bad = [sid for sid, w in eager.engine.weights.items() if not torch.equal(graph.engine.weights[sid], w)]
    badtm = [k for k, w in eager.tms[0].w.items() if not torch.equal(graph.tms[0].w[k], w)]
    print(tag, "tables differ:", bad[:5], len(bad), "tm differ:", badtm, flush=True)


cmp("init")
# eager determinism: two eager models, same steps
e2, _ = _c2_slice_model(dt, 0.05)
for m in (eager, e2):
    m.train_step({0: kj[0]}, {0: gy[0]})
torch.cuda.synchronize()
print("eager vs eager after 1 step:", all(torch.equal(eager.engine.weights[s], e2.engine.weights[s]) for s in eager.engine.weights),
      all(torch.equal(eager.tms[0].w[k], e2.tms[0].w[k]) for k in eager.tms[0].w), flush=True)
del e2
eager.train_step({0: kj[0]}, {0: gy[0]})
st = {0: KJT(kj[0].lengths.clone(), kj[0].values.clone(), kj[0].nnz_per_feature, c["B"])}
g_static = {0: gy[0].clone()}
replay, g_outs = graph.capture(st, g_static, warmup=2)
cmp("after capture (2 warmups each)")
for i in (1, 2):
    st[0].lengths.copy_(kj[i].lengths)
    st[0].values.copy_(kj[i].values)
    g_static[0].copy_(gy[i])
    replay()
    e_out = eager.train_step({0: kj[i]}, {0: gy[i]})
    torch.cuda.synchronize()
    bx = graph.engine.buf[0]["X"]; ex = eager.engine.buf[0]["X"]
    print(i, "X equal", torch.equal(bx, ex), "Y equal", torch.equal(graph.engine.buf[0]["Y"], eager.engine.buf[0]["Y"]),
          "out equal", torch.equal(g_outs[0], e_out[0]), flush=True)
    if not torch.equal(bx, ex):
        d = (bx.float() - ex.float()).abs()
        nz = d.nonzero()
        print("  X diff count", nz.shape[0], "first", nz[:5].tolist(), "max", float(d.max()), flush=True)
    cmp(f"after replay {i}")
