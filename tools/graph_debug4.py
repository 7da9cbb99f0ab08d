"""Is graph memory clobbered by allocations made after capture?"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import torch
from test_gpu_c2_parity import _c2_slice_model, _batches, C2S
from paper_2403_00877_b200.pipeline import KJT

dt = torch.bfloat16
c = C2S
eager, _ = _c2_slice_model(dt, 0.05)
kj, gy = _batches(3, dt, eager.out_width)
for _ in range(3):
    eager.train_step({0: kj[0]}, {0: gy[0]})
torch.cuda.synchronize()
Y3 = eager.engine.buf[0]["Y"].clone()
W3 = {s: w.clone() for s, w in eager.engine.weights.items()}
eager.train_step({0: kj[0]}, {0: gy[0]})
torch.cuda.synchronize()
Y4 = eager.engine.buf[0]["Y"].clone()
del eager
torch.cuda.empty_cache()
graph, _ = _c2_slice_model(dt, 0.05)
st = {0: KJT(kj[0].lengths.clone(), kj[0].values.clone(), kj[0].nnz_per_feature, c["B"])}
g_static = {0: gy[0].clone()}
replay, g_outs = graph.capture(st, g_static, warmup=2)
replay()
torch.cuda.synchronize()
print("immediate replay: Y==Y3", torch.equal(graph.engine.buf[0]["Y"], Y3), "nan", int(graph.engine.buf[0]["Y"].float().isnan().sum()),
      "tables==W3", all(torch.equal(graph.engine.weights[s], W3[s]) for s in W3), flush=True)
junk = torch.full((1 << 28,), float("nan"), device="cuda")
del junk
replay()
torch.cuda.synchronize()
print("after junk alloc: Y==Y4", torch.equal(graph.engine.buf[0]["Y"], Y4), "nan", int(graph.engine.buf[0]["Y"].float().isnan().sum()), flush=True)
