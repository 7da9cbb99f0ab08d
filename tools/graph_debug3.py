"""Bisect the graph-vs-eager mismatch of the full train step (C2 slice)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import torch
from test_gpu_c2_parity import _c2_slice_model, _batches, C2S
from paper_2403_00877_b200.pipeline import KJT, SpttEngine

dt = torch.bfloat16
variant = sys.argv[1] if len(sys.argv) > 1 else "none"
if variant in ("inline_side", "both"):
    SpttEngine._side_stream = lambda self: torch.cuda.current_stream()
    SpttEngine._side_stream2 = lambda self: torch.cuda.current_stream()
if variant in ("no_prepare", "both"):
    import paper_2403_00877_b200.pipeline as PL
    orig = PL.K.pooled_lookup_bwd_prepare
    def fwd_no_prep(self, kjts, save=False, check_indices=False, _o=SpttEngine.forward):
        out = _o(self, kjts, save=False, check_indices=check_indices)
        return out
    # keep save semantics for the TM but skip the prepare: patch the kernel wrapper
    PL.K.pooled_lookup_bwd_prepare = lambda *a, **k: None
    _orig_upd = SpttEngine._embedding_update
    def upd(self, lr, opt, eps):
        self._prepared = {}
        return _orig_upd(self, lr, opt, eps)
    SpttEngine._embedding_update = upd
c = C2S
eager, _ = _c2_slice_model(dt, 0.05)
graph, _ = _c2_slice_model(dt, 0.05)
kj, gy = _batches(3, dt, eager.out_width)
eager.train_step({0: kj[0]}, {0: gy[0]})
eager.train_step({0: kj[0]}, {0: gy[0]})
st = {0: KJT(kj[0].lengths.clone(), kj[0].values.clone(), kj[0].nnz_per_feature, c["B"])}
g_static = {0: gy[0].clone()}
replay, g_outs = graph.capture(st, g_static, warmup=2)
torch.cuda.synchronize()
same = all(torch.equal(graph.engine.weights[s], eager.engine.weights[s]) for s in eager.engine.weights)
print(variant, "state equal before replay:", same, flush=True)
# replay the SAME batch as the static one (no copies)
replay()
e_out = eager.train_step({0: kj[0]}, {0: gy[0]})
torch.cuda.synchronize()
print(variant, "replay(static batch): X", torch.equal(graph.engine.buf[0]["X"], eager.engine.buf[0]["X"]),
      "Y", torch.equal(graph.engine.buf[0]["Y"], eager.engine.buf[0]["Y"]),
      "tables", all(torch.equal(graph.engine.weights[s], eager.engine.weights[s]) for s in eager.engine.weights),
      "tm", {k: torch.equal(graph.tms[0].w[k], eager.tms[0].w[k]) for k in eager.tms[0].w}, flush=True)
yg, ye = graph.engine.buf[0]["Y"].float(), eager.engine.buf[0]["Y"].float()
d = (yg - ye).abs()
print("  Y maxdiff", float(d.max()), "count", int((d > 0).sum()), "nan", int(yg.isnan().sum()), flush=True)
