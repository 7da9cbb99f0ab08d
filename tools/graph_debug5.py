"""Which tensor of the captured step first goes NaN?"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import torch
from test_gpu_c2_parity import _c2_slice_model, _batches, C2S
from paper_2403_00877_b200.pipeline import KJT

dt = torch.bfloat16
c = C2S
variant = sys.argv[1]
graph, _ = _c2_slice_model(dt, 0.05)
kj, gy = _batches(1, dt, graph.out_width)
st = {0: KJT(kj[0].lengths.clone(), kj[0].values.clone(), kj[0].nnz_per_feature, c["B"])}
g_static = {0: gy[0].clone()}
nan = lambda t: int(t.float().isnan().sum())
if variant == "fwd":
    s = torch.cuda.Stream(); s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        graph.engine.forward(st, save=False)
    torch.cuda.current_stream().wait_stream(s); torch.cuda.synchronize()
    ye = graph.engine.buf[0]["Y"].clone()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr):
        graph.engine.forward(st, save=False)
    graph.engine.buf[0]["Y"].zero_()
    gr.replay(); torch.cuda.synchronize()
    print("fwd-only graph: Y==eager", torch.equal(graph.engine.buf[0]["Y"], ye), "nan", nan(graph.engine.buf[0]["Y"]), flush=True)
    sys.exit()
replay, g_outs = graph.capture(st, g_static, warmup=2)
torch.cuda.synchronize()
print("before replay: X nan", nan(graph.engine.buf[0]["X"]), "Y nan", nan(graph.engine.buf[0]["Y"]),
      "w nan", {k: nan(v) for k, v in graph.tms[0].w.items()}, flush=True)
xs, us = graph.tms[0]._saved
print("saved ptrs xs", [hex(t.data_ptr()) for t in xs], "us", [hex(t.data_ptr()) for t in us],
      "X", hex(graph.engine.buf[0]["X"].data_ptr()), "Y", hex(graph.engine.buf[0]["Y"].data_ptr()), flush=True)
replay(); torch.cuda.synchronize()
print("after replay: X nan", nan(graph.engine.buf[0]["X"]), "xs nan", [nan(t) for t in xs], "us nan", [nan(t) for t in us],
      "Y nan", nan(graph.engine.buf[0]["Y"]), "w nan", {k: nan(v) for k, v in graph.tms[0].w.items()}, flush=True)
print("absmax xs", [float(t.float().abs().max()) for t in xs], "us", [float(t.float().abs().max()) for t in us], flush=True)
