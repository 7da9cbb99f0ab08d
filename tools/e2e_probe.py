"""Diagnose the e2e loop: per-step device time of H2D, D2D staging copy and the
graph replay (run on a B200)."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2403_00877_b200 as P  # noqa: E402
from paper_2403_00877_b200.fabric import LoopbackFabric  # noqa: E402
from paper_2403_00877_b200.pipeline import KJT  # noqa: E402
from paper_2403_00877_b200.sptt import SPTT, device_world, random_kjt  # noqa: E402

dev = torch.device("cuda", 0)
torch.cuda.set_device(0)
F, B, R, N, L = 26, 8192, 1_000_000, 128, 20
topo, layout, placement, assignment = device_world(1, 1, 1, F, R, N, torch.bfloat16, [0], device=dev)
cfg = P.TMConfig(kind="dcn", out_dim=64, cross_layers=3)
m = SPTT(topo, layout, placement, assignment, {f: "sum" for f in range(F)}, B, LoopbackFabric(1, dev), tm=cfg,
         dtype=torch.bfloat16, device=dev, lr=1e-3)
gen = torch.Generator(device=dev).manual_seed(0)
kj = random_kjt(F, B, R, L, gen, dev)
gout = {0: (torch.randn(B, m.out_width, device=dev, generator=gen) * 1e-3).to(torch.bfloat16)}
st = {0: KJT(kj.lengths.clone(), kj.values.clone(), kj.nnz_per_feature, B)}
replay, outs = m.capture(st, gout)
hl, hv = kj.lengths.cpu().pin_memory(), kj.values.cpu().pin_memory()
print("pinned:", hl.is_pinned(), hv.is_pinned())
ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
for it in range(5):
    ev[0].record()
    st[0].lengths.copy_(hl, non_blocking=True)
    st[0].values.copy_(hv, non_blocking=True)
    ev[1].record()
    replay()
    ev[2].record()
    torch.cuda.synchronize()
    print(f"h2d {ev[0].elapsed_time(ev[1]):.3f} ms  step {ev[1].elapsed_time(ev[2]):.3f} ms")
t0 = time.perf_counter()
for it in range(20):
    replay()
torch.cuda.synchronize()
print(f"20 replays {1e3 * (time.perf_counter() - t0) / 20:.3f} ms/step")

# --- the bench.py e2e loop, verbatim structure, timed
K = 20
hosts = [(hl, hv, kj.nnz_per_feature)] * 4
cs = torch.cuda.Stream()
stage = [(torch.empty_like(st[0].lengths), torch.empty_like(st[0].values)) for _ in range(2)]
ready = [torch.cuda.Event() for _ in range(2)]
free = [torch.cuda.Event() for _ in range(2)]
losses = torch.zeros(K, dtype=torch.float32).pin_memory()
loss_buf = torch.zeros(K, dtype=torch.float32, device=dev)


def prefetch(j):
    hl_, hv_, _ = hosts[j % len(hosts)]
    with torch.cuda.stream(cs):
        cs.wait_event(free[j % 2])
        stage[j % 2][0].copy_(hl_, non_blocking=True)
        stage[j % 2][1].copy_(hv_, non_blocking=True)
        ready[j % 2].record(cs)


for rep in range(3):
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for evn in free:
        evn.record()
    prefetch(0)
    t0 = time.perf_counter()
    for i in range(K):
        cur = i % 2
        torch.cuda.current_stream().wait_event(ready[cur])
        st[0].lengths.copy_(stage[cur][0], non_blocking=True)
        st[0].values.copy_(stage[cur][1], non_blocking=True)
        free[cur].record()
        if i + 1 < K:
            prefetch(i + 1)
        replay()
        torch.dot(outs[0].view(-1).float(), gout[0].view(-1).float(), out=loss_buf[i])
        losses[i:i + 1].copy_(loss_buf[i:i + 1], non_blocking=True)
    t1 = time.perf_counter()
    e.record()
    torch.cuda.synchronize()
    print(f"e2e loop: {s.elapsed_time(e) / K:.3f} ms/step device, host issue {1e3 * (t1 - t0) / K:.3f} ms/step")
