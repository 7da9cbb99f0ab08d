"""Microbenchmark of the pooled lookup forward and the fused backward (prepare /
apply) on the C2 shape: 26 tables x 1M rows x 128, bf16, B=8192, pooling 20.

    python tools/lookup_bench.py [dtype]      (needs a B200)
"""

import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2403_00877_b200 import _lib as L  # noqa: E402
from paper_2403_00877_b200 import kernels as K  # noqa: E402


def timeit(fn, reps=10):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


def main():
    dt = {"bf16": torch.bfloat16, "fp32": torch.float32}[sys.argv[1] if len(sys.argv) > 1 else "bf16"]
    F, R, N, B, P = 26, 1_000_000, 128, 8192, 20
    dev = torch.device("cuda")
    g = torch.Generator(device=dev).manual_seed(0)
    tabs = [torch.empty(R, N, device=dev, dtype=torch.float32).uniform_(-1, 1, generator=g).to(dt) for _ in range(F)]
    out = torch.empty(F * B * N, device=dev, dtype=dt)
    grad = torch.randn(F * B * N, device=dev, generator=g).to(dt) * 1e-3
    lens = torch.full((F * B,), P, dtype=torch.int32, device=dev)
    idx = torch.randint(0, R, (F * B * P,), generator=g, device=dev, dtype=torch.int32)
    offs = K.lengths_to_offsets(lens)
    kb = 0
    fsegs, bsegs = [], []
    for f in range(F):
        fsegs.append(K.Segment(weights=tabs[f], out=out, out_offset=f * B * N, out_ld=N, bag_begin=f * B, nbags=B,
                               pooling=L.POOL_SUM, key_base=kb))
        bsegs.append(K.Segment(weights=tabs[f], out=grad, out_offset=f * B * N, out_ld=N, bag_begin=f * B, nbags=B,
                               pooling=L.POOL_SUM, key_base=kb))
        kb += R
    ft, bt = K.SegmentTable(fsegs, dev), K.SegmentTable(bsegs, dev)
    nnz = F * B * P
    ws = K.pooled_lookup_bwd_workspace(nnz, kb, F * B, dev)
    es = tabs[0].element_size()
    fwd_bytes = nnz * N * es + nnz * 4 + (F * B + 1) * 8 + F * B * N * es
    ms = timeit(lambda: K.pooled_lookup_fwd(ft, offs, idx))
    print(f"lookup fwd   {ms * 1e3:8.1f} us  {fwd_bytes / ms / 1e6:8.1f} GB/s (algorithmic)")
    ms_p = timeit(lambda: K.pooled_lookup_bwd_prepare(bt, offs, idx, nnz, kb, ws))
    print(f"bwd prepare  {ms_p * 1e3:8.1f} us")
    ms_a = timeit(lambda: K.pooled_lookup_bwd_apply(bt, nnz, kb, L.OPT_SGD, 1e-4, 0.0, ws))
    uniq = 4_100_000  # ~unique rows for uniform 1M rows x 163,840 draws per table
    bwd_bytes = F * B * N * es + 2 * uniq * N * es
    print(f"bwd apply    {ms_a * 1e3:8.1f} us  {bwd_bytes / ms_a / 1e6:8.1f} GB/s (grad + 2 x unique rows)")


if __name__ == "__main__":
    main()
