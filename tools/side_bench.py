"""Fused crossnet-backward tail (dmt_dcn_side_fused) vs the per-layer form
(3 x dmt_dcn_dx0_term + 3 x dmt_column_sum) at the C2 shape, CUDA-event timed:

    python tools/side_bench.py          (needs a B200)
"""

import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2403_00877_b200 import kernels as K  # noqa: E402


def timeit(fn, reps=20):
    for _ in range(3):
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
    rows, cols, nl = 8192, 3328, 3
    g = torch.Generator(device="cuda").manual_seed(0)
    mk = lambda: torch.randn(rows, cols, device="cuda", generator=g).to(torch.bfloat16)  # noqa: E731
    gs, us, gus = [mk() for _ in range(nl)], [mk() for _ in range(nl)], [mk() for _ in range(nl)]
    dx0 = torch.empty(rows, cols, device="cuda")
    sums = [torch.empty(cols, device="cuda") for _ in range(nl)]

    def split():
        for l in range(nl - 1, -1, -1):
            K.dcn_dx0_term(gs[l], us[l], dx0, accumulate=l != nl - 1)
            K.column_sum(gus[l], out=sums[l])

    fused = lambda: K.dcn_side_fused(gs, us, gus, dx0, sums)  # noqa: E731
    nbytes = (3 * nl * rows * cols * 2 + rows * cols * 4)
    for name, fn in (("split", split), ("fused", fused)):
        ms = timeit(fn)
        print(f"{name:6s} {ms * 1e3:7.1f} us  ({nbytes / ms / 1e6:6.0f} GB/s of the fused pass's bytes)", flush=True)


if __name__ == "__main__":
    main()
