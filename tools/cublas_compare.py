"""Our plain GEMM vs cuBLAS on the C2 DCN shape, one launch each, for an ncu
capture that compares the two kernels' L2 / TMA / tensor-pipe metrics:

    ncu --set full -k regex:'gemm_kernel|nvjet|sm100' -c 4 python tools/cublas_compare.py

Without ncu it prints CUDA-event times (20 reps) of both, per shape.
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
    dt = torch.bfloat16
    once = "--once" in sys.argv
    g = torch.Generator(device="cuda").manual_seed(0)
    for (R, M, N) in [(8192, 3328, 3328), (8192, 1664, 3328)]:
        a = torch.randn(R, M, device="cuda", generator=g).to(dt)
        w = (torch.randn(N, M, device="cuda", generator=g) / M ** 0.5).to(dt)
        out = torch.empty(R, N, device="cuda", dtype=dt)
        ours = lambda: K.gemm(a, w, out)  # noqa: E731
        ref = lambda: torch.matmul(a, w.t(), out=out)  # noqa: E731
        if once:
            ours()
            ref()
            torch.cuda.synchronize()
            continue
        fl = 2 * R * M * N
        t0, t1 = timeit(ours), timeit(ref)
        print(f"{R}x{N}x{M}: dmt {t0 * 1e3:6.1f} us {fl / t0 / 1e9:6.0f} TF   cuBLAS {t1 * 1e3:6.1f} us "
              f"{fl / t1 / 1e9:6.0f} TF", flush=True)


if __name__ == "__main__":
    main()
