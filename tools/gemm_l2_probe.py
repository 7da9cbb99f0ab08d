"""L2 traffic of this package's plain bf16 GEMM vs cuBLAS at the C2 crossnet
shape (8192 x 3328 x 3328), one launch each after warm-up -- run under ncu:

    ncu --metrics lts__t_bytes.sum,lts__throughput.avg.pct_of_peak_sustained_elapsed,... python tools/gemm_l2_probe.py
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2403_00877_b200 import kernels as K  # noqa: E402


def main():
    R, M = 8192, 3328
    g = torch.Generator(device="cuda").manual_seed(0)
    x = torch.randn(R, M, device="cuda", generator=g).to(torch.bfloat16)
    W = (torch.randn(M, M, device="cuda", generator=g) / M ** 0.5).to(torch.bfloat16)
    out = torch.empty(R, M, device="cuda", dtype=torch.bfloat16)
    for _ in range(3):
        K.gemm(x, W, out)
        torch.matmul(x, W.t())
    torch.cuda.synchronize()
    K.gemm(x, W, out)
    torch.matmul(x, W.t())
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
