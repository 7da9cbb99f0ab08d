"""DRAM / L2 traffic of the DCN GEMM epilogues in isolation (run under ncu):
the C2 dX GEMM plain vs with the DCN_BWD epilogue (and its parts), and the
forward crossnet GEMM, one launch each after a warm-up.

    ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
        -k regex:gemm_kernel python tools/epi_traffic.py
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2403_00877_b200 import _lib as L  # noqa: E402
from paper_2403_00877_b200 import kernels as K  # noqa: E402


def main():
    dt = torch.bfloat16
    R, M = 8192, 3328
    g = torch.Generator(device="cuda").manual_seed(0)
    mk = lambda *s: torch.randn(*s, device="cuda", generator=g).to(dt)  # noqa: E731
    x0, xl, u, gu, gres = mk(R, M), mk(R, M), mk(R, M), mk(R, M), mk(R, M)
    W = (torch.randn(M, M, device="cuda", generator=g) / M ** 0.5).to(dt)
    b = torch.randn(M, device="cuda", generator=g)
    out, aux = torch.empty(R, M, device="cuda", dtype=dt), torch.empty(R, M, device="cuda", dtype=dt)
    cases = {
        "dx_plain": lambda: K.gemm(gu, W, out, trans_b=True),
        "dx_dcn_bwd": lambda: K.gemm(gu, W, out, trans_b=True, epilogue=L.EPI_DCN_BWD, c=gres, beta=1.0, x0=x0,
                                     aux=aux),
        "dx_acc_c": lambda: K.gemm(gu, W, out, trans_b=True, epilogue=L.EPI_ACC, c=gres, beta=1.0),
        "dx_dcn_bwd_noc": lambda: K.gemm(gu, W, out, trans_b=True, epilogue=L.EPI_DCN_BWD, x0=x0, aux=aux),
        "fwd_cross": lambda: K.gemm(xl, W, out, bias=b, epilogue=L.EPI_CROSS, x0=x0, xl=xl, aux=u),
        "fwd_plain": lambda: K.gemm(xl, W, out),
    }
    sel = sys.argv[1:] or list(cases)
    for name in sel:
        for _ in range(3):
            cases[name]()
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(10):
            cases[name]()
        e.record()
        torch.cuda.synchronize()
        print(f"{name:16s} {s.elapsed_time(e) / 10 * 1e3:7.1f} us", flush=True)


if __name__ == "__main__":
    main()
