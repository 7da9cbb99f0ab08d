"""Microbenchmark of dmt_gemm on the DCN shapes of the bench step vs cuBLAS.

    python tools/gemm_bench.py            (needs a B200)
Prints one line per case: shape, epilogue, ms, TFLOP/s (dmt) and cuBLAS ms.
"""

import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2403_00877_b200 import _lib as L  # noqa: E402
from paper_2403_00877_b200 import kernels as K  # noqa: E402


TUNE = [0]
_gemm = K.gemm


def _tuned(*a, **kw):
    return _gemm(*a, tune_flags=TUNE[0], **kw)


K.gemm = _tuned


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
    R, M, P = 8192, 3328, 1664
    if len(sys.argv) > 1:
        R, M, P = (int(x) for x in sys.argv[1:4])
    g = torch.Generator(device="cuda").manual_seed(0)
    x0 = torch.randn(R, M, device="cuda", generator=g).to(dt)
    xl = torch.randn(R, M, device="cuda", generator=g).to(dt)
    W = (torch.randn(M, M, device="cuda", generator=g) / M ** 0.5).to(dt)
    Wp = (torch.randn(P, M, device="cuda", generator=g) / M ** 0.5).to(dt)
    b = torch.randn(M, device="cuda", generator=g)
    bp = torch.randn(P, device="cuda", generator=g)
    out = torch.empty(R, M, device="cuda", dtype=dt)
    u = torch.empty(R, M, device="cuda", dtype=dt)
    y = torch.empty(R, P, device="cuda", dtype=dt)
    gy = torch.randn(R, P, device="cuda", generator=g).to(dt)
    dW = torch.empty(M, M, device="cuda", dtype=torch.float32)
    dx0 = torch.zeros(R, M, device="cuda", dtype=torch.float32)
    gu = torch.empty(R, M, device="cuda", dtype=dt)
    part = torch.empty(K.colsum_rows(R), M, device="cuda", dtype=torch.float32)
    cases = [
        ("fwd cross", 2 * R * M * M, lambda: K.gemm(xl, W, out, bias=b, epilogue=L.EPI_CROSS, x0=x0, xl=xl, aux=u),
         lambda: torch.matmul(xl, W.t())),
        ("fwd cross no-aux", 2 * R * M * M, lambda: K.gemm(xl, W, out, bias=b, epilogue=L.EPI_CROSS, x0=x0, xl=xl),
         None),
        ("fwd plain", 2 * R * M * M, lambda: K.gemm(xl, W, out), None),
        ("fwd proj", 2 * R * P * M, lambda: K.gemm(xl, Wp, y, bias=bp, epilogue=L.EPI_BIAS),
         lambda: torch.matmul(xl, Wp.t())),
        ("bwd dW (MN,MN)", 2 * R * M * M, lambda: K.gemm(gu, xl, dW, trans_a=True, trans_b=True),
         lambda: torch.matmul(gu.t(), xl)),
        ("bwd dX dcn_bwd", 2 * R * M * M,
         lambda: K.gemm(gu, W, out, trans_b=True, epilogue=L.EPI_DCN_BWD, c=out, beta=1.0, x0=x0, xl=u, aux=xl,
                        aux2=dx0, aux2_accum=True), lambda: torch.matmul(gu, W)),
        ("bwd dX dcn_bwd +colsum", 2 * R * M * M,
         lambda: K.gemm(gu, W, out, trans_b=True, epilogue=L.EPI_DCN_BWD, c=out, beta=1.0, x0=x0, xl=u, aux=xl,
                        aux2=dx0, aux2_accum=True, colsum_part=part), None),
        ("bwd dX final legacy", 2 * R * M * M,
         lambda: K.gemm(gu, W, out, trans_b=True, epilogue=L.EPI_DCN_FINAL, c=u, beta=1.0, aux2=dx0), None),
        ("bwd dX dcn_bwd pairs", 2 * R * M * M,
         lambda: K.gemm(gu, W, out, trans_b=True, epilogue=L.EPI_DCN_BWD, c=u, beta=1.0, x0=x0, aux=xl,
                        colsum_part=part), None),
        ("bwd dX final 3 pairs", 2 * R * M * M,
         lambda: K.gemm(gu, W, out, trans_b=True, epilogue=L.EPI_DCN_FINAL, c=u, beta=1.0,
                        pairs=[(x0, u), (xl, u), (x0, xl)]), None),
        ("bwd dX dcn_bwd side", 2 * R * M * M,
         lambda: K.gemm(gu, W, out, trans_b=True, epilogue=L.EPI_DCN_BWD, c=u, beta=1.0, x0=x0, aux=xl), None),
        ("bwd g proj dcn side", 2 * R * M * P,
         lambda: K.gemm(gy, Wp, out, trans_b=True, epilogue=L.EPI_DCN_BWD, x0=x0, aux=xl), None),
        ("bwd dX plain (K,MN)", 2 * R * M * M, lambda: K.gemm(gu, W, out, trans_b=True), None),
        ("bwd dW fused sgd", 2 * R * M * M,
         lambda: K.gemm(gu, xl, W, trans_a=True, trans_b=True, epilogue=L.EPI_ACC, beta=1.0, alpha=-1e-9), None),
        ("bwd dWp", 2 * R * M * P, lambda: K.gemm(gy, xl, torch.empty(P, M, device="cuda"), trans_a=True,
                                                  trans_b=True), lambda: torch.matmul(gy.t(), xl)),
        ("bwd g proj dcn_bwd", 2 * R * M * P,
         lambda: K.gemm(gy, Wp, out, trans_b=True, epilogue=L.EPI_DCN_BWD, x0=x0, xl=u, aux=xl, aux2=dx0),
         lambda: torch.matmul(gy, Wp)),
    ]
    variants = [("auto", 0), ("single", L.GEMM_SINGLE_CTA), ("pair", L.GEMM_CLUSTER)] + [
        (f"bn{64 * j}", j << L.GEMM_BN_SHIFT) for j in (3, 4)] + [
        (f"bn{64 * j}pr", (j << L.GEMM_BN_SHIFT) | L.GEMM_CLUSTER) for j in (3, 4)]
    if os.environ.get("GB_QUICK"):  # default choice and per-thread (non-TMA) direct stores only
        variants = [("auto", 0), ("notma", L.GEMM_NO_TMA_STORE)]
    for name, flops, fn, ref in cases:
        line = f"{name:22s}"
        for vname, fl in variants:
            TUNE[0] = fl
            ms = timeit(fn)
            line += f" {vname} {ms * 1e3:6.1f}us {flops / ms / 1e9:6.0f}TF"
        TUNE[0] = 0
        if ref is not None:
            rms = timeit(ref)
            line += f"   cuBLAS {rms * 1e3:6.1f}us {flops / rms / 1e9:6.0f}TF"
        print(line, flush=True)


if __name__ == "__main__":
    main()
