"""Accuracy of the fp32 GEMM path (3xTF32 on tcgen05) vs torch fp32 (no TF32)
and fp64, on the C2 tower-module shapes.  Prints max-norm relative errors."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2403_00877_b200 import _lib as L, kernels as K

torch.backends.cuda.matmul.allow_tf32 = False
dev = torch.device("cuda")
g = torch.Generator(device="cuda").manual_seed(0)


def rel(a, b):
    return float((a.double() - b).abs().max() / b.abs().max())


for (m, n, k) in [(8192, 3328, 3328), (3328, 3328, 8192), (8192, 3328, 512), (8192, 1664, 3328)]:
    a = torch.randn(m, k, device=dev, generator=g)
    b = torch.randn(n, k, device=dev, generator=g)
    want = a.double() @ b.double().T
    out = torch.empty(m, n, device=dev)
    K.gemm(a, b, out)
    t32 = a @ b.T
    print(f"gemm {m}x{n}x{k}: dmt 3xTF32 {rel(out, want):.3e}  torch fp32 {rel(t32, want):.3e}", flush=True)

# DCN forward at C2 (3 layers + projection)
rows, M, P = 8192, 3328, 1664
x0 = (torch.rand(rows, M, device=dev, generator=g) * 2 - 1) * 2.58
Ws = [(torch.rand(M, M, device=dev, generator=g) * 2 - 1) / M ** 0.5 for _ in range(3)]
bs = [(torch.rand(M, device=dev, generator=g) * 2 - 1) / M ** 0.5 for _ in range(3)]
Wp = (torch.rand(P, M, device=dev, generator=g) * 2 - 1) / M ** 0.5
bp = (torch.rand(P, device=dev, generator=g) * 2 - 1) / M ** 0.5


def fwd(xd, mm, cross):
    xl = xd
    for W, b in zip(Ws, bs):
        xl = cross(xl, W, b, xd)
    return mm(xl, Wp) + bp.to(xl.dtype)


ref = fwd(x0.double(), lambda x, W: x @ W.double().T,
          lambda xl, W, b, x0_: x0_ * (xl @ W.double().T + b.double()) + xl)
t32 = fwd(x0, lambda x, W: x @ W.T, lambda xl, W, b, x0_: x0_ * (xl @ W.T + b) + xl)


def dcross(xl, W, b, x0_):
    o = torch.empty_like(xl)
    K.gemm(xl, W, o, bias=b, epilogue=L.EPI_CROSS, x0=x0_, xl=xl)
    return o


def dmm(x, W):
    o = torch.empty(x.shape[0], W.shape[0], device=dev)
    K.gemm(x, W, o)
    return o


dm = fwd(x0, dmm, dcross)
print(f"DCN fwd C2: dmt {rel(dm, ref):.3e}  torch fp32 {rel(t32, ref):.3e}", flush=True)
