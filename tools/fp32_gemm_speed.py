"""fp32 (3xTF32) GEMM time at the C2 shape for the current DMT_TF32_KCHUNK."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2403_00877_b200 import kernels as K, _lib as L

g = torch.Generator(device="cuda").manual_seed(0)
m, n, k = 8192, 3328, 3328
a = torch.randn(m, k, device="cuda", generator=g)
b = torch.randn(n, k, device="cuda", generator=g)
hi_a, lo_a = K.split_tf32(a)
hi_b, lo_b = K.split_tf32(b)
out = torch.empty(m, n, device="cuda")
x0 = torch.randn(m, n, device="cuda", generator=g)
bias = torch.randn(n, device="cuda", generator=g)


def run():
    K.gemm(a, b, out, b_split=(hi_b, lo_b), bias=bias, epilogue=L.EPI_CROSS, x0=x0, xl=x0)


for _ in range(3):
    run()
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(10):
    run()
e.record()
torch.cuda.synchronize()
ms = s.elapsed_time(e) / 10
print(f"kchunk={os.environ.get('DMT_TF32_KCHUNK', 'default')} fp32 cross gemm {m}x{n}x{k}: {ms:.3f} ms "
      f"({2 * m * n * k / ms / 1e9:.0f} TFLOP/s fp32-equivalent)", flush=True)
