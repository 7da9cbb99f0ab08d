"""Time dmt_column_sum on the DCN bias-gradient shape (8192 x 3328 bf16)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2403_00877_b200 import kernels as K  # noqa: E402

x = torch.randn(8192, 3328, device="cuda").to(torch.bfloat16)
out = torch.empty(3328, device="cuda")
for _ in range(3):
    K.column_sum(x, out)
torch.cuda.synchronize()
# graph-replayed so host launch overhead does not hide the kernel time
gr = torch.cuda.CUDAGraph()
with torch.cuda.graph(gr):
    for _ in range(50):
        K.column_sum(x, out)
gr.replay()
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
gr.replay()
e.record()
torch.cuda.synchronize()
ms = s.elapsed_time(e) / 50
print(f"column_sum 8192x3328 bf16: {ms * 1e3:.1f} us  {x.numel() * 2 / ms / 1e6:.0f} GB/s")
