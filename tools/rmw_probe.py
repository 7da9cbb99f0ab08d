"""Achievable HBM bandwidth of random 256-byte row read-modify-write (the
embedding-backward apply's access pattern) vs random row reads (the lookup's):
torch index ops over a 6.6 GB bf16 table with 3.93 M unique random rows (the C2
step's unique-row count).  Prints GB/s of algorithmic bytes."""
import torch

rows, dim, U = 26_000_000, 128, 3_929_004
dev = torch.device("cuda")
W = torch.zeros(rows, dim, dtype=torch.bfloat16, device=dev)
idx = torch.randperm(rows, device=dev)[:U]
upd = torch.ones(U, dim, dtype=torch.bfloat16, device=dev)


def timeit(fn, n=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(n):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / n


row_bytes = dim * 2
ms = timeit(lambda: W.index_select(0, idx))
print(f"random row gather  (read {U} rows + write dense): {ms * 1e3:.0f} us  "
      f"{U * row_bytes * 2 / ms / 1e6:.0f} GB/s", flush=True)
ms = timeit(lambda: W.index_add_(0, idx, upd))
print(f"random row RMW index_add_ (read+write {U} rows, read dense upd): {ms * 1e3:.0f} us  "
      f"{U * row_bytes * 3 / ms / 1e6:.0f} GB/s", flush=True)
ms = timeit(lambda: W.index_copy_(0, idx, upd))
print(f"random row scatter index_copy_ (write {U} rows): {ms * 1e3:.0f} us  "
      f"{U * row_bytes * 2 / ms / 1e6:.0f} GB/s", flush=True)
