"""Probe: map a peer buffer via PeerFabric.share and write it with a libdmt kernel.

    torchrun --nproc-per-node 2 tools/p2p_probe.py
"""
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2403_00877_b200 import kernels as K  # noqa: E402
from paper_2403_00877_b200.fabric import PeerFabric  # noqa: E402

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(rank)
dev = torch.device("cuda", rank)
dist.init_process_group("nccl", device_id=dev)
fab = PeerFabric(world, rank, world, dev)
buf = torch.zeros(1 << 20, device=dev)
src = torch.full((1 << 20,), float(rank + 1), device=dev)
peer = fab.share({"buf": buf})
other = (rank + 1) % world
pb = peer[other]["buf"]
print(rank, "peer buffer of rank", pb.rank, hex(pb.data_ptr()), flush=True)
# libdmt batched copy kernel writing peer memory
K.CopyTable([(src.data_ptr(), pb.data_ptr() + 4096 * 4, 4096 * 4)], dev).run()
torch.cuda.synchronize()
print(rank, "kernel store done", flush=True)
fab.barrier_(list(range(world)))
torch.cuda.synchronize()
got = buf[4096:8192]
print(rank, "kernel copy", "ok" if bool((got == float(other + 1)).all()) else "MISMATCH", flush=True)
fab.close()
dist.destroy_process_group()
