"""Collective backends of the exchange: NCCL (one process per GPU) and an
in-process loopback that hosts several simulated ranks on one device.

Both implement the reference's all-to-all semantics (towersim/simnet.py:117-146):
member j of ``group`` receives one payload per source, in group order.  Payloads
here are flat device buffers with per-destination element splits; the
receiver's buffer is the concatenation of the sources' pieces in group order.
"""

from __future__ import annotations

import os
from typing import Optional, Sequence

import torch

from . import kernels as K
from .errors import ProtocolError
from .simnet import CommTrace


def _offsets(splits: Sequence[int]) -> list[int]:
    out, acc = [], 0
    for s in splits:
        out.append(acc)
        acc += int(s)
    return out


class Fabric:
    local_ranks: list[int]
    world_size: int

    def alltoallv(self, group: Sequence[int], label: str, send: dict, send_splits: dict, recv: dict,
                  recv_splits: dict, trace: Optional[CommTrace] = None, elem_bytes: int = 4) -> None:
        raise NotImplementedError

    def exchange_counts(self, group: Sequence[int], counts: dict) -> dict:
        """counts[r][j] = elements r sends to group[j]  ->  recv[r][j] from group[j]."""
        raise NotImplementedError

    def all_reduce_(self, group: Sequence[int], tensors: dict) -> None:
        raise NotImplementedError


class LoopbackFabric(Fabric):
    """All G ranks in this process on one device; delivery = one batched-copy
    kernel launch per collective (dmt_batched_copy)."""

    def __init__(self, world_size: int, device=None):
        self.world_size = world_size
        self.local_ranks = list(range(world_size))
        self.device = device or torch.device("cuda")

    def alltoallv(self, group, label, send, send_splits, recv, recv_splits, trace=None, elem_bytes=4):
        n = len(group)
        copies = []
        for i, src in enumerate(group):
            if len(send_splits[src]) != n:
                raise ProtocolError(f"rank {src} supplied {len(send_splits[src])} splits for {label!r}, expected {n}")
        for j, dst in enumerate(group):
            roffs = _offsets(recv_splits[dst])
            for i, src in enumerate(group):
                cnt = int(send_splits[src][j])
                if cnt != int(recv_splits[dst][i]):
                    raise ProtocolError(f"{label!r}: {src}->{dst} sends {cnt} but {recv_splits[dst][i]} expected")
                if trace is not None:
                    trace.record_elements(label, src, dst, cnt, elem_bytes)
                if cnt == 0:
                    continue
                soff = _offsets(send_splits[src])[j]
                s, d = send[src], recv[dst]
                es = s.element_size()
                sp, dp = s.data_ptr() + soff * es, d.data_ptr() + roffs[i] * es
                if sp != dp:  # aliased identity exchange (singleton group) moves nothing
                    copies.append((sp, dp, cnt * es))
        K.CopyTable(copies, self.device).run()

    def exchange_counts(self, group, counts):
        return {dst: [counts[src][j] for src in group] for j, dst in enumerate(group)}

    def all_reduce_(self, group, tensors):
        # every rank of a loopback tower shares one module; nothing to do
        return None


class NcclFabric(Fabric):
    """One rank per process; torch.distributed NCCL groups for the world, each
    tower (colour r // W) and each peer class (colour r % W), created once in a
    fixed order on every rank."""

    def __init__(self, world_size: int, rank: int, W: int, backend_device=None):
        import torch.distributed as dist

        self.dist = dist
        self.world_size = world_size
        self.rank = rank
        self.local_ranks = [rank]
        self.W = W
        self.T = world_size // W
        self.device = backend_device or torch.device("cuda", torch.cuda.current_device())
        self.groups = {tuple(range(world_size)): None}  # None = default (world) group
        for t in range(self.T):
            ranks = tuple(range(t * W, (t + 1) * W))
            g = dist.new_group(list(ranks)) if len(ranks) < world_size else None
            self.groups[ranks] = g
        for c in range(W):
            ranks = tuple(t * W + c for t in range(self.T))
            g = dist.new_group(list(ranks)) if 1 < len(ranks) < world_size else None
            self.groups.setdefault(ranks, g)

    def _pg(self, group):
        key = tuple(group)
        if key not in self.groups:
            self.groups[key] = self.dist.new_group(list(key))
        return self.groups[key]

    def alltoallv(self, group, label, send, send_splits, recv, recv_splits, trace=None, elem_bytes=4):
        r = self.rank
        if trace is not None:
            for j, dst in enumerate(group):
                trace.record_elements(label, r, dst, int(send_splits[r][j]), elem_bytes)
        if len(group) == 1:
            n = int(send_splits[r][0])
            if n and send[r].data_ptr() != recv[r].data_ptr():
                recv[r][:n].copy_(send[r][:n])
            return
        self.dist.all_to_all_single(recv[r][: sum(recv_splits[r])], send[r][: sum(send_splits[r])],
                                    output_split_sizes=[int(x) for x in recv_splits[r]],
                                    input_split_sizes=[int(x) for x in send_splits[r]],
                                    group=self._pg(group))

    def exchange_counts(self, group, counts):
        r = self.rank
        if len(group) == 1:
            return {r: list(counts[r])}
        s = torch.tensor(counts[r], dtype=torch.int64, device=self.device)
        o = torch.empty_like(s)
        self.dist.all_to_all_single(o, s, group=self._pg(group))
        return {r: o.cpu().tolist()}  # host sync: ragged step-a value splits

    def all_reduce_(self, group, tensors):
        if len(group) == 1:
            return
        pg = self._pg(group)
        for t in tensors.values():
            self.dist.all_reduce(t, group=pg)


class PeerBuffer:
    """A peer rank's exchange buffer mapped into this process: enough of the
    tensor interface (data_ptr / element_size / dtype / numel) for descriptor
    tables, which is all the producing kernels need."""

    def __init__(self, ptr: int, dtype, numel: int, rank: int):
        self.ptr, self.dtype, self._numel, self.rank = ptr, dtype, numel, rank

    def data_ptr(self) -> int:
        return self.ptr

    def element_size(self) -> int:
        return torch.empty((), dtype=self.dtype).element_size()

    def numel(self) -> int:
        return self._numel


class PeerFabric(NcclFabric):
    """NCCL plumbing plus NVLink peer memory: receive buffers of every rank are
    mapped into every other rank's address space (CUDA IPC through
    torch.multiprocessing's CUDA-tensor sharing), so producing kernels can
    write their exchange blocks straight into the consumer GPU's buffer.  A
    collective step then reduces to one tiny stream-ordered NCCL all-reduce per
    group used as a completion barrier (capturable in CUDA graphs)."""

    p2p = True

    # barriers of the world / tower / class groups run as device kernels over
    # NVLink (dmt_peer_barrier); DMT_PEER_BARRIER=nccl keeps the NCCL one
    device_barrier = os.environ.get("DMT_PEER_BARRIER", "device") == "device"

    def __init__(self, world_size: int, rank: int, W: int, backend_device=None):
        super().__init__(world_size, rank, W, backend_device)
        self._flag = torch.zeros(1, dtype=torch.float32, device=self.device)
        self._opened: dict = {}
        self._bar_args: dict = {}
        if self.device_barrier and world_size <= 8:
            # flags[kind][member] (kind 0 world, 1 tower, 2 class) + epochs
            self._bar_flags = torch.zeros((3, world_size), dtype=torch.int32, device=self.device)
            self._bar_epoch = torch.zeros(3, dtype=torch.int32, device=self.device)
            self._bar_err = torch.zeros(1, dtype=torch.int32, device=self.device)
            self._bar_peers = self.share({"barrier_flags": self._bar_flags})

    def share(self, tensors: dict) -> dict:
        """Collective over the world: every rank contributes {name: tensor};
        returns {rank: {name: buffer}} where a peer's buffer is a PeerBuffer
        mapped into THIS device's context (CUDA IPC opened under the accessing
        device, peer access enabled lazily -- the NVLink P2P transport) and the
        own rank's entries are the original tensors."""
        import ctypes as C

        from . import _lib as L

        lib = L.lib()
        mine = {}
        for k, v in tensors.items():
            h = (C.c_char * 64)()
            off = C.c_int64()
            L.check(lib.dmt_ipc_export(C.c_void_p(v.data_ptr()), h, C.byref(off)), "dmt_ipc_export")
            mine[k] = (bytes(h), off.value, v.dtype, v.numel())
        allv = [None] * self.world_size
        self.dist.all_gather_object(allv, mine)
        out = {}
        for r, objs in enumerate(allv):
            if r == self.rank:
                out[r] = dict(tensors)
                continue
            mapped = {}
            for k, (h, off, dtype, numel) in objs.items():
                base = self._opened.get((r, h))
                if base is None:
                    p = C.c_void_p()
                    L.check(lib.dmt_ipc_open(C.create_string_buffer(h, 64), C.byref(p)), "dmt_ipc_open")
                    base = self._opened[(r, h)] = p.value
                mapped[k] = PeerBuffer(base + off, dtype, numel, r)
            out[r] = mapped
        return out

    def close(self) -> None:
        from . import _lib as L

        for base in self._opened.values():
            L.lib().dmt_ipc_close(base)
        self._opened.clear()

    def _barrier_kind(self, group) -> Optional[int]:
        g = tuple(group)
        r, W = self.rank, self.W
        if g == tuple(range(self.world_size)):
            return 0
        if g == tuple(range((r // W) * W, (r // W + 1) * W)):
            return 1
        if g == tuple(t * W + r % W for t in range(self.T)):
            return 2
        return None

    def barrier_(self, group) -> None:
        """Completion barrier for peer writes: every member's preceding kernels
        (stream order) finished before any member passes it."""
        if len(group) == 1:
            return
        kind = self._barrier_kind(group) if self.device_barrier and self.world_size <= 8 else None
        if kind is not None:
            import ctypes as C

            from . import _lib as L

            args = self._bar_args.get(kind)
            if args is None:
                others = [m for m in group if m != self.rank]
                es = 4
                remote = [self._bar_peers[m]["barrier_flags"].data_ptr() + (kind * self.world_size + self.rank) * es
                          for m in others]
                local = [self._bar_flags.data_ptr() + (kind * self.world_size + m) * es for m in others]
                args = ((C.c_void_p * len(others))(*remote), (C.c_void_p * len(others))(*local), len(others))
                self._bar_args[kind] = args
            L.check(L.lib().dmt_peer_barrier(self._bar_epoch.data_ptr() + 4 * kind, args[0], args[1], args[2],
                                             self._bar_err.data_ptr(), L.stream_ptr()), "dmt_peer_barrier")
            return
        self.dist.all_reduce(self._flag, group=self._pg(group))


def slice_bounds(n: int, parts: int, i: int, align: int = 16) -> tuple[int, int]:
    """[begin, end) of part i when n elements are split into ``parts`` nearly
    equal, ``align``-aligned pieces."""
    step = -(-n // parts)
    step = -(-step // align) * align
    return min(n, i * step), min(n, (i + 1) * step)


def peer_allreduce_sgd(fabric, group, weights: dict, peer_g: dict, peer_w: dict, lr: float, device) -> None:
    """Data-parallel gradient all-reduce fused with SGD over NVLink peer memory
    as a reduce-scatter + all-gather: member i sums slice i of every member's
    fp32 gradient buffer (group order -- bit-identical to the loopback
    engine's rank-order sum), applies SGD to that slice of its own replica,
    then every member copies the other members' updated slices.  Per member
    ~(N-1)/N x (4 + weight bytes) per parameter cross the links, against
    (N-1) x 4 for every member reading every peer's whole gradient.
    ``peer_g[m][k]`` / ``peer_w[m][k]``: member m's gradient buffer / weight."""
    me = fabric.rank
    pos = group.index(me)
    n_grp = len(group)
    fabric.barrier_(group)  # every member's gradient buffers are complete
    for k, w in weights.items():
        b, e = slice_bounds(w.numel(), n_grp, pos)
        K.peer_sum_sgd(w, [peer_g[m][k] for m in group], lr, b, e)
    fabric.barrier_(group)  # every member's slice is updated
    copies = []
    for k, w in weights.items():
        es = w.element_size()
        for i, m in enumerate(group):
            if m == me:
                continue
            b, e = slice_bounds(w.numel(), n_grp, i)
            if e > b:
                copies.append((peer_w[m][k].data_ptr() + b * es, w.data_ptr() + b * es, (e - b) * es))
    K.CopyTable(copies, device).run()
