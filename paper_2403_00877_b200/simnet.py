"""Byte accounting of the exchange collectives.

Mirror of towersim/simnet.py:18-107: every message of a collective is logged
as (label, src, dst, nbytes, link) with the reference's 4-bytes-per-element
wire convention (simnet.py:18), so the reference's byte-conservation checks
(c == f cross bytes, TM bytes / CR) run unchanged against the GPU path.  The
GPU exchange fills the trace from its real split sizes; ``wire_bytes`` keeps
the true on-wire size in the compute dtype alongside.
"""

from __future__ import annotations

from typing import NamedTuple, Optional

from .topology import CROSS_HOST, INTRA_HOST, ClusterTopology, link_class

BYTES_PER_ELEMENT = 4


class TraceEntry(NamedTuple):
    label: str
    src: int
    dst: int
    nbytes: int
    link: str


class CommTrace:
    """simnet.py:55-107: append-only message log of one run.

    Messages whose sizes only the device knows (the capacity-padded step a of
    ragged batches: the payload is each slot's actual nnz, not its capacity)
    are recorded from device counters (``record_device``) and resolved on the
    first query -- one host read, outside the step."""

    def __init__(self, topo: ClusterTopology):
        self.topo = topo
        self._entries: list[TraceEntry] = []
        self._pending: list = []
        self.wire_bytes: dict[str, int] = {}

    @property
    def entries(self) -> list[TraceEntry]:
        self._flush()
        return self._entries

    def record(self, label: str, src: int, dst: int, nbytes: int) -> None:
        self._entries.append(TraceEntry(label, src, dst, nbytes, link_class(src, dst, self.topo)))

    def record_device(self, label: str, src: int, dsts, counts, elem_bytes: int) -> None:
        """counts: device int64 tensor of elements src sends to each of dsts
        (e.g. from dmt_kjt_slot_offsets), read when the trace is queried."""
        self._pending.append((label, src, list(dsts), counts.clone(), int(elem_bytes)))

    def _flush(self) -> None:
        while self._pending:
            label, src, dsts, counts, eb = self._pending.pop(0)
            for dst, n in zip(dsts, counts.cpu().tolist()):
                self.record_elements(label, src, dst, int(n), eb)

    def record_elements(self, label: str, src: int, dst: int, elements: int, elem_bytes: int) -> None:
        self.record(label, src, dst, BYTES_PER_ELEMENT * int(elements))
        if src != dst:
            self.wire_bytes[label] = self.wire_bytes.get(label, 0) + int(elements) * int(elem_bytes)

    def byte_totals(self, label: Optional[str] = None) -> tuple[int, int]:
        intra = cross = 0
        for e in self.entries:
            if label is not None and e.label != label:
                continue
            if e.link == INTRA_HOST:
                intra += e.nbytes
            elif e.link == CROSS_HOST:
                cross += e.nbytes
        return intra, cross

    def labels(self) -> list[str]:
        seen: dict[str, None] = {}
        for e in self.entries:
            seen.setdefault(e.label, None)
        return list(seen)

    def sent_by_rank(self, label: str) -> dict[int, int]:
        out: dict[int, int] = {}
        for e in self.entries:
            if e.label == label:
                out[e.src] = out.get(e.src, 0) + e.nbytes
        return out

    def save(self, path) -> None:
        with open(path, "w", encoding="utf-8") as fh:
            for e in self.entries:
                fh.write(f"{e.label}\t{e.src}\t{e.dst}\t{e.nbytes}\t{e.link}\n")

    @staticmethod
    def load(path, topo: ClusterTopology) -> "CommTrace":
        trace = CommTrace(topo)
        with open(path, encoding="utf-8") as fh:
            for line in fh:
                label, src, dst, nbytes, link = line.rstrip("\n").split("\t")
                trace._entries.append(TraceEntry(label, int(src), int(dst), int(nbytes), link))
        return trace
