"""Typed torch-facing wrappers over the libdmt C ABI (include/dmt.h).

Each wrapper takes device tensors, validates shapes/dtypes on the host, calls
the C entry point on the current CUDA stream and maps non-zero status codes to
the reference exception classes.  No wrapper has a CPU path.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Optional, Sequence

import torch

from . import _lib as L
from .errors import DomainError, ShapeError, TableLookupError


def _dt(t: torch.Tensor) -> int:
    try:
        return L.TORCH_DT[t.dtype]
    except KeyError:
        raise DomainError(f"unsupported dtype {t.dtype}") from None


_TABLE_CACHE: dict = {}


def device_table(ctype, items: Sequence, device) -> tuple[torch.Tensor, object]:
    """Upload a list of ctypes structs; returns (device bytes, host array).

    Content-addressed: an identical table (same descriptors, same buffer
    pointers) is uploaded once and reused, so steady-state steps issue no
    host->device descriptor copies -- which is what makes a whole training
    step capturable as one CUDA graph."""
    arr = (ctype * max(1, len(items)))()
    for i, it in enumerate(items):
        arr[i] = it
    nbytes = C.sizeof(ctype) * max(1, len(items))
    raw = C.string_at(C.addressof(arr), nbytes)
    key = (ctype.__name__, str(device), raw)
    dev = _TABLE_CACHE.get(key)
    if dev is None:
        dev = _upload(raw, device)
        if len(_TABLE_CACHE) > 4096 and not torch.cuda.is_current_stream_capturing():
            _TABLE_CACHE.clear()
        _TABLE_CACHE[key] = dev
    return dev, arr


_PINNED_KEEPALIVE: list = []


def _upload(raw: bytes, device) -> torch.Tensor:
    """Bytes -> device.  Inside CUDA-graph capture the copy is recorded from a
    pinned host buffer that is kept alive (its content never changes, so every
    replay re-installs the same descriptors)."""
    if torch.cuda.is_current_stream_capturing():
        host = torch.frombuffer(bytearray(raw), dtype=torch.uint8).pin_memory()
        _PINNED_KEEPALIVE.append(host)
        dev = torch.empty(len(raw), dtype=torch.uint8, device=device)
        dev.copy_(host, non_blocking=True)
        return dev
    return torch.frombuffer(bytearray(raw), dtype=torch.uint8).to(device)


_INT_CACHE: dict = {}


def device_ints(values: Sequence[int], dtype: torch.dtype, device) -> torch.Tensor:
    """Content-addressed small integer array on the device (e.g. slot offsets)."""
    key = (tuple(int(v) for v in values), dtype, str(device))
    t = _INT_CACHE.get(key)
    if t is None:
        host = torch.tensor(key[0] or (0,), dtype=dtype)
        t = _upload(host.numpy().tobytes(), device).view(dtype)
        if len(_INT_CACHE) > 4096 and not torch.cuda.is_current_stream_capturing():
            _INT_CACHE.clear()
        _INT_CACHE[key] = t
    return t


# ------------------------------------------------------------------ KJT ----
def lengths_to_offsets(lengths: torch.Tensor) -> torch.Tensor:
    if lengths.dtype != torch.int32 or not lengths.is_cuda:
        raise DomainError("lengths must be a CUDA int32 tensor")
    lengths = lengths.contiguous()
    n = lengths.numel()
    out = torch.empty(n + 1, dtype=torch.int64, device=lengths.device)
    ws = torch.empty(max(1, L.lib().dmt_lengths_to_offsets_workspace_size(n)), dtype=torch.uint8,
                     device=lengths.device)
    L.check(L.lib().dmt_lengths_to_offsets(lengths.data_ptr(), n, out.data_ptr(), ws.data_ptr(), L.stream_ptr()),
            "dmt_lengths_to_offsets")
    return out


def kjt_bucketize(lengths, offsets, values, B: int, slot_feature: torch.Tensor,
                  slot_value_offset: torch.Tensor, out_lengths: torch.Tensor, out_values: torch.Tensor) -> None:
    n_slots = slot_feature.numel()
    L.check(L.lib().dmt_kjt_bucketize(lengths.data_ptr(), offsets.data_ptr(), values.data_ptr(), B, n_slots,
                                      slot_feature.data_ptr(), slot_value_offset.data_ptr(),
                                      out_lengths.data_ptr(), out_values.data_ptr(), L.stream_ptr()),
            "dmt_kjt_bucketize")


def kjt_bucketize_peer(lengths, offsets, values, B: int, slot_feature: torch.Tensor, slot_dst: torch.Tensor) -> None:
    """Step a with every slot written straight into its owner's receive
    buffers (slot_dst: device table of dmt_slot_dst)."""
    L.check(L.lib().dmt_kjt_bucketize_peer(lengths.data_ptr(), offsets.data_ptr(), values.data_ptr(), B,
                                           slot_feature.numel(), slot_feature.data_ptr(), slot_dst.data_ptr(),
                                           L.stream_ptr()), "dmt_kjt_bucketize_peer")


def kjt_slot_offsets(offsets: torch.Tensor, B: int, slot_feature: torch.Tensor, out: torch.Tensor) -> torch.Tensor:
    """Device-side packed slot offsets: out[s+1] - out[s] = nnz of slot s."""
    L.check(L.lib().dmt_kjt_slot_offsets(offsets.data_ptr(), B, slot_feature.numel(), slot_feature.data_ptr(),
                                         out.data_ptr(), L.stream_ptr()), "dmt_kjt_slot_offsets")
    return out


def kjt_compact(src: torch.Tensor, offsets: torch.Tensor, B: int, seg_src_start: torch.Tensor,
                dst: torch.Tensor) -> None:
    L.check(L.lib().dmt_kjt_compact(src.data_ptr(), offsets.data_ptr(), B, seg_src_start.numel(),
                                    seg_src_start.data_ptr(), dst.data_ptr(), L.stream_ptr()), "dmt_kjt_compact")


def kjt_check_capacity(offsets: torch.Tensor, B: int, capacity: torch.Tensor, flag: torch.Tensor) -> None:
    L.check(L.lib().dmt_kjt_check_capacity(offsets.data_ptr(), B, capacity.numel(), capacity.data_ptr(),
                                           flag.data_ptr(), L.stream_ptr()), "dmt_kjt_check_capacity")


# --------------------------------------------------------- pooled lookup ----
@dataclass
class Segment:
    """One lookup segment (dmt_lookup_segment)."""

    weights: torch.Tensor      # shard rows (rows, ld) -- row r at weights[r - row_begin]
    out: torch.Tensor          # base tensor of the output
    out_offset: int            # element offset of bag 0's row in `out`
    out_ld: int
    bag_begin: int
    nbags: int
    pooling: int
    row_begin: int = 0
    row_filter: bool = False
    key_base: int = 0
    state: Optional[torch.Tensor] = None
    table_rows: int = 0  # row-wise shards: global index range check (0 = off)

    def struct(self) -> L.LookupSegment:
        w = self.weights
        es = w.element_size()
        return L.LookupSegment(
            weights=w.data_ptr(),
            out=self.out.data_ptr() + self.out_offset * self.out.element_size(),
            state=self.state.data_ptr() if self.state is not None else None,
            ld=w.stride(0),
            out_ld=self.out_ld,
            bag_begin=self.bag_begin,
            row_begin=self.row_begin,
            key_base=self.key_base,
            rows=w.shape[0],
            width=w.shape[1],
            nbags=self.nbags,
            pooling=self.pooling,
            row_filter=1 if self.row_filter else 0,
            table_rows=self.table_rows,
        )


class SegmentTable:
    """Device + host copies of a segment list (reusable while buffers live)."""

    def __init__(self, segments: Sequence[Segment], device):
        self.segments = list(segments)
        self.n = len(self.segments)
        self.dev, self.host = device_table(L.LookupSegment, [s.struct() for s in self.segments], device)
        dts = {s.weights.dtype for s in self.segments}
        if len(dts) > 1:
            raise DomainError(f"segments mix dtypes {dts}")
        self.dtype = dts.pop() if dts else torch.float32


def pooled_lookup_fwd(table: SegmentTable, offsets: torch.Tensor, indices: torch.Tensor,
                      err: Optional[torch.Tensor] = None) -> None:
    if table.n == 0:
        return
    if indices.dtype != torch.int32 or offsets.dtype != torch.int64:
        raise DomainError("indices must be int32 and offsets int64")
    L.check(L.lib().dmt_pooled_lookup_fwd(table.dev.data_ptr(), C.addressof(table.host), table.n,
                                          offsets.data_ptr(), indices.data_ptr(), L.TORCH_DT[table.dtype],
                                          err.data_ptr() if err is not None else None, L.stream_ptr()),
            "dmt_pooled_lookup_fwd")


def raise_lookup_errors(err: torch.Tensor) -> None:
    bits = int(err.item())
    if bits & L.EBIT_BAGLEN:
        raise TableLookupError("pooling=none requires bags of length 1")
    if bits & L.EBIT_INDEX:
        raise TableLookupError("embedding index out of range")


def pooled_lookup_bwd_workspace(nnz: int, key_space: int, nbags: int, device) -> torch.Tensor:
    n = L.lib().dmt_pooled_lookup_bwd_workspace_size(nnz, key_space, nbags)
    return torch.empty(max(1, n), dtype=torch.uint8, device=device)


def pooled_lookup_bwd(table: SegmentTable, offsets, indices, nnz: int, key_space: int, optimizer: int,
                      lr: float, eps: float, workspace: torch.Tensor) -> None:
    if table.n == 0 or nnz == 0:
        return
    L.check(L.lib().dmt_pooled_lookup_bwd(table.dev.data_ptr(), C.addressof(table.host), table.n,
                                          offsets.data_ptr(), indices.data_ptr(), nnz, key_space,
                                          L.TORCH_DT[table.dtype], optimizer, lr, eps, workspace.data_ptr(),
                                          workspace.numel(), L.stream_ptr()),
            "dmt_pooled_lookup_bwd")


def pooled_lookup_bwd_prepare(table: SegmentTable, offsets, indices, nnz: int, key_space: int,
                              workspace: torch.Tensor) -> None:
    if table.n == 0 or nnz == 0:
        return
    L.check(L.lib().dmt_pooled_lookup_bwd_prepare(table.dev.data_ptr(), C.addressof(table.host), table.n,
                                                  offsets.data_ptr(), indices.data_ptr(), nnz, key_space,
                                                  L.TORCH_DT[table.dtype], workspace.data_ptr(), workspace.numel(),
                                                  L.stream_ptr()), "dmt_pooled_lookup_bwd_prepare")


def pooled_lookup_bwd_apply(table: SegmentTable, nnz: int, key_space: int, optimizer: int, lr: float, eps: float,
                            workspace: torch.Tensor) -> None:
    if table.n == 0 or nnz == 0:
        return
    L.check(L.lib().dmt_pooled_lookup_bwd_apply(table.dev.data_ptr(), C.addressof(table.host), table.n, nnz,
                                                key_space, L.TORCH_DT[table.dtype], optimizer, lr, eps,
                                                workspace.data_ptr(), workspace.numel(), L.stream_ptr()),
            "dmt_pooled_lookup_bwd_apply")


# ------------------------------------------------------------ assemble ----
@dataclass
class Block:
    dst_col: int
    width: int
    srcs: list  # [(tensor, element offset, ld)]
    groups: int = 0  # summed blocks: bit s = source s starts a new inner sum (dmt_assemble_block.groups)


class AssembleTable:
    def __init__(self, blocks: Sequence[Block], dst: torch.Tensor, rows: int, device):
        structs, srcs = [], []
        vec_ok = True
        es = dst.element_size()
        vec = 16 // es
        self.max_width = 0
        for b in blocks:
            if b.width == 0:
                continue
            structs.append(L.AssembleBlock(dst_col=b.dst_col, width=b.width, nsrc=len(b.srcs),
                                           first_src=len(srcs), groups=b.groups))
            self.max_width = max(self.max_width, b.width)
            if b.width % vec or b.dst_col % vec:
                vec_ok = False
            for t, off, ld in b.srcs:
                p = t.data_ptr() + off * es
                srcs.append(L.Src(ptr=p, ld=ld))
                if p % 16 or ld % vec:
                    vec_ok = False
        if dst.data_ptr() % 16 or dst.stride(0) % vec:
            vec_ok = False
        self.vec_ok = vec_ok
        self.n = len(structs)
        self.rows = rows
        self.dst = dst
        self.blocks_dev, self.blocks_host = device_table(L.AssembleBlock, structs, device)
        self.srcs_dev, self.srcs_host = device_table(L.Src, srcs, device)

    def run(self) -> None:
        if self.n == 0 or self.rows == 0:
            return
        mw = -self.max_width if self.vec_ok else self.max_width
        L.check(L.lib().dmt_assemble(self.blocks_dev.data_ptr(), self.n, mw, self.srcs_dev.data_ptr(), self.rows,
                                     self.dst.data_ptr(), self.dst.stride(0), _dt(self.dst), L.stream_ptr()),
                "dmt_assemble")


def assemble(blocks: Sequence[Block], dst: torch.Tensor, rows: int) -> None:
    AssembleTable(blocks, dst, rows, dst.device).run()


class CopyTable:
    def __init__(self, copies: Sequence[tuple[int, int, int]], device):
        structs = [L.Copy(src=s, dst=d, bytes=n) for s, d, n in copies if n > 0]
        self.n = len(structs)
        self.max_bytes = max((c.bytes for c in structs), default=0)
        self.dev, self.host = device_table(L.Copy, structs, device)

    def run(self) -> None:
        if self.n:
            L.check(L.lib().dmt_batched_copy(self.dev.data_ptr(), self.n, self.max_bytes, L.stream_ptr()),
                    "dmt_batched_copy")


class Copy2DTable:
    """Batched strided 2-D copies [(src tensor, src elem off, src_ld, dst tensor, dst off, dst_ld, rows, width)]."""

    def __init__(self, copies: Sequence[tuple], device):
        structs = []
        self.elem = None
        self.max_elems = 0
        self.vec = True
        for st, so, sld, dt, do, dld, rows, width in copies:
            if rows * width == 0:
                continue
            es = st.element_size()
            if self.elem is None:
                self.elem = es
            elif es != self.elem:
                raise DomainError("Copy2DTable mixes element sizes")
            sp, dp = st.data_ptr() + so * es, dt.data_ptr() + do * es
            if sp % 16 or dp % 16 or (sld * es) % 16 or (dld * es) % 16 or (width * es) % 16:
                self.vec = False
            structs.append(L.Copy2D(src=sp, dst=dp, src_ld=sld, dst_ld=dld, rows=rows, width=width))
            self.max_elems = max(self.max_elems, rows * width)
        self.n = len(structs)
        self.dev, self.host = device_table(L.Copy2D, structs, device)

    def run(self) -> None:
        if self.n:
            L.check(L.lib().dmt_batched_copy2d(self.dev.data_ptr(), self.n, -self.elem if self.vec else self.elem,
                                               self.max_elems, L.stream_ptr()), "dmt_batched_copy2d")


# ---------------------------------------------------------------- GEMM -----
def _aligned_operand(x: torch.Tensor) -> torch.Tensor:
    """TMA needs 16-byte aligned base and row stride: pad K with zeros if not."""
    es = x.element_size()
    if x.stride(1) == 1 and x.data_ptr() % 16 == 0 and (x.stride(0) * es) % 16 == 0:
        return x
    k = x.shape[1]
    kp = ((k * es + 15) // 16) * 16 // es
    y = torch.zeros((x.shape[0], kp), dtype=x.dtype, device=x.device)
    assemble([Block(0, k, [(x, 0, x.stride(0))])], y, x.shape[0]) if x.stride(1) == 1 else y[:, :k].copy_(x)
    return y


def split_tf32(x: torch.Tensor):
    """(hi, lo) tf32 split.  A 2-D operand keeps a 16-byte aligned row stride
    (TMA): a padded row-major view is split over its whole padded rows."""
    if x.dim() == 2 and not x.is_contiguous():
        k = x.shape[1]
        if x.stride(1) == 1 and x.stride(0) >= k:
            kp = x.stride(0)
        else:
            kp = (k + 3) // 4 * 4
        full = torch.zeros((x.shape[0], kp), dtype=x.dtype, device=x.device)
        full[:, :k].copy_(x)
        hi, lo = split_tf32(full)
        return hi[:, :k], lo[:, :k]
    x = x.contiguous()
    hi = torch.empty_like(x)
    lo = torch.empty_like(x)
    L.check(L.lib().dmt_split_tf32(x.data_ptr(), hi.data_ptr(), lo.data_ptr(), x.numel(), L.stream_ptr()),
            "dmt_split_tf32")
    return hi, lo


def gemm(a: torch.Tensor, b: torch.Tensor, out: torch.Tensor, *, bias: Optional[torch.Tensor] = None,
         epilogue: int = L.EPI_NONE, x0=None, xl=None, aux=None, beta: float = 0.0,
         rows_per_group: int = 0, ld_group: int = 0, ld_d: Optional[int] = None,
         b_split=None, trans_a: bool = False, trans_b: bool = False, c=None, aux2=None,
         aux2_accum: bool = False, alpha: Optional[float] = None, tune_flags: int = 0,
         pairs=(), colsum_part: Optional[torch.Tensor] = None, out_groups: Sequence[int] = (),
         col_groups: Sequence[tuple] = (), col_group_width: int = 0) -> torch.Tensor:
    """out[m, n] = epi(sum_k A[m, k] B[n, k]) on tcgen05 (bf16/f16 -> kind::f16,
    fp32 -> 3xTF32).  A = a (m, k), or a^T when ``trans_a`` (a stored (k, m));
    B = b (n, k), or b^T when ``trans_b`` (b stored (k, n)).  Transposed
    operands are read MN-major by TMA (no transpose pass).  ``b_split`` may
    carry a cached (hi, lo) tf32 split of an fp32 b.  ``pairs`` [(g, u), ...]
    adds sum g*u in the DCN_FINAL epilogue; ``colsum_part`` receives the fused
    per-tile column sums of gu (DCN_BWD; finish with column_sum_parts).
    ``out_groups`` (device addresses, with ``rows_per_group``): row block j is
    stored at out_groups[j] (row stride ld_d) instead of into ``out`` -- the
    GEMM fused with a scatter to peers' buffers.  ``col_groups`` [(address,
    row stride)] with ``col_group_width``: column block g is stored at its own
    address instead (the dX GEMM scattering shards to their owners)."""
    if a.dim() != 2 or b.dim() != 2:
        raise ShapeError("gemm operands must be 2-D")
    m, k = (a.shape[1], a.shape[0]) if trans_a else (a.shape[0], a.shape[1])
    n, kb = (b.shape[1], b.shape[0]) if trans_b else (b.shape[0], b.shape[1])
    if k != kb:
        raise ShapeError(f"gemm inner dims differ: {k} vs {kb}")
    if a.dtype != b.dtype:
        raise DomainError("gemm operands must share a dtype")
    if m == 0 or n == 0:
        return out
    if k == 0:
        raise ShapeError("gemm with k == 0")
    in_dt = _dt(a)
    a_lo = b_lo = None
    if a.dtype == torch.float32 and (trans_a or trans_b):
        # tcgen05 kind::tf32 takes K-major operands only (MN-major is a 16-bit
        # feature, like wgmma's transpose); the fp32 parity path transposes.
        if trans_a:
            a, trans_a = transpose(a), False
        if trans_b:
            b, trans_b, b_split = transpose(b), False, None
    if a.dtype == torch.float32:
        a_hi, a_lo = split_tf32(_aligned_operand(a))
        if b_split is not None:
            b_hi, b_lo = b_split
        else:
            b_hi, b_lo = split_tf32(_aligned_operand(b))
        a, b = a_hi, b_hi
    else:
        a = _aligned_operand(a)
        b = _aligned_operand(b)
    if bias is not None and (bias.dtype != torch.float32 or not bias.is_contiguous()):
        bias = bias.float().contiguous()
    flags = ((L.GEMM_TRANS_A if trans_a else 0) | (L.GEMM_TRANS_B if trans_b else 0)
             | (L.GEMM_AUX2_ACCUM if aux2_accum else 0) | (L.GEMM_SCALE_ACC if alpha is not None else 0)
             | tune_flags)
    args = L.GemmArgs(
        a=a.data_ptr(), b=b.data_ptr(), d=out.data_ptr(), bias=L.ptr(bias), x0=L.ptr(x0), xl=L.ptr(xl),
        aux=L.ptr(aux), c=L.ptr(c), aux2=L.ptr(aux2), m=m, n=n, k=k, lda=a.stride(0), ldb=b.stride(0),
        ld_d=ld_d if ld_d is not None else out.stride(0),
        ld_x=(x0.stride(0) if x0 is not None else (aux2.stride(0) if aux2 is not None else
                                                   (pairs[0][0].stride(0) if pairs else 0))),
        rows_per_group=rows_per_group, ld_group=ld_group,
        beta=beta, alpha=alpha if alpha is not None else 1.0, in_dtype=in_dt, out_dtype=_dt(out),
        epilogue=epilogue, flags=flags, npairs=len(pairs), colsum_part=L.ptr(colsum_part))
    if len(pairs) > L.GEMM_MAX_PAIRS:
        raise DomainError(f"at most {L.GEMM_MAX_PAIRS} epilogue pairs")
    # split-K for few output tiles over a long K (tower-module / MLP weight
    # gradients: e.g. DLRM dW_feat is 64 x 128 over K = T*B*F rows) -- one tile
    # per CTA would leave all but a handful of the 148 SMs idle
    ks = splitk_factor(m, n, k, a.element_size()) if (epilogue in (L.EPI_NONE, L.EPI_ACC) and not rows_per_group
                                                      and colsum_part is None and not pairs) else 1
    if ks > 1:
        args.ksplit = ks
        ws = torch.empty(ks * m * n, dtype=torch.float32, device=out.device)
        args.splitk_ws = ws.data_ptr()
    for j, (g, u) in enumerate(pairs):
        args.pair_g[j], args.pair_u[j] = g.data_ptr(), u.data_ptr()
    if col_groups:
        if len(col_groups) > L.GEMM_MAX_COL_GROUPS or col_group_width * len(col_groups) != n:
            raise DomainError("col_groups must tile the output columns (at most 32 blocks)")
        args.n_col_groups = len(col_groups)
        args.col_group_width = col_group_width
        for j, (ptr, ld) in enumerate(col_groups):
            args.col_group[j] = int(ptr)
            args.col_group_ld[j] = int(ld)
    if out_groups:
        if len(out_groups) > L.GEMM_MAX_OUT_GROUPS or not rows_per_group:
            raise DomainError("out_groups needs rows_per_group and at most 8 groups")
        args.n_out_groups = len(out_groups)
        for j, ptr in enumerate(out_groups):
            args.out_group[j] = int(ptr)
    L.check(L.lib().dmt_gemm_ex(C.byref(args), L.ptr(a_lo), L.ptr(b_lo), L.stream_ptr()), "dmt_gemm")
    return out


def splitk_factor(m: int, n: int, k: int, es: int) -> int:
    """K splits for an (m, n, k) GEMM: enough units to cover the SMs when the
    output has few 128 x 128 tiles, each split keeping >= 8 K blocks."""
    tiles = -(-m // 128) * -(-n // 128)
    kb = -(-(k * es) // 128)
    if tiles >= 74 or kb < 16:
        return 1
    return max(1, min(148 // tiles, kb // 8, 64))


def bce_with_logits(z: torch.Tensor, y: torch.Tensor, scale: float, dz: Optional[torch.Tensor] = None,
                    loss: Optional[torch.Tensor] = None):
    """dz = scale (sigmoid(z) - y); loss[0] = scale * sum BCE(z, y) (fp32)."""
    n = z.numel()
    if not z.is_contiguous() or not y.is_contiguous():
        raise ShapeError("bce_with_logits needs contiguous logits and labels")
    if y.numel() != n:
        raise ShapeError(f"labels {tuple(y.shape)} do not match logits {tuple(z.shape)}")
    if dz is None:
        dz = torch.empty_like(z)
    if loss is None:
        loss = torch.empty(1, dtype=torch.float32, device=z.device)
    L.check(L.lib().dmt_bce_with_logits(z.data_ptr(), y.data_ptr(), n, _dt(z), float(scale), dz.data_ptr(),
                                        loss.data_ptr(), L.stream_ptr()), "dmt_bce_with_logits")
    return dz, loss


def colsum_rows(m: int) -> int:
    return int(L.lib().dmt_gemm_colsum_rows(m))


def column_sum_parts(part: torch.Tensor, out: Optional[torch.Tensor] = None) -> torch.Tensor:
    """out[c] = sum_r part[r, c] (fp64 in row order): finishes fused bias grads."""
    rows, cols = part.shape
    if out is None:
        out = torch.empty(cols, dtype=torch.float32, device=part.device)
    L.check(L.lib().dmt_column_sum_parts(part.data_ptr(), rows, cols, out.data_ptr(), L.stream_ptr()),
            "dmt_column_sum_parts")
    return out


def transpose(x: torch.Tensor) -> torch.Tensor:
    r, c = x.shape
    out = torch.empty((c, r), dtype=x.dtype, device=x.device)
    L.check(L.lib().dmt_transpose(x.data_ptr(), r, c, x.stride(0), out.data_ptr(), out.stride(0), _dt(x),
                                  L.stream_ptr()), "dmt_transpose")
    return out


def column_sum(x: torch.Tensor, out: Optional[torch.Tensor] = None) -> torch.Tensor:
    r, c = x.shape
    if out is None:
        out = torch.empty(c, dtype=torch.float32, device=x.device)
    ws = torch.empty(max(1, L.lib().dmt_column_sum_workspace_size(r, c)), dtype=torch.uint8, device=x.device)
    L.check(L.lib().dmt_column_sum(x.data_ptr(), r, c, x.stride(0), out.data_ptr(), _dt(x), ws.data_ptr(),
                                   ws.numel(), L.stream_ptr()), "dmt_column_sum")
    return out


def cross_bwd_pointwise(g, x0, u, gu, dx0) -> None:
    L.check(L.lib().dmt_cross_bwd_pointwise(g.data_ptr(), x0.data_ptr(), u.data_ptr(), gu.data_ptr(),
                                            dx0.data_ptr(), g.numel(), _dt(g), L.stream_ptr()),
            "dmt_cross_bwd_pointwise")


def dcn_dx0_term(g: torch.Tensor, u: torch.Tensor, dx0: torch.Tensor, accumulate: bool) -> None:
    """dx0 (+)= g * u (fp32 dx0; g, u contiguous in the compute dtype)."""
    if dx0.dtype != torch.float32 or g.shape != u.shape or g.numel() != dx0.numel():
        raise ShapeError("dcn_dx0_term: g, u of one shape, fp32 dx0 of the same size")
    if not (g.is_contiguous() and u.is_contiguous() and dx0.is_contiguous()):
        raise ShapeError("dcn_dx0_term: contiguous operands")
    L.check(L.lib().dmt_dcn_dx0_term(g.data_ptr(), u.data_ptr(), dx0.data_ptr(), g.numel(), _dt(g), int(accumulate),
                                     L.stream_ptr()), "dmt_dcn_dx0_term")


def dcn_side_fused(gs: list, us: list, gus: Optional[list], dx0: torch.Tensor, colsums: Optional[list]) -> None:
    """dx0 = sum_{l=L-1..0} gs[l] * us[l] (fp32) and colsums[l] = column sums of
    gus[l]: dx0 in one streaming pass, then the column sums (bit-identical to
    the dcn_dx0_term sequence + column_sum)."""
    import ctypes as C

    n = len(gs)
    sums = colsums is not None
    if not (1 <= n <= 4) or len(us) != n or (sums and (gus is None or len(gus) != n or len(colsums) != n)):
        raise ShapeError("dcn_side_fused: 1..4 layers, one g / u (/ gu / colsum) each")
    rows, cols = gs[0].shape
    for t in (*gs, *us, *(gus if sums else ())):
        if tuple(t.shape) != (rows, cols) or not t.is_contiguous() or t.dtype != gs[0].dtype:
            raise ShapeError("dcn_side_fused: contiguous [rows, cols] operands of one dtype")
    if dx0.dtype != torch.float32 or dx0.numel() != rows * cols or not dx0.is_contiguous():
        raise ShapeError("dcn_side_fused: contiguous fp32 dx0 of the same size")
    ws = torch.empty(max(1, L.lib().dmt_dcn_side_fused_workspace_size(rows, cols, n)), dtype=torch.uint8,
                     device=dx0.device)
    arr = C.c_void_p * n
    L.check(L.lib().dmt_dcn_side_fused(arr(*[t.data_ptr() for t in gs]), arr(*[t.data_ptr() for t in us]),
                                       arr(*[t.data_ptr() for t in gus]) if sums else None, n, rows, cols,
                                       dx0.data_ptr(), arr(*[t.data_ptr() for t in colsums]) if sums else None,
                                       _dt(gs[0]), ws.data_ptr(), ws.numel(), L.stream_ptr()), "dmt_dcn_side_fused")


def sgd_dense(w: torch.Tensor, g: torch.Tensor, lr: float) -> None:
    if g.dtype != torch.float32:
        raise DomainError("dense gradients are fp32")
    L.check(L.lib().dmt_sgd_dense(w.data_ptr(), g.data_ptr(), w.numel(), lr, _dt(w), L.stream_ptr()),
            "dmt_sgd_dense")


def peer_sum_sgd(w: torch.Tensor, grads: list, lr: float, begin: int = 0, end: Optional[int] = None) -> None:
    """w -= lr * sum(grads) (fp32, summed in list order) over elements [begin,
    end) (``begin`` a multiple of 4); ``grads`` are this rank's and
    peer-mapped (PeerBuffer) gradient buffers of w's size."""
    import ctypes as C

    end = w.numel() if end is None else end
    for g in grads:
        if g.dtype != torch.float32 or g.numel() != w.numel():
            raise DomainError("peer gradients must be fp32 buffers of the weight's size")
    if begin % 4 or not 0 <= begin <= end <= w.numel():
        raise DomainError("peer_sum_sgd range must start at a multiple of 4 inside the weight")
    if end == begin:
        return
    arr = (C.c_void_p * len(grads))(*[g.data_ptr() + 4 * begin for g in grads])
    L.check(L.lib().dmt_peer_sum_sgd(w.data_ptr() + begin * w.element_size(), arr, len(grads), end - begin, lr,
                                     _dt(w), L.stream_ptr()), "dmt_peer_sum_sgd")


def convert(x: torch.Tensor, dtype: torch.dtype) -> torch.Tensor:
    out = torch.empty(x.shape, dtype=dtype, device=x.device)
    L.check(L.lib().dmt_convert(x.data_ptr(), _dt(x), out.data_ptr(), _dt(out), x.numel(), L.stream_ptr()),
            "dmt_convert")
    return out


# ------------------------------------------------------- DLRM interaction ---
def dot_interaction_fwd(dense: torch.Tensor, sparse: torch.Tensor, num_sparse: int,
                        out: Optional[torch.Tensor] = None) -> torch.Tensor:
    """out (B, D + P) = [dense | <V_i, V_j> (i > j)], V = [dense | sparse as
    (B, num_sparse, D)] (dmt_dot_interaction_fwd; P = (F+1)F/2)."""
    B, D = dense.shape
    width = D + (num_sparse + 1) * num_sparse // 2
    if sparse.shape[0] != B or sparse.shape[1] < num_sparse * D:
        raise ShapeError(f"sparse {tuple(sparse.shape)} does not hold {num_sparse} x {D} per sample")
    if dense.dtype != sparse.dtype:
        raise DomainError("dense and sparse operands must share a dtype")
    if out is None:
        out = torch.empty((B, width), dtype=dense.dtype, device=dense.device)
    L.check(L.lib().dmt_dot_interaction_fwd(dense.data_ptr(), dense.stride(0), sparse.data_ptr(), sparse.stride(0),
                                            num_sparse, D, B, out.data_ptr(), out.stride(0), _dt(dense),
                                            L.stream_ptr()), "dmt_dot_interaction_fwd")
    return out


def dot_interaction_bwd(grad_out: torch.Tensor, dense: torch.Tensor, sparse: torch.Tensor, num_sparse: int,
                        d_dense: Optional[torch.Tensor] = None, d_sparse: Optional[torch.Tensor] = None):
    B, D = dense.shape
    if d_dense is None:
        d_dense = torch.empty_like(dense)
    if d_sparse is None:
        d_sparse = torch.empty((B, num_sparse * D), dtype=dense.dtype, device=dense.device)
    L.check(L.lib().dmt_dot_interaction_bwd(grad_out.data_ptr(), grad_out.stride(0), dense.data_ptr(), dense.stride(0),
                                            sparse.data_ptr(), sparse.stride(0), num_sparse, D, B,
                                            d_dense.data_ptr(), d_dense.stride(0), d_sparse.data_ptr(),
                                            d_sparse.stride(0), _dt(dense), L.stream_ptr()), "dmt_dot_interaction_bwd")
    return d_dense, d_sparse


def relu_bwd(dy: torch.Tensor, y: torch.Tensor, out: Optional[torch.Tensor] = None) -> torch.Tensor:
    """dz = dy * (y > 0) (contiguous operands)."""
    if out is None:
        out = torch.empty_like(dy)
    L.check(L.lib().dmt_relu_bwd(dy.data_ptr(), y.data_ptr(), out.data_ptr(), dy.numel(), _dt(dy), L.stream_ptr()),
            "dmt_relu_bwd")
    return out
