"""numpy emulation of the device pipeline driven by the real ExchangePlan.

Test helper only: every buffer layout, split and assemble block the GPU engine
uses comes from paper_2403_00877_b200.plan; the kernels are replaced by numpy
(pooling via the oracle).  If the emulation reproduces the oracle's SPTT /
flat outputs, the host-side routing plan is right independent of any GPU.
"""

from __future__ import annotations

import numpy as np

import oracle


def _owner_kjt(plan, r, lengths, values, offs):
    """Owner r's received KJT in the plan's (p, k, b) order (step a)."""
    G, F, B = lengths.shape
    lens, idx = [], []
    for p in range(G):
        for sid in plan.by_owner[r]:
            f = plan.fpos[plan.shards[sid].table_id]
            base = (p * F + f) * B
            lens.append(lengths[p, f])
            idx.append(values[offs[base]:offs[base + B]])
    lens = np.concatenate(lens) if lens else np.zeros(0, np.int64)
    idx = np.concatenate(idx) if idx else np.zeros(0, np.int64)
    return lens, idx


def lookup_send_buffer(plan, placement_tables, r, lengths, values, sptt):
    """Step b into the plan's send layout (fused permute) for owner r."""
    offs = oracle.kjt_offsets(lengths)
    lens, idx = _owner_kjt(plan, r, lengths, values, offs)
    boff = np.concatenate([[0], np.cumsum(lens)])
    size = plan.send_d_size(r) if sptt else plan.send_c_size(r)
    buf = np.zeros(max(1, size))
    for (p, k, off, w) in plan.lookup_out_offsets(r, sptt):
        sid = plan.by_owner[r][k]
        sh = plan.shards[sid]
        shard = (sh.table_id, sh.rank, sh.scheme, sh.row_range, sh.col_range)
        b0 = (p * plan.S[r] + k) * plan.B
        seg_lens = lens[b0:b0 + plan.B]
        seg_idx = idx[boff[b0]:boff[b0 + plan.B]]
        mat, _ = oracle.towersim_port._shard_pool(placement_tables, shard, seg_lens, seg_idx,
                                                  plan.pooling[sh.table_id])
        for b in range(plan.B):
            buf[off + b * w: off + b * w + w] = mat[b]
    return buf


def alltoallv_np(group, send, send_splits, recv_splits):
    recv = {}
    for j, dst in enumerate(group):
        parts = []
        for i, src in enumerate(group):
            so = int(sum(send_splits[src][:j]))
            parts.append(send[src][so:so + int(send_splits[src][j])])
            assert int(send_splits[src][j]) == int(recv_splits[dst][i])
        recv[dst] = np.concatenate(parts) if parts else np.zeros(0)
    return recv


def assemble_np(fblocks, src, rows, width):
    out = np.zeros((rows, width))
    for fb in fblocks:
        if fb.rowwise:
            acc = np.zeros((rows, fb.width))
            for pc in fb.pieces:
                acc += src[pc.offset:pc.offset + rows * pc.ld].reshape(rows, pc.ld)
            out[:, fb.dst_col:fb.dst_col + fb.width] = acc
        else:
            for pc in fb.pieces:
                blk = src[pc.offset:pc.offset + rows * pc.ld].reshape(rows, pc.ld)
                out[:, fb.dst_col + pc.c0:fb.dst_col + pc.c0 + pc.width] = blk
    return out


def emulate_sptt(plan, tables, lengths, values, ranks=None, a2a=alltoallv_np):
    """Pass-through SPTT forward for `ranks` (default all); returns {rank: (B, out)}."""
    G = plan.G
    ranks = list(range(G)) if ranks is None else ranks
    send = {r: lookup_send_buffer(plan, tables, r, lengths, values, True) for r in range(G)}
    recv_d = {}
    for t in range(plan.T):
        g = plan.layout.tower_ranks(t, plan.topo)
        recv_d.update(a2a(g, send, {r: plan.d_send_splits(r) for r in g}, {r: plan.d_recv_splits(r) for r in g}))
    Y = {r: assemble_np(plan.e_blocks(r), recv_d[r], plan.T * plan.B, plan.x_width(r)).reshape(-1)
         for r in range(G)}
    recv_f = {}
    for c in range(plan.W):
        g = [t * plan.W + c for t in range(plan.T)]
        recv_f.update(a2a(g, Y, {r: plan.f_send_splits(r) for r in g}, {r: plan.f_recv_splits(r) for r in g}))
    out = {}
    for r in ranks:
        o = np.zeros((plan.B, plan.out_width()))
        for col, w, off in plan.out_blocks_tower():
            o[:, col:col + w] = recv_f[r][off:off + plan.B * w].reshape(plan.B, w)
        out[r] = o
    return out


def emulate_flat(plan, tables, lengths, values, a2a=alltoallv_np):
    G = plan.G
    send = {r: lookup_send_buffer(plan, tables, r, lengths, values, False) for r in range(G)}
    world = list(range(G))
    recv = a2a(world, send, {r: plan.c_send_splits(r) for r in world}, {r: plan.c_recv_splits(r) for r in world})
    return {r: assemble_np(plan.c_blocks(), recv[r], plan.B, plan.flat_width()) for r in world}
