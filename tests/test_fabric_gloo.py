"""Multi-process (gloo, CPU) test of the distributed exchange protocol.

Each process is one rank and runs the real NcclFabric class (its
torch.distributed group construction, split handling and count exchange)
with the gloo backend on CPU tensors; the device kernels are replaced by the
numpy plan emulation.  The per-rank SPTT / flat outputs must equal the
oracle's (the reference's) for 2x1, 2x2 and 4x1 layouts, and the tower
all-reduce must sum TM gradients inside each tower only.
"""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, hosts, rph, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import sys

        here = os.path.dirname(os.path.abspath(__file__))
        sys.path.insert(0, here)
        sys.path.insert(0, os.path.dirname(here))
        import oracle
        import paper_2403_00877_b200 as P
        from paper_2403_00877_b200.fabric import NcclFabric
        from paper_2403_00877_b200.plan import ExchangePlan
        from plan_emulation import assemble_np, lookup_send_buffer

        topo = P.ClusterTopology(hosts, rph)
        layout = P.TowerLayout(hosts)
        F, rows, N, B = 6, 30, 4, 3
        feats = list(range(F))
        assignment = {f: min(f * hosts // F, hosts - 1) for f in feats}
        tabs = oracle.uniform_tables({f: (rows, N) for f in feats}, 3)
        tables = {f: P.EmbeddingTable(f, rows, N, tabs[f]) for f in feats}
        placement = P.shard_tables(tables, {f: P.TablePlan("column_wise", 2 if rph > 1 else 1, assignment[f])
                                            for f in feats}, topo, layout)
        lengths, values, pooling = oracle.make_bags(world, {f: rows for f in feats}, B, {f: (0, 4) for f in feats}, 5)
        plan = ExchangePlan(topo, layout, placement.shards, feats, {f: N for f in feats}, pooling, B,
                            feature_towers=assignment)
        fab = NcclFabric(world, rank, layout.group_width(topo), torch.device("cpu"))

        def a2a(group, send, ss, rs):
            out = {rank: torch.zeros(max(1, int(sum(rs[rank]))), dtype=torch.float64)}
            fab.alltoallv(group, "x", {rank: torch.from_numpy(send[rank])}, ss, out, rs)
            return {rank: out[rank].numpy()}

        # step a counts exchange (the only host-synchronising collective)
        nnz = [int(lengths[rank, f].sum()) for f in feats]
        counts = fab.exchange_counts(list(range(world)), {rank: plan.a_send_value_splits(nnz)})
        want_counts = [plan.a_send_value_splits([int(lengths[p, f].sum()) for f in feats])[rank]
                       for p in range(world)]
        assert counts[rank] == want_counts
        # steps b-f for this rank only
        send = {rank: lookup_send_buffer(plan, tabs, rank, lengths, values, True)}
        rd = a2a(plan.group_of(rank), send, {r: plan.d_send_splits(r) for r in plan.group_of(rank)},
                 {r: plan.d_recv_splits(r) for r in plan.group_of(rank)})
        X = assemble_np(plan.e_blocks(rank), rd[rank], plan.T * plan.B, plan.x_width(rank)).reshape(-1)
        cg = plan.class_group_of(rank)
        rf = a2a(cg, {rank: X}, {r: plan.f_send_splits(r) for r in cg}, {r: plan.f_recv_splits(r) for r in cg})
        out = np.zeros((B, plan.out_width()))
        for col, w, off in plan.out_blocks_tower():
            out[:, col:col + w] = rf[rank][off:off + B * w].reshape(B, w)
        shards = [(s.table_id, s.rank, s.scheme, s.row_range, s.col_range) for s in placement.shards]
        want, _, _, _ = oracle.tower_forward(lengths, values, feats, pooling, tabs, shards, assignment,
                                             oracle.OTopo(hosts, rph))
        ok = np.array_equal(out, want[rank])
        # the flat baseline's step c over the world, same lookup kernels' layout
        world_g = list(range(world))
        sc = {rank: lookup_send_buffer(plan, tabs, rank, lengths, values, False)}
        rc = a2a(world_g, sc, {r: plan.c_send_splits(r) for r in world_g}, {r: plan.c_recv_splits(r) for r in world_g})
        flat = assemble_np(plan.c_blocks(), rc[rank], B, plan.flat_width())
        want_flat, _, _, _ = oracle.baseline_forward(lengths, values, feats, pooling, tabs, shards,
                                                     oracle.OTopo(hosts, rph))
        ok = ok and np.array_equal(flat.reshape(B, -1), want_flat[rank])
        # tower all-reduce: sum of rank ids over the tower's ranks
        g = {"w": torch.full((3,), float(rank))}
        fab.all_reduce_(plan.group_of(rank), g)
        ok = ok and float(g["w"][0]) == float(sum(plan.group_of(rank)))
        q.put((rank, bool(ok), None))
    except Exception as e:  # pragma: no cover - surfaced by the parent
        import traceback

        q.put((rank, False, traceback.format_exc()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("hosts,rph", [(2, 1), (2, 2), (4, 1), (2, 4), (4, 2)])
def test_sptt_protocol_over_gloo(hosts, rph):
    """Process-per-rank SPTT (steps a-f) and flat (step c) protocol, including
    the north-star 8-rank layouts 2 towers x 4 and 4 towers x 2."""
    world = hosts * rph
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, hosts, rph, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    for rank, ok, err in res:
        assert ok, f"rank {rank}: {err}"
