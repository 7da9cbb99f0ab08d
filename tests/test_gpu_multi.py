"""Multi-GPU (NCCL, one process per GPU) SPTT parity: the distributed train step
must reproduce the single-process loopback engine bit for bit (same kernels,
same reduction orders) and therefore the oracle.  Skipped on boxes with fewer
than 2 GPUs (the driver's round-end GPU tests run on one GPU; run this with
`gpurun --gpus 2|4`)."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _build(hosts, rph, dev, tm_kind="dcn"):
    import paper_2403_00877_b200 as P
    from paper_2403_00877_b200.pipeline import KJT
    from paper_2403_00877_b200.sptt import build_world

    F, rows, N, B = 8, 64, 32, 6
    topo, layout, placement, assignment = build_world(hosts, rph, 1, F, rows, N, seed=4, scheme="column_wise",
                                                      shards_per_table=2)
    G = topo.world_size
    pooling = {f: "sum" for f in range(F)}
    if tm_kind == "dlrm":  # default DLRM flavour: zero-size flat weights (flat_outputs = 0)
        cfg = P.TMConfig(kind="dlrm", out_dim=8, per_feature_outputs=1, flat_outputs=0, seed=1)
    else:
        cfg = P.TMConfig(kind="dcn", out_dim=8, cross_layers=2, seed=1)
    rng = np.random.default_rng(21)
    lens = rng.integers(0, 6, size=(G, F, B)).astype(np.int32)
    vals = rng.integers(0, rows, size=int(lens.sum())).astype(np.int64)
    offs = np.concatenate([[0], np.cumsum(lens.reshape(-1))])
    kjts = {}
    for r in range(G):
        seg = vals[offs[r * F * B]:offs[(r + 1) * F * B]]
        kjts[r] = KJT(torch.from_numpy(lens[r].reshape(-1)).to(dev), torch.from_numpy(seg.astype(np.int32)).to(dev),
                      [int(lens[r, f].sum()) for f in range(F)], B)
    return topo, layout, placement, assignment, pooling, cfg, kjts, B


def _worker(rank, world, port, hosts, rph, q, kind="nccl", steps=1, tm_kind="dcn", mode="sptt", capacity=False):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist

    torch.cuda.set_device(rank)
    dev = torch.device("cuda", rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)
    try:
        import sys

        here = os.path.dirname(os.path.abspath(__file__))
        sys.path.insert(0, os.path.dirname(here))
        from paper_2403_00877_b200.fabric import LoopbackFabric, NcclFabric, PeerFabric
        from paper_2403_00877_b200.sptt import SPTT

        topo, layout, placement, assignment, pooling, cfg, kjts, B = _build(hosts, rph, dev, tm_kind)
        Fab = PeerFabric if kind == "peer" else NcclFabric
        fab = Fab(world, rank, layout.group_width(topo), dev)
        dist_model = SPTT(topo, layout, placement, assignment, pooling, B, fab, tm=cfg, dtype=torch.float32,
                          device=dev, lr=0.005, mode=mode)
        # reference: every rank on this GPU through the loopback fabric
        topo2, layout2, placement2, _, _, _, kjts2, _ = _build(hosts, rph, dev, tm_kind)
        ref = SPTT(topo2, layout2, placement2, assignment, pooling, B, LoopbackFabric(world, dev), tm=cfg,
                   dtype=torch.float32, device=dev, lr=0.005, mode=mode)
        if capacity:  # capacity-padded step a (peer fabric: straight into the owners' buffers)
            caps = [max(kjts[r].nnz_per_feature[f] for r in range(world)) + 3 for f in range(len(pooling))]
            dist_model.set_capacity(caps)
            ref.set_capacity(caps)
        gen = np.random.default_rng(5)
        O = dist_model.out_width
        grads = {r: torch.from_numpy(gen.normal(size=(B, O)).astype(np.float32)).to(dev) for r in range(world)}
        # lr is small: at W = 4 every tower module sees 4B rows and lr 0.05
        # drives the DCN (quadratic in x) into divergence by step 3 -- two
        # diverging trajectories cannot be compared (tools/debug_peer.py).
        # The tower all-reduce of the TM weight gradients sums W contributions
        # in NCCL's ring order; the loopback engine sums them in rank order.
        # For W <= 2 the two agree bit for bit (fp add commutes); for W > 2 the
        # TM weights of step 2+ differ by fp32 reassociation, so later outputs
        # are held to the north-star fp32 tolerance (rtol 1e-5) instead.
        # Step 0 (no weights updated yet) is held to 1e-6 element-wise for any
        # W; later steps at W > 2 to a 1e-4 relative (Frobenius) error, the
        # amplified reassociation of the summed TM gradients.
        # The peer fabric sums the members' TM gradients in tower-rank order
        # (dmt_peer_sum_sgd), exactly as the loopback engine does: outputs,
        # TM weights and embedding shards must then be bit-identical at any W.
        # the group whose dense gradients are all-reduced: the tower (SPTT) or
        # the world (the flat baseline's global TM)
        W = layout.group_width(topo) if mode == "sptt" else topo.world_size
        exact = kind == "peer"
        ok, worst = True, 0.0
        for step in range(steps):  # several steps: peer-written buffers are reused
            out_d = dist_model.train_step({rank: kjts[rank]}, {rank: grads[rank]})
            out_r = ref.train_step(kjts2, grads)
            torch.cuda.synchronize()
            d, r_ = out_d[rank].double(), out_r[rank].double()
            if exact:
                worst = max(worst, float((d - r_).abs().max()))
                ok = ok and torch.equal(out_d[rank], out_r[rank])
            elif step == 0 or W <= 2:
                worst = max(worst, float((d - r_).abs().max()))
                ok = ok and torch.allclose(d, r_, rtol=1e-6, atol=1e-6)
            else:
                rel = float((d - r_).norm() / r_.norm().clamp_min(1e-30))
                worst = max(worst, rel)
                ok = ok and rel <= 1e-4
        for sid in dist_model.engine.weights:
            a, b = dist_model.engine.weights[sid], ref.engine.weights[sid]
            ok = ok and (torch.equal(a, b) if exact else torch.allclose(a, b, rtol=1e-5, atol=1e-6))
        t = rank // W
        if exact and t in dist_model.tms:
            for k, w in dist_model.tms[t].w.items():
                if not torch.equal(w, ref.tms[t].w[k]):
                    ok, worst = False, float((w.double() - ref.tms[t].w[k].double()).abs().max())
        if exact and dist_model.global_tm is not None:
            for k, w in dist_model.global_tm.w.items():
                if not torch.equal(w, ref.global_tm.w[k]):
                    ok, worst = False, float((w.double() - ref.global_tm.w[k].double()).abs().max())
        q.put((rank, bool(ok), None if ok else f"worst out error {worst:.3e}"))
    except Exception:  # pragma: no cover
        import traceback

        q.put((rank, False, traceback.format_exc()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("tm_kind", ["dcn", "dlrm"])
@pytest.mark.parametrize("kind,steps", [("nccl", 1), ("peer", 3)])
@pytest.mark.parametrize("hosts,rph", [(2, 1), (1, 2), (2, 2), (4, 1), (1, 4)])
def test_distributed_step_matches_loopback(hosts, rph, kind, steps, tm_kind):
    world = hosts * rph
    if torch.cuda.device_count() < world:
        pytest.skip(f"needs {world} GPUs")
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, hosts, rph, q, kind, steps, tm_kind)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    for rank, ok, err in res:
        assert ok, f"rank {rank}: {err}"


@pytest.mark.parametrize("kind", ["nccl", "peer"])
@pytest.mark.parametrize("hosts,rph", [(2, 1), (2, 2), (4, 1)])
def test_distributed_flat_baseline_matches_loopback(hosts, rph, kind):
    """The flat all-to-all baseline (global DCN) over NCCL and over the NVLink
    peer-store transport SPTT uses: the peer form (lookup -> receivers'
    buffers, c^-1 -> owners', global TM peer all-reduce) must equal the
    loopback engine bit for bit."""
    world = hosts * rph
    if torch.cuda.device_count() < world:
        pytest.skip(f"needs {world} GPUs")
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, hosts, rph, q, kind, 3, "dcn", "flat"))
             for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    for rank, ok, err in res:
        assert ok, f"rank {rank}: {err}"


@pytest.mark.parametrize("kind", ["nccl", "peer"])
@pytest.mark.parametrize("hosts,rph", [(2, 2), (4, 1)])
def test_distributed_capacity_padded_step_a(hosts, rph, kind):
    """Ragged batches through the capacity-padded step a (static splits; on
    the peer fabric the bucketize stores every slot straight into its owner's
    receive buffers, one barrier instead of two all-to-alls): bit-identical
    to the loopback engine."""
    world = hosts * rph
    if torch.cuda.device_count() < world:
        pytest.skip(f"needs {world} GPUs")
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, hosts, rph, q, kind, 3, "dcn", "sptt", True))
             for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    for rank, ok, err in res:
        assert ok, f"rank {rank}: {err}"
