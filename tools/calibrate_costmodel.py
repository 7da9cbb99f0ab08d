"""Calibrate the exchange cost model on this box and predict the bench layout.

    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 \
        tools/calibrate_costmodel.py [--towers T] [--bench bench_nN.json]

1. Device-times NCCL all-to-alls (CUDA events, max over members) over the
   world group and, concurrently, over every tower group (W ranks) and every
   peer-class group (T ranks) at 1..256 MB per member.
2. Fits alpha / beta / efficiency (costmodel.calibrate; one NVLink host, so
   every group is the scale-up link class).
3. Computes the bytes of one bench step from the exchange plan on the host
   (costmodel.plan_trace: the same per-rank bytes a traced run records, pinned
   against the reference's traces in tests/test_plan_cpu.py) for SPTT and
   flat, and costs them with the fitted parameters: predicted exposed exchange
   per step (a + 2 (d + f) for SPTT -- the backward mirrors d and f -- and
   a + 2 c flat), all as NCCL collectives.
4. With --bench, prints the bench's device-timed exposed exchange alongside.
Rank 0 prints one JSON line.
"""

from __future__ import annotations

import argparse
import json
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2403_00877_b200 import costmodel as cm  # noqa: E402
from paper_2403_00877_b200.simnet import CommTrace  # noqa: E402

SIZES = [1 << 20, 4 << 20, 16 << 20, 64 << 20, 256 << 20]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--towers", type=int, default=2)
    ap.add_argument("--bench", default=None)
    ap.add_argument("--batch", type=int, default=8192)
    ap.add_argument("--tables", type=int, default=26)
    args = ap.parse_args()
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", 0)))
    dev = torch.device("cuda", torch.cuda.current_device())
    dist.init_process_group("nccl", device_id=dev)
    T = args.towers
    W = world // T
    towers = [dist.new_group(list(range(t * W, (t + 1) * W))) for t in range(T)]
    classes = [dist.new_group([t * W + c for t in range(T)]) for c in range(W)]
    samples = []
    samples += cm.measure_alltoall(list(range(world)), SIZES, pg=None)
    if W > 1:
        samples += cm.measure_alltoall(list(range(W)), SIZES, pg=towers[rank // W])
    if T > 1 and W > 1:
        samples += cm.measure_alltoall(list(range(T)), SIZES, pg=classes[rank % W])
    params = cm.calibrate(samples)

    # bytes of one step of the bench layout from the plan (host side, no run):
    # C2 per GPU, fixed pooling 20, bf16 embeddings on the wire, int32 indices
    from paper_2403_00877_b200.embedding import EmbeddingTable, TablePlan, shard_tables
    from paper_2403_00877_b200.plan import ExchangePlan
    from paper_2403_00877_b200.topology import ClusterTopology, TowerLayout
    from paper_2403_00877_b200.towermod import TMConfig, tm_output_width

    # towers model hosts (T "hosts" of W GPUs, sptt.device_world); on one
    # NVSwitch box every group runs over NVLink: scale-out := scale-up
    import dataclasses

    topo, layout = ClusterTopology(T, W), TowerLayout(T, 1)
    params = dataclasses.replace(params, alpha_out=params.alpha_up, beta_out=params.beta_up)
    F, N = args.tables, 128
    base, extra = divmod(F, T)
    assign, f = {}, 0
    for t in range(T):
        for _ in range(base + (1 if t < extra else 0)):
            assign[f] = t
            f += 1
    import numpy as np

    tables = {t: EmbeddingTable(t, 8, N, np.zeros((8, N), dtype=np.float32)) for t in range(F)}
    placement = shard_tables(tables, {t: TablePlan("table_wise", 1, assign[t]) for t in range(F)}, topo, layout)
    feats = list(range(F))
    tm = TMConfig(kind="dcn", out_dim=64, cross_layers=3, seed=0)
    widths = {t: tm_output_width(tm, sum(1 for f in feats if assign[f] == t), N) for t in range(T)}
    pooling = {f: "sum" for f in feats}
    nnz = {r: [args.batch * 20] * F for r in range(world)}
    pred = {}
    for mode in ("sptt", "flat"):
        plan = ExchangePlan(topo, layout if mode == "sptt" else TowerLayout(1, T), placement.shards, feats,
                            {f: N for f in feats}, pooling, args.batch,
                            feature_towers=assign if mode == "sptt" else None, tower_widths=widths)
        tr = cm.plan_trace(plan, nnz, elem_bytes=2, mode=mode)
        c = cm.pipeline_cost(tr, topo, params, layout=layout if mode == "sptt" else None)
        mirrored = sum(v for k, v in c.per_step.items() if k in ("c", "d", "f"))  # backward f^-1 / d^-1 / c^-1
        pred[mode] = {"per_step_ms": {k: v * 1e3 for k, v in c.per_step.items()},
                      "exposed_fwd_ms": c.exposed_comm * 1e3,
                      "exposed_fwd_bwd_ms": (c.exposed_comm + mirrored) * 1e3}
    if rank == 0:
        out = {"world": world, "towers": T, "gpus_per_tower": W,
               "fit": {"alpha_up_us": params.alpha_up * 1e6, "beta_up_GBs": params.beta_up / 1e9,
                       "efficiency": params.efficiency},
               "samples": [{"world": s.world, "MB": s.per_rank_bytes / 2 ** 20, "us": s.seconds * 1e6}
                           for s in samples],
               "predicted": pred}
        if args.bench:
            try:
                b = json.loads(open(args.bench).read().strip().splitlines()[-1])
                out["measured"] = {"sptt_exposed_ms": b.get("exposed_comm_ms_per_step"),
                                   "flat_exposed_ms": (b.get("flat_baseline") or {}).get("exposed_comm_ms_per_step")}
            except Exception as ex:  # pragma: no cover
                out["measured"] = repr(ex)
        print(json.dumps(out), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
