"""Debug: distributed (peer / nccl) vs loopback per step, 1 host x 4 ranks."""
import os
import sys

import numpy as np
import torch
import torch.multiprocessing as mp

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))


def worker(rank, world, port, hosts, rph, kind, tmk, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist

    torch.cuda.set_device(rank)
    dev = torch.device("cuda", rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)
    import paper_2403_00877_b200 as P
    from paper_2403_00877_b200.fabric import LoopbackFabric, NcclFabric, PeerFabric
    from paper_2403_00877_b200.sptt import SPTT
    from test_gpu_multi import _build

    topo, layout, placement, assignment, pooling, cfg, kjts, B = _build(hosts, rph, dev)
    if tmk == "none":
        cfg = None
    Fab = PeerFabric if kind == "peer" else NcclFabric
    fab = Fab(world, rank, layout.group_width(topo), dev)
    dm = SPTT(topo, layout, placement, assignment, pooling, B, fab, tm=cfg, dtype=torch.float32, device=dev, lr=0.05)
    topo2, layout2, placement2, _, _, _, kjts2, _ = _build(hosts, rph, dev)
    ref = SPTT(topo2, layout2, placement2, assignment, pooling, B, LoopbackFabric(world, dev), tm=cfg,
               dtype=torch.float32, device=dev, lr=0.05)
    gen = np.random.default_rng(5)
    O = dm.plan.out_width()
    grads = {r: torch.from_numpy(gen.normal(size=(B, O)).astype(np.float32)).to(dev) for r in range(world)}
    lines = []
    for step in range(3):
        od = dm.train_step({rank: kjts[rank]}, {rank: grads[rank]})
        orf = ref.train_step(kjts2, grads)
        torch.cuda.synchronize()
        do = float((od[rank] - orf[rank]).abs().max())
        dw = max(float((dm.engine.weights[s] - ref.engine.weights[s]).abs().max()) for s in dm.engine.weights)
        dt = 0.0
        for t, tm in dm.tms.items():
            for k in tm.w:
                dt = max(dt, float((tm.w[k].float() - ref.tms[t].w[k].float()).abs().max()))
        lines.append(f"rank {rank} step {step}: out {do:.3e} emb {dw:.3e} tm {dt:.3e}")
    q.put("\n".join(lines))
    dist.destroy_process_group()


if __name__ == "__main__":
    hosts, rph = int(sys.argv[1]), int(sys.argv[2])
    world = hosts * rph
    for kind in ("peer", "nccl"):
        for tmk in ("dcn", "none"):
            ctx = mp.get_context("spawn")
            q = ctx.Queue()
            import socket
            s = socket.socket(); s.bind(("127.0.0.1", 0)); port = s.getsockname()[1]; s.close()
            ps = [ctx.Process(target=worker, args=(r, world, port, hosts, rph, kind, tmk, q)) for r in range(world)]
            [p.start() for p in ps]
            res = [q.get(timeout=300) for _ in range(world)]
            [p.join(60) for p in ps]
            print(f"== {kind} tm={tmk} {hosts}x{rph}")
            print("\n".join(sorted(res)), flush=True)
