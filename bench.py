"""Benchmark of the DMT / SPTT hot path on B200 (contract: see DESIGN.md §Measurement).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl dmt|reference]

A *step* = one SPTT training pass over one synthetic batch per GPU: step a
bucketing + index all-to-all, pooled lookup, tower exchange, DCN tower module
forward, synthetic upstream gradient, reverse exchange, TM backward + tower
all-reduce + SGD, fused embedding backward/SGD.  N=1 runs BASELINE.json
configs[1] (26 tables x 1M rows x dim 128, pooling 20, batch 8192, DCN TM);
N>1 runs the same per-GPU workload with towers over the GPUs (weak scaling)
and times the flat all-to-all baseline (global DCN) alongside.
Prints ONE JSON line on rank 0.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "samples/sec/box (device-timed) DCN+SPTT at 1/2/4/8 B200; lookup HBM GB/s"
UNIT = "samples/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="dmt", choices=["dmt", "reference"])
    ap.add_argument("--dtype", default="bf16", choices=["bf16", "fp32"])
    ap.add_argument("--tables", type=int, default=26)
    ap.add_argument("--rows", type=int, default=1_000_000)
    ap.add_argument("--dim", type=int, default=128)
    ap.add_argument("--pool", type=int, default=20)
    ap.add_argument("--pool-dist", default="fixed", choices=["fixed", "powerlaw"],
                    help="fixed L = --pool (C2/C3), or power-law lengths with mean --pool, max 200 (C5; ragged "
                         "nnz -> eager steps, no CUDA graph)")
    ap.add_argument("--batch", type=int, default=8192)
    ap.add_argument("--tm", default="dcn", choices=["dcn", "dlrm", "passthrough"])
    ap.add_argument("--tm-out", type=int, default=64)
    ap.add_argument("--cross-layers", type=int, default=3)
    ap.add_argument("--top", default="none", choices=["none", "dcn"],
                    help="full DCN + SPTT model: a data-parallel crossnet head to one logit + BCE loss on "
                         "synthetic labels (instead of a synthetic upstream gradient)")
    ap.add_argument("--towers", type=int, default=0, help="0 = auto (1 at N=1, else 2)")
    ap.add_argument("--no-flat", action="store_true", help="skip the flat-baseline comparison at N>1")
    ap.add_argument("--fabric", default="peer", choices=["peer", "nccl"],
                    help="N>1 SPTT exchange: NVLink peer stores + barrier (peer) or NCCL all-to-alls")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU baseline (profiling runs)")
    ap.add_argument("--cpu-sample", type=int, default=256, help="samples per CPU-baseline step")
    return ap.parse_args()


# --------------------------------------------------------------------------- #
# clocks sampler (nvidia-smi during the timed region)
# --------------------------------------------------------------------------- #
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines: list[str] = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sms, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sms.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        sms.sort()
        med = sms[len(sms) // 2] if sms else None
        return {"sm_mhz": med, "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sms)}


# --------------------------------------------------------------------------- #
# reference arm / CPU baseline: the oracle port on the host cores
# --------------------------------------------------------------------------- #
def cpu_reference_step_fn(args, sample: int):
    """One bounded CPU step of the same workload: oracle pooled lookup over 26
    tables (100k-row slices), DCN tower module forward + backward (float64
    numpy/BLAS) and the embedding SGD update -- the reference algorithm
    restated in oracle/ (the reference itself is forward-only Python)."""
    import numpy as np

    import oracle

    rng = np.random.default_rng(0)
    F, N, L = args.tables, args.dim, args.pool
    rows = min(args.rows, 100_000)
    tables = {t: rng.uniform(-1, 1, (rows, N)).astype(np.float32) for t in range(F)}
    cfg = {"kind": args.tm if args.tm != "passthrough" else "dlrm", "out_dim": args.tm_out,
           "per_feature_outputs": 1, "flat_outputs": 0, "cross_layers": args.cross_layers, "seed": 0}
    w = oracle.init_tm_weights(cfg, F, N, salt=0)
    lens = np.full(sample, L, dtype=np.int64)

    def step():
        idx = {t: rng.integers(0, rows, size=sample * L) for t in range(F)}
        x = np.stack([oracle.pool(tables[t], lens, idx[t], "sum") for t in range(F)], axis=1)
        y = oracle.tm_forward(x, cfg, w)
        dx, dw = oracle.tm_backward(x, cfg, w, np.ones_like(y) / y.size)
        for t in range(F):
            uniq, g = oracle.embedding_row_grads(rows, lens, idx[t], dx[:, t, :])
            tables[t][uniq] -= (0.01 * g).astype(np.float32)
        return y

    return step


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    n = os.cpu_count() or 1
    for v in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):
        os.environ.setdefault(v, str(n))
    step = cpu_reference_step_fn(args, args.cpu_sample)
    for _ in range(args.warmup):
        step()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    dt = time.perf_counter() - t0
    val = args.cpu_sample * args.steps / dt
    sample = (f"{args.cpu_sample} samples/step of the C2 workload ({args.tables} tables, 100k-row slices, "
              f"dim {args.dim}, pooling {args.pool}, {args.tm} TM fwd+bwd + SGD), oracle numpy port, float64")
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": val, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1000 * dt / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": _config(args, args.gpus),
        "cpu_baseline": {"value": val, "unit": UNIT, "cores": n, "kind": "port", "sample": sample},
        "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


def cpu_baseline(args) -> dict:
    """Bounded (~10-30 s) run of the oracle port on this host, single process."""
    import numpy as np  # noqa: F401

    n = os.cpu_count() or 1
    step = cpu_reference_step_fn(args, args.cpu_sample)
    step()
    t0 = time.perf_counter()
    k = 0
    while time.perf_counter() - t0 < 10.0 and k < 50:
        step()
        k += 1
    dt = time.perf_counter() - t0
    return {"value": args.cpu_sample * k / dt, "unit": UNIT, "cores": n, "kind": "port",
            "sample": f"{k} steps x {args.cpu_sample} samples of the C2 workload (100k-row table slices), "
                      f"oracle numpy port (float64; BLAS threads={n} for the TM GEMMs, lookup loops 1 thread)"}


def _config(args, N):
    T = _towers(args, N)
    if args.pool_dist == "powerlaw":
        wl = (f"C5-style: {args.tables} tables x {args.rows} rows x dim {args.dim}, power-law pooling (mean "
              f"{args.pool}, max 200), batch {args.batch}/GPU, {args.tm} TM, SPTT {T} x {N // T}")
    elif N == 1:
        wl = f"C2 (BASELINE configs[1]): 26 tables x 1M rows x dim 128, pooling 20, batch 8192/GPU, {args.tm} TM"
    else:
        wl = f"C2 per GPU, SPTT {T} towers x {N // T} GPUs, flat all-to-all alongside"
    return {"workload": wl,
            "tables": args.tables, "rows": args.rows, "dim": args.dim, "pooling_factor": args.pool,
            "batch_per_gpu": args.batch, "global_batch": args.batch * N, "tm": args.tm, "tm_out_dim": args.tm_out,
            "cross_layers": args.cross_layers, "top": args.top, "towers": T, "gpus_per_tower": N // T, "optimizer": "sgd",
            "pooling_dist": args.pool_dist,
            "parallelism": f"embedding model-parallel in tower, TM data-parallel in tower (T={T}, W={N // T})",
            "exchange": "loopback" if N == 1 else ("nvlink peer stores + barrier" if args.fabric == "peer"
                                                   else "nccl all-to-all"),
            "l2": "inputs larger than L2 (tables >= 6.6 GB bf16, uniform random rows), no flush"}


def _traffic(args, N) -> dict:
    """Per-launch DRAM traffic (dram__bytes_read.sum + dram__bytes_write.sum)
    of the roofline kernels from the committed ncu --set full capture of this
    exact N=1 workload (profiles/traffic.json, written by tools/make_traffic.py);
    {} for any other configuration."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as fh:
            t = json.load(fh)
    except Exception:
        return {}
    want = {"gpus": 1, "tables": args.tables, "rows": args.rows, "dim": args.dim, "pool": args.pool,
            "batch": args.batch, "tm": args.tm, "tm_out": args.tm_out, "cross_layers": args.cross_layers,
            "dtype": args.dtype}
    if N != 1 or any(t.get("config", {}).get(k) != v for k, v in want.items()):
        return {}
    return t.get("kernels", {})


def _towers(args, N):
    if args.towers:
        return args.towers
    return 1 if N == 1 else 2


# --------------------------------------------------------------------------- #
# the B200 arm
# --------------------------------------------------------------------------- #
def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
        return
    import torch
    import torch.distributed as dist

    import paper_2403_00877_b200 as P
    from paper_2403_00877_b200 import _lib
    from paper_2403_00877_b200.fabric import LoopbackFabric, NcclFabric, PeerFabric
    from paper_2403_00877_b200.pipeline import KJT, PhaseTimers
    from paper_2403_00877_b200.sptt import SPTT, device_world, random_kjt

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    N = world
    if args.gpus != N and world == 1 and args.gpus > 1:
        print(json.dumps({"error": f"--gpus {args.gpus} needs torchrun with {args.gpus} processes"}))
        sys.exit(2)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    dtype = torch.bfloat16 if args.dtype == "bf16" else torch.float32
    es = 2 if dtype == torch.bfloat16 else 4
    T = _towers(args, N)
    W = N // T
    topo_args = (T, W, 1)
    B, F, Nd, Lp = args.batch, args.tables, args.dim, args.pool
    topo, layout, placement, assignment = device_world(*topo_args, F, args.rows, Nd, dtype, [rank], seed=0, device=dev)
    pooling = {f: "sum" for f in range(F)}

    def make_fabric(kind="nccl"):
        if world == 1:
            return LoopbackFabric(1, dev)
        return (PeerFabric if kind == "peer" else NcclFabric)(N, rank, W, dev)

    fabric = make_fabric(args.fabric)
    tm_cfg = None if args.tm == "passthrough" else P.TMConfig(kind=args.tm, out_dim=args.tm_out, cross_layers=args.cross_layers,
                                                             per_feature_outputs=1, flat_outputs=0, seed=0)
    top_cfg = (P.TMConfig(kind="dcn", out_dim=1, cross_layers=args.cross_layers, seed=0) if args.top == "dcn"
               else None)
    model = SPTT(topo, layout, placement, assignment, pooling, B, fabric, tm=tm_cfg, dtype=dtype, device=dev,
                 mode="sptt", lr=1e-3, top=top_cfg)
    gen = torch.Generator(device=dev).manual_seed(1234 + rank)
    if args.pool_dist == "powerlaw":
        from paper_2403_00877_b200.sptt import powerlaw_lengths, random_kjt_lengths

        batches = [{rank: random_kjt_lengths(powerlaw_lengths(F, B, 100 * i + rank, mean=float(Lp)), args.rows, gen,
                                             dev)} for i in range(4)]
    else:
        batches = [{rank: random_kjt(F, B, args.rows, Lp, gen, dev)} for _ in range(4)]
    gout = {rank: (torch.randn(B, model.out_width, generator=gen, device=dev) * 1e-3).to(dtype)}
    labels = {rank: (torch.rand(B, generator=gen, device=dev) < 0.25).float()}  # synthetic CTR labels

    def step(m, kj):
        if m.top is not None:
            return m.train_step_bce(kj, labels)
        return m.train_step(kj, gout)

    def barrier():
        if world > 1:
            dist.barrier(device_ids=[local])

    def timed_eager(m, K, Wm):
        """Eager steps with per-phase CUDA events (phase breakdown + fallback)."""
        for i in range(Wm):
            step(m, batches[i % len(batches)])
        torch.cuda.synchronize()
        barrier()
        timers = PhaseTimers()
        m.engine.timers = timers
        calls0 = _lib.CALLS[0]
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for i in range(K):
            step(m, batches[i % len(batches)])
        e.record()
        torch.cuda.synchronize()
        barrier()
        m.engine.timers = None
        return s.elapsed_time(e), timers, (_lib.CALLS[0] - calls0) // max(K, 1)

    def timed_eager_h2d(m, hosts, K):
        """e2e without a CUDA graph (ragged batches): every step copies its
        pinned host KJT to the device, runs the step and reads a scalar back."""
        from paper_2403_00877_b200.pipeline import KJT as _KJT

        out = torch.zeros(1, dtype=torch.float32).pin_memory()
        for i in range(2):
            hl, hv, nz = hosts[i % len(hosts)]
            step(m, {rank: _KJT(hl.to(dev, non_blocking=True), hv.to(dev, non_blocking=True), nz, B)})
        torch.cuda.synchronize()
        barrier()
        s_, e_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s_.record()
        for i in range(K):
            hl, hv, nz = hosts[i % len(hosts)]
            o = step(m, {rank: _KJT(hl.to(dev, non_blocking=True), hv.to(dev, non_blocking=True), nz, B)})
            out.copy_(o[rank].reshape(-1)[:1].float(), non_blocking=True)
        e_.record()
        torch.cuda.synchronize()
        barrier()
        return max_over_ranks(s_.elapsed_time(e_))

    def max_over_ranks(ms):
        t = torch.tensor([ms], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def timed_graph(m, K, host_inputs=None, timers=None):
        """The timed region: K CUDA-graph replays of the whole train step.  Each
        step first copies its batch into the graph's static input buffers
        (device->device, or pinned host->device for e2e) inside the region."""
        st = {rank: KJT(batches[0][rank].lengths.clone(), batches[0][rank].values.clone(),
                        batches[0][rank].nnz_per_feature, B)}
        replay, outs = m.capture(st, gout, timers=timers, labels=labels if m.top is not None else None)
        torch.cuda.synchronize()
        barrier()
        torch.cuda.synchronize()
        if host_inputs is not None:
            # e2e input pipeline: the pinned host batch of step i+1 is copied to
            # a device staging buffer on a copy stream while step i runs; each
            # step's loss is read back to pinned host memory asynchronously.
            cs = torch.cuda.Stream()
            stage = [(torch.empty_like(st[rank].lengths), torch.empty_like(st[rank].values)) for _ in range(2)]
            ready = [torch.cuda.Event() for _ in range(2)]
            free = [torch.cuda.Event() for _ in range(2)]
            losses = torch.zeros(max(K, 1), dtype=torch.float32).pin_memory()
            loss_buf = torch.zeros(max(K, 1), dtype=torch.float32, device=dev)

            def prefetch(j):
                hl, hv, _ = host_inputs[j % len(host_inputs)]
                with torch.cuda.stream(cs):
                    cs.wait_event(free[j % 2])
                    stage[j % 2][0].copy_(hl, non_blocking=True)
                    stage[j % 2][1].copy_(hv, non_blocking=True)
                    ready[j % 2].record(cs)

        def run(n):
            if host_inputs is None:
                for i in range(n):
                    src = batches[i % len(batches)][rank]
                    st[rank].lengths.copy_(src.lengths, non_blocking=True)
                    st[rank].values.copy_(src.values, non_blocking=True)
                    replay()
                return
            for ev in free:
                ev.record()
            prefetch(0)
            for i in range(n):
                cur = i % 2
                torch.cuda.current_stream().wait_event(ready[cur])
                st[rank].lengths.copy_(stage[cur][0], non_blocking=True)
                st[rank].values.copy_(stage[cur][1], non_blocking=True)
                free[cur].record()
                if i + 1 < n:
                    prefetch(i + 1)
                replay()
                if m.top is not None:  # the BCE loss of this step
                    loss_buf[i:i + 1].copy_(outs[rank])
                else:  # <y, g> of the synthetic upstream gradient
                    torch.dot(outs[rank].view(-1).float(), gout[rank].view(-1).float(), out=loss_buf[i])
                losses[i:i + 1].copy_(loss_buf[i:i + 1], non_blocking=True)

        run(min(K, max(3, args.warmup)))  # untimed warm-up of this exact loop
        torch.cuda.synchronize()
        barrier()
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        run(K)
        e.record()
        torch.cuda.synchronize()
        barrier()
        return max_over_ranks(s.elapsed_time(e))

    # per-phase breakdown (eager, instrumented) -- also the fallback timing
    eager_ms, timers, calls = timed_eager(model, args.steps, args.warmup)
    ph = {k: v / args.steps for k, v in timers.ms().items()}
    ph_source = "eager"
    graph_ok = True
    clocks = ClockSampler(local)
    clocks.start()
    gtimers = PhaseTimers(external=True)
    try:
        if args.pool_dist != "fixed":
            raise RuntimeError("ragged per-batch nnz: eager steps (step-a counts exchange per batch)")
        total_ms = timed_graph(model, args.steps, timers=gtimers)
        # phases of the last replay (events are graph nodes, re-recorded each replay)
        ph = {k: v for k, v in gtimers.ms().items()}
        ph_source = "cuda-graph replay"
    except Exception as ex:  # capture unsupported (e.g. collective backend): eager numbers
        graph_ok = False
        graph_err = repr(ex)[:200]
        total_ms = max_over_ranks(eager_ms)
    clk = clocks.stop()
    ms_step = total_ms / args.steps
    value = N * B * args.steps / (total_ms / 1000.0)

    # e2e through the public API with host (pinned) inputs
    e2e = None
    if not args.no_e2e:
        hosts = []
        for bt in batches:
            kj = bt[rank]
            hosts.append((kj.lengths.cpu().pin_memory(), kj.values.cpu().pin_memory(), kj.nnz_per_feature))
        if graph_ok:
            e_ms = timed_graph(model, args.steps, host_inputs=hosts)
        else:  # eager: H2D of each step's KJT from pinned host memory inside the region
            e_ms = timed_eager_h2d(model, hosts, args.steps)
        h2d = hosts[0][0].numel() * 4 + hosts[0][1].numel() * 4
        e2e = {"value": N * B * args.steps / (e_ms / 1000.0), "unit": UNIT, "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": 4}

    # roofline of the lookup kernel: algorithmic bytes per launch
    p = model.plan
    bags = p.owner_bags(rank)
    nnz = model.engine._owner[rank][2] if args.pool_dist != "fixed" else bags * Lp
    look_bytes = nnz * Nd * es + nnz * 4 + (bags + 1) * 8 + bags * Nd * es
    import json as _j

    peaks = {}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            peaks = _j.load(fh)
        hbm, tf = peaks["hbm_gbs"], peaks["bf16_tflops_sustained"]
        peak_src = "measured (MEASURED_PEAKS.json)"
    except Exception:
        hbm, tf = 6650.0, 1400.0
        peak_src = "fallback (B200_PROFILING.md)"
    traffic = _traffic(args, N)
    n_look = max(1, timers.count("lookup_fwd") // args.steps)
    look_ms = ph.get("lookup_fwd", 0.0) / n_look
    look_gbs = look_bytes / (look_ms * 1e-3) / 1e9 if look_ms else 0.0
    tl = traffic.get("pooled_fwd", {})
    roof_lookup = {"bound": "hbm", "achieved": look_gbs, "peak": hbm, "unit": "GB/s", "frac": look_gbs / hbm,
                   "traffic": tl.get("dram_bytes_per_launch"), "traffic_source": tl.get("source"),
                   "kernel": "dmt::pooled_fwd_kernel", "algorithmic_bytes": look_bytes,
                   "launch_ms": look_ms, "peak_source": peak_src}
    roof = roof_lookup
    if tm_cfg is not None and args.tm == "dcn":
        t_own = p.tower_of(rank)
        Ft = len(p.tower_features[t_own])
        rows = p.T * B
        fwd = P.tm_flops(tm_cfg, Ft, Nd, rows)
        tm_flops_step = 3.0 * fwd  # fwd + (dX, dW) backward
        tm_ms = ph.get("tm_fwd", 0.0) + ph.get("tm_bwd", 0.0)
        if top_cfg is not None:  # the head's crossnet GEMMs over the SPTT output
            tm_flops_step += 3.0 * P.tm_flops(top_cfg, 1, model.out_width, B)
            tm_ms += ph.get("top_fwd", 0.0) + ph.get("top_bwd", 0.0)
        if tm_ms > look_ms:
            ach = tm_flops_step / (tm_ms * 1e-3) / 1e12
            tg = traffic.get("gemm_dcn_step", {})
            nl = tg.get("launches")
            roof = {"bound": "tensor", "achieved": ach, "peak": tf, "unit": "TFLOP/s", "frac": ach / tf,
                    "traffic": tg.get("dram_bytes_per_launch"), "traffic_source": tg.get("source"),
                    "kernel": "dmt::gemm::gemm_kernel (the DCN fwd+bwd GEMMs of one step)",
                    "launches_per_step": nl,
                    "algorithmic_flops": tm_flops_step,
                    "algorithmic_flops_per_launch": tm_flops_step / nl if nl else None,
                    "ms": tm_ms, "ms_note": "tm_fwd + tm_bwd phases (CUDA events): GEMMs plus the small "
                                           "column-sum / copy kernels between them, so achieved is a lower bound",
                    "peak_source": peak_src + " bf16 sustained"}
    result = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": N, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": args.dtype, "data": "synthetic (uniform random rows, random-init tables and TM weights)",
        "config": _config(args, N), "roofline": roof, "roofline_lookup": roof_lookup,
        "lookup_hbm_gbs": look_gbs, "phases_ms_per_step": ph, "phases_source": ph_source, "cuda_graph": graph_ok,
        "eager_ms_per_step": max_over_ranks(eager_ms) / args.steps,
        "exposed_comm_ms_per_step": ph.get("exchange", 0.0), "clocks": clk, "e2e": e2e,
        "gpu_launches": calls * args.steps,
        "gpu_launches_note": "libdmt entry-point calls per step x steps (each >= 1 kernel; replayed from a CUDA graph)",
    }
    # flat all-to-all baseline alongside (N > 1)
    if N > 1 and not args.no_flat:
        del model
        torch.cuda.empty_cache()
        flat = SPTT(topo, layout, placement, assignment, pooling, B, fabric, tm=tm_cfg, dtype=dtype, device=dev,
                    mode="flat", lr=1e-3, top=top_cfg)
        gout = {rank: (torch.randn(B, flat.out_width, generator=gen, device=dev) * 1e-3).to(dtype)}
        fe_ms, f_t, _ = timed_eager(flat, args.steps, args.warmup)
        fph = {k: v / args.steps for k, v in f_t.ms().items()}
        try:
            ft = PhaseTimers(external=True)
            f_ms = timed_graph(flat, args.steps, timers=ft) if graph_ok else max_over_ranks(fe_ms)
            if graph_ok:
                fph = {k: v for k, v in ft.ms().items()}
        except Exception:
            f_ms = max_over_ranks(fe_ms)
        result["flat_baseline"] = {"value": N * B * args.steps / (f_ms / 1000.0), "ms_per_step": f_ms / args.steps,
                                   "exposed_comm_ms_per_step": fph.get("exchange", 0.0), "phases_ms_per_step": fph}
    if rank == 0 and N == 1 and not args.no_cpu:
        result["cpu_baseline"] = cpu_baseline(args)
    if not graph_ok:
        result["cuda_graph_error"] = graph_err
    if rank == 0:
        print(json.dumps(result), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
