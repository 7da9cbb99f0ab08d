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
                         "nnz through the capacity-padded step a, CUDA-graph replayed)")
    ap.add_argument("--batch", type=int, default=8192)
    ap.add_argument("--tm", default="dcn", choices=["dcn", "dlrm", "passthrough"])
    ap.add_argument("--tm-out", type=int, default=64)
    ap.add_argument("--cross-layers", type=int, default=3)
    ap.add_argument("--model", default="dcn", choices=["dcn", "dlrm"],
                    help="dcn: the DCN tower-module SPTT step (C2 / C4); dlrm: the C3 model -- DLRM (bottom MLP, "
                         "dot interaction, top MLP, BCE) around SPTT with DLRM tower modules (c=1, p=0, D=--tm-out); "
                         "the flat baseline interacts the full embeddings")
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
    ap.add_argument("--no-c1", action="store_true", help="skip the C1 reference-API legs")
    ap.add_argument("--lr", type=float, default=1e-2, help="embedding (sparse) learning rate")
    ap.add_argument("--dense-lr", type=float, default=1e-4, help="tower-module / head learning rate")
    ap.add_argument("--no-fp32", action="store_true", help="skip the fp32 C2 record at N=1")
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


# --------------------------------------------------------------------------- #
# C1 through the reference's public API (BASELINE configs[0]):
# the same harness drives the reference package (towersim, installed in
# baseline/_ref) on the host cores and this package on the GPU
# --------------------------------------------------------------------------- #
C1 = dict(hosts=2, ranks_per_host=4, towers=2, tables=26, rows=100_000, dim=64, batch=512, lo=10, hi=30)


def c1_inputs(TS, multi_hot: bool):
    """C1: ClusterTopology(2, 4), TowerLayout(2), 26 float32 U(-1, 1) tables
    (default_rng([0, t]), embedding.py:58-60) x 100k rows x 64, features
    0-12 -> tower 0, 13-25 -> tower 1, table-wise; B = 512 per rank, single-hot
    or L ~ U[10, 30]; batch seed 1 (make_batch, embedding.py:259-295)."""
    import numpy as np

    c = C1
    topo = TS.ClusterTopology(c["hosts"], c["ranks_per_host"])
    layout = TS.TowerLayout(c["towers"])
    tables = {t: TS.EmbeddingTable(t, c["rows"], c["dim"], np.random.default_rng([0, t]).uniform(
        -1.0, 1.0, size=(c["rows"], c["dim"])).astype(np.float32)) for t in range(c["tables"])}
    assignment = {t: (0 if t < c["tables"] // 2 else 1) for t in range(c["tables"])}
    placement = TS.shard_tables(tables, {t: TS.TablePlan("table_wise", 1, assignment[t]) for t in tables}, topo,
                                layout)
    hot = {t: ((c["lo"], c["hi"]) if multi_hot else 1) for t in tables}
    batch = TS.make_batch(topo, tables, c["batch"], hot, seed=1)
    return topo, placement, batch, TS.TowerPlan(layout, assignment)


def c1_time(TS, repeats: int = 3) -> dict:
    """samples/s = G * B / wall of tower_exchange (SPTT) and baseline_exchange
    (flat), best of ``repeats`` after one warm-up, single- and multi-hot."""
    out = {}
    G = C1["hosts"] * C1["ranks_per_host"]
    for multi in (False, True):
        topo, placement, batch, plan = c1_inputs(TS, multi)
        for name, fn in (("tower_exchange", lambda: TS.tower_exchange(batch, placement, plan, topo)),
                         ("baseline_exchange", lambda: TS.baseline_exchange(batch, placement, topo))):
            fn()
            best = float("inf")
            for _ in range(repeats):
                t0 = time.perf_counter()
                fn()
                best = min(best, time.perf_counter() - t0)
            out[f"{name}_{'multi' if multi else 'single'}_hot"] = {"samples_per_s": G * C1["batch"] / best,
                                                                    "wall_s": best}
    return out


def reference_c1() -> dict:
    """The reference's own forward path (towersim 0.1.0 from baseline/_ref,
    pip-installed from /root/reference) at full-size C1 on the host cores."""
    ref = os.path.join(ROOT, "baseline", "_ref")
    if ref not in sys.path:
        sys.path.insert(0, ref)
    try:
        import towersim as TS  # noqa: N812
    except Exception as ex:
        return {"unavailable": f"towersim not importable from baseline/_ref: {ex!r}"[:200]}
    n = os.cpu_count() or 1
    res = c1_time(TS)
    res.update({"impl": "towersim 0.1.0 (the reference, unmodified, baseline/_ref)", "cores": n,
                "threads_note": "lookup / exchange loops are single-threaded Python; BLAS threads only for TMs",
                "workload": "C1 (BASELINE configs[0]): 8 simulated ranks 2 towers x 4, 26 tables x 100k x 64 "
                            "float32, B = 512 / rank, pass-through TMs, forward only (the reference has no "
                            "backward)"})
    return res


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
    cfg = _config(args, args.gpus)
    # what this arm actually ran: a bounded sample of the workload
    cfg.update({"workload": "bounded CPU sample of " + cfg["workload"] + f": {args.cpu_sample} samples per step, "
                            f"26 tables sliced to {min(args.rows, 100_000)} rows, float64",
                "rows": min(args.rows, 100_000), "batch_per_gpu": args.cpu_sample,
                "global_batch": args.cpu_sample, "exchange": "none (one process)"})
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": val, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1000 * dt / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": cfg,
        "cpu_baseline": {"value": val, "unit": UNIT, "cores": n, "kind": "port", "sample": sample},
        "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "reference_c1": reference_c1() if not args.no_c1 else None,
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
    if args.model == "dlrm":
        wl = (f"C3-style DLRM + SPTT: {args.tables} tables x {args.rows} rows x dim {args.dim}, pooling {args.pool}, "
              f"batch {args.batch}/GPU, DLRM tower modules D={args.tm_out}, 13 dense features, bottom 512-256-D, "
              f"top 512-256-1, SPTT {T} x {N // T}")
    elif args.pool_dist == "powerlaw":
        wl = (f"C5-style: {args.tables} tables x {args.rows} rows x dim {args.dim}, power-law pooling (mean "
              f"{args.pool}, max 200), batch {args.batch}/GPU, {args.tm} TM, SPTT {T} x {N // T}")
    elif N == 1:
        wl = f"C2 (BASELINE configs[1]): 26 tables x 1M rows x dim 128, pooling 20, batch 8192/GPU, {args.tm} TM"
    else:
        wl = f"C2 per GPU, SPTT {T} towers x {N // T} GPUs, flat all-to-all alongside"
    return {"workload": wl,
            "tables": args.tables, "rows": args.rows, "dim": args.dim, "pooling_factor": args.pool,
            "batch_per_gpu": args.batch, "global_batch": args.batch * N, "tm": args.tm, "tm_out_dim": args.tm_out,
            "cross_layers": args.cross_layers, "top": args.top, "model": args.model, "towers": T, "gpus_per_tower": N // T, "optimizer": "sgd",
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
def _log(msg):
    if os.environ.get("DMT_BENCH_VERBOSE"):
        print(f"[bench] {msg}", file=sys.stderr, flush=True)


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            pk = json.load(fh)
        return pk["hbm_gbs"], pk["bf16_tflops"], pk.get("bf16_tflops_sustained"), "measured (MEASURED_PEAKS.json)"
    except Exception:
        return 6650.0, 1650.0, None, "fallback (B200_PROFILING.md)"


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
        return
    import torch
    import torch.distributed as dist

    import paper_2403_00877_b200 as P
    from paper_2403_00877_b200 import _lib
    from paper_2403_00877_b200 import kernels as K
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
    T = _towers(args, N)
    W = N // T
    B, F, Nd, Lp = args.batch, args.tables, args.dim, args.pool
    pooling = {f: "sum" for f in range(F)}
    hbm, tf_burst, tf_sust, peak_src = _peaks()

    def make_fabric(kind="nccl"):
        if world == 1:
            return LoopbackFabric(1, dev)
        return (PeerFabric if kind == "peer" else NcclFabric)(N, rank, W, dev)

    fabric = make_fabric(args.fabric)
    if args.model == "dlrm":
        args.tm = "dlrm"
    tm_cfg = None if args.tm == "passthrough" else P.TMConfig(kind=args.tm, out_dim=args.tm_out, cross_layers=args.cross_layers,
                                                             per_feature_outputs=1, flat_outputs=0, seed=0)
    top_cfg = (P.TMConfig(kind="dcn", out_dim=1, cross_layers=args.cross_layers, seed=0) if args.top == "dcn"
               else None)

    def barrier():
        if world > 1:
            dist.barrier(device_ids=[local])

    def max_over_ranks(ms):
        t = torch.tensor([ms], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    class Arm:
        """One model + its synthetic batches in one compute dtype."""

        def __init__(self, dtype, mode="sptt"):
            self.dtype = dtype
            self.es = 2 if dtype == torch.bfloat16 else 4
            topo, layout, placement, assignment = device_world(T, W, 1, F, args.rows, Nd, dtype, [rank], seed=0,
                                                               device=dev)
            dlrm = args.model == "dlrm"
            self.model = SPTT(topo, layout, placement, assignment, pooling, B, fabric,
                              tm=(None if dlrm and mode == "flat" else tm_cfg), dtype=dtype,
                              device=dev, mode=mode, lr=args.lr, dense_lr=args.dense_lr,
                              top=None if dlrm else top_cfg)
            self.dlrm = None
            if dlrm:
                from paper_2403_00877_b200.dlrm import DLRM

                self.dlrm = DLRM(self.model, 16, bottom=(512, 256), top=(512, 256), seed=0)
            gen = torch.Generator(device=dev).manual_seed(1234 + rank)
            if args.pool_dist == "powerlaw":
                from paper_2403_00877_b200.sptt import powerlaw_lengths, random_kjt_lengths

                self.batches = [{rank: random_kjt_lengths(powerlaw_lengths(F, B, 100 * i + rank, mean=float(Lp)),
                                                          args.rows, gen, dev)} for i in range(4)]
                # capacity-padded step a: per-feature capacity = the largest
                # nnz of any rank's batch (no count exchange, CUDA-graph capturable)
                cap = torch.tensor([max(bt[rank].nnz_per_feature[f] for bt in self.batches) for f in range(F)],
                                   dtype=torch.int64, device=dev)
                if world > 1:
                    dist.all_reduce(cap, op=dist.ReduceOp.MAX)
                cap = [(int(c) + 63) // 64 * 64 for c in cap.cpu()]
                self.model.set_capacity(cap)
            else:
                self.batches = [{rank: random_kjt(F, B, args.rows, Lp, gen, dev)} for _ in range(4)]
            self.gout = {rank: (torch.randn(B, self.model.out_width, generator=gen, device=dev) * 1e-3).to(dtype)}
            self.labels = {rank: (torch.rand(B, generator=gen, device=dev) < 0.25).float()}  # synthetic CTR labels
            # 13 Criteo-like dense features (padded to 16 columns, zero)
            self.dense = {rank: torch.nn.functional.pad(torch.randn(B, 13, generator=gen, device=dev), (0, 3)).to(dtype)}

        def step(self, kj):
            m = self.model
            if self.dlrm is not None:
                return self.dlrm.train_step(kj, self.dense, self.labels)
            if m.top is not None:
                return m.train_step_bce(kj, self.labels)
            return m.train_step(kj, self.gout)

        def timed_eager(self, K_, Wm):
            """Eager steps with per-phase CUDA events (phase breakdown + fallback)."""
            m = self.model
            for i in range(Wm):
                self.step(self.batches[i % len(self.batches)])
            torch.cuda.synchronize()
            barrier()
            timers = PhaseTimers()
            m.engine.timers = timers
            calls0 = _lib.CALLS[0]
            s_, e_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s_.record()
            for i in range(K_):
                self.step(self.batches[i % len(self.batches)])
            e_.record()
            torch.cuda.synchronize()
            barrier()
            m.engine.timers = None
            return s_.elapsed_time(e_), timers, (_lib.CALLS[0] - calls0) // max(K_, 1)

        def timed_eager_h2d(self, hosts, K_):
            """e2e without a CUDA graph (ragged batches): every step copies its
            pinned host KJT to the device, runs the step and reads a scalar back."""
            out = torch.zeros(1, dtype=torch.float32).pin_memory()
            for i in range(2):
                hl, hv, nz = hosts[i % len(hosts)]
                self.step({rank: KJT(hl.to(dev, non_blocking=True), hv.to(dev, non_blocking=True), nz, B)})
            torch.cuda.synchronize()
            barrier()
            s_, e_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s_.record()
            for i in range(K_):
                hl, hv, nz = hosts[i % len(hosts)]
                o = self.step({rank: KJT(hl.to(dev, non_blocking=True), hv.to(dev, non_blocking=True), nz, B)})
                out.copy_(o[rank].reshape(-1)[:1].float(), non_blocking=True)
            e_.record()
            torch.cuda.synchronize()
            barrier()
            return max_over_ranks(s_.elapsed_time(e_))

        def capture(self, timers=None):
            m = self.model
            v0 = self.batches[0][rank].values
            if m.engine.capacity is not None:  # ragged: a static values buffer of the capacity
                vals = torch.zeros(sum(m.engine.capacity), dtype=v0.dtype, device=dev)
                vals[: v0.numel()].copy_(v0)
            else:
                vals = v0.clone()
            self.st = {rank: KJT(self.batches[0][rank].lengths.clone(), vals,
                                 self.batches[0][rank].nnz_per_feature, B)}
            if self.dlrm is not None:
                self.replay, self.outs = self.dlrm.capture(self.st, self.dense, self.labels, timers=timers)
            else:
                self.replay, self.outs = m.capture(self.st, self.gout, timers=timers,
                                                   labels=self.labels if m.top is not None else None)
            torch.cuda.synchronize()

        def timed_graph(self, K_, host_inputs=None):
            """The timed region: K CUDA-graph replays of the whole train step.  Each
            step first copies its batch into the graph's static input buffers
            (device->device, or pinned host->device for e2e) inside the region."""
            m, st, outs = self.model, self.st, self.outs
            barrier()
            torch.cuda.synchronize()
            if host_inputs is not None:
                # e2e input pipeline: the pinned host batch of step i+1 is copied to
                # a device staging buffer on a copy stream while step i runs; each
                # step's loss is read back to pinned host memory asynchronously.
                cs = torch.cuda.Stream()
                nv = max(h[1].numel() for h in host_inputs)
                stage = [(torch.empty_like(st[rank].lengths), torch.empty(nv, dtype=st[rank].values.dtype, device=dev))
                         for _ in range(2)]
                ready = [torch.cuda.Event() for _ in range(2)]
                free = [torch.cuda.Event() for _ in range(2)]
                losses = torch.zeros(max(K_, 1), dtype=torch.float32).pin_memory()
                loss_buf = torch.zeros(max(K_, 1), dtype=torch.float32, device=dev)

                def prefetch(j):
                    hl, hv, _ = host_inputs[j % len(host_inputs)]
                    with torch.cuda.stream(cs):
                        cs.wait_event(free[j % 2])
                        stage[j % 2][0].copy_(hl, non_blocking=True)
                        stage[j % 2][1][: hv.numel()].copy_(hv, non_blocking=True)
                        ready[j % 2].record(cs)

            def run(n):
                if host_inputs is None:
                    for i in range(n):
                        src = self.batches[i % len(self.batches)][rank]
                        st[rank].lengths.copy_(src.lengths, non_blocking=True)
                        st[rank].values[: src.values.numel()].copy_(src.values, non_blocking=True)
                        self.replay()
                    return
                for ev in free:
                    ev.record()
                prefetch(0)
                for i in range(n):
                    cur = i % 2
                    torch.cuda.current_stream().wait_event(ready[cur])
                    st[rank].lengths.copy_(stage[cur][0], non_blocking=True)
                    nvi = host_inputs[i % len(host_inputs)][1].numel()
                    st[rank].values[:nvi].copy_(stage[cur][1][:nvi], non_blocking=True)
                    free[cur].record()
                    if i + 1 < n:
                        prefetch(i + 1)
                    self.replay()
                    if m.top is not None or self.dlrm is not None:  # the BCE loss of this step
                        loss_buf[i:i + 1].copy_(outs[rank])
                    else:  # <y, g> of the synthetic upstream gradient
                        torch.dot(outs[rank].view(-1).float(), self.gout[rank].view(-1).float(), out=loss_buf[i])
                    losses[i:i + 1].copy_(loss_buf[i:i + 1], non_blocking=True)

            run(min(K_, max(3, args.warmup)))  # untimed warm-up of this exact loop
            torch.cuda.synchronize()
            barrier()
            torch.cuda.synchronize()
            s_, e_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s_.record()
            run(K_)
            e_.record()
            torch.cuda.synchronize()
            barrier()
            return max_over_ranks(s_.elapsed_time(e_))

        def measure(self, K_, Wm, clocks=None):
            """Eager phase breakdown, then the CUDA-graph timed region."""
            eager_ms, timers, calls = self.timed_eager(K_, Wm)
            self.eager_timers = timers
            ph = {k: v / K_ for k, v in timers.ms().items()}
            src, graph_ok, err = "eager", True, None
            if clocks is not None:
                clocks.start()
            # the events are graph nodes: they must live as long as the graph
            gtimers = self.gtimers = PhaseTimers(external=True)
            try:
                self.capture(timers=gtimers)
                total = self.timed_graph(K_)
                ph = dict(gtimers.ms())  # phases of the last replay (events are graph nodes)
                src = "cuda-graph replay"
            except Exception as ex:  # capture unsupported (e.g. collective backend): eager numbers
                graph_ok, err = False, repr(ex)[:200]
                total = max_over_ranks(eager_ms)
            clk = clocks.stop() if clocks is not None else None
            return {"total_ms": total, "ms_step": total / K_, "ph": ph, "ph_source": src, "graph_ok": graph_ok,
                    "graph_err": err, "eager_ms_step": max_over_ranks(eager_ms) / K_, "calls": calls, "clocks": clk}

        # -- algorithmic bytes / flops of one step on this rank -------------------
        def lookup_bytes(self):
            p = self.model.plan
            bags = p.owner_bags(rank)
            nnz = int(self.model.engine._owner[rank][0][-1])  # actual occurrences (capacity mode pads)
            return nnz * Nd * self.es + nnz * 4 + (bags + 1) * 8 + bags * Nd * self.es, nnz, bags

        def unique_rows(self):
            """Unique (shard, row) keys the last forward touched on this owner."""
            eng = self.model.engine
            offsets, vals, nnz = eng._owner[rank]
            off = offsets.cpu()
            keys = []
            for seg in eng.seg_bwd[rank].segments:
                a, b = int(off[seg.bag_begin]), int(off[seg.bag_begin + seg.nbags])
                keys.append(vals[a:b].long() + seg.key_base)
            return int(torch.unique(torch.cat(keys)).numel()) if keys else 0

        def bwd_bytes(self, nnz, bags, U):
            return bags * Nd * self.es + nnz * 4 + 2 * U * Nd * self.es

        def tm_flops(self):
            if tm_cfg is None or args.tm != "dcn":
                return 0.0
            p = self.model.plan
            Ft = len(p.tower_features[p.tower_of(rank)]) if self.model.global_tm is None else F
            fl = 3.0 * P.tm_flops(tm_cfg, Ft, Nd, (p.T if self.model.global_tm is None else 1) * B)
            if top_cfg is not None:
                fl += 3.0 * P.tm_flops(top_cfg, 1, self.model.out_width, B)
            return fl

        def exchange_bytes(self):
            """Bytes this rank sends to other ranks per step (forward + backward
            mirrors, + the tower all-reduce of the TM gradients at W > 1)."""
            p = self.model.plan
            if p.G == 1:
                return 0, {}
            nnz_pf = self.batches[0][rank].nnz_per_feature
            vs = p.a_send_value_splits(nnz_pf)
            ls = p.a_send_length_splits()
            a = sum((vs[o] + ls[o]) * 4 for o in range(p.G) if o != rank)
            bpr = p.bytes_per_rank(self.es)
            parts = {"a": a}
            if self.model.engine.mode == "flat":
                parts["c"] = 2 * bpr["c"]
            else:
                parts["d"] = 2 * bpr.get("d", 0)
                parts["f"] = 2 * bpr.get("f", 0)
                t = p.tower_of(rank)
                if W > 1 and t in self.model.tms:
                    nw = sum(v.numel() for v in self.model.tms[t].w.values())
                    parts["tm_allreduce"] = int(2 * (W - 1) / W * nw * 4)
            return sum(parts.values()), parts

    # ---- headline: bf16 (or --dtype) SPTT --------------------------------------
    dtype = torch.bfloat16 if args.dtype == "bf16" else torch.float32
    _log("build arm")
    arm = Arm(dtype)
    _log("measure")
    clocks = ClockSampler(local)
    r = arm.measure(args.steps, args.warmup, clocks)
    ms_step, ph = r["ms_step"], r["ph"]
    value = N * B * args.steps / (r["total_ms"] / 1000.0)

    # e2e through the public API with host (pinned) inputs
    e2e = None
    _log("e2e")
    if not args.no_e2e:
        hosts = [(bt[rank].lengths.cpu().pin_memory(), bt[rank].values.cpu().pin_memory(), bt[rank].nnz_per_feature)
                 for bt in arm.batches]
        e_ms = arm.timed_graph(args.steps, host_inputs=hosts) if r["graph_ok"] else arm.timed_eager_h2d(hosts, args.steps)
        h2d = hosts[0][0].numel() * 4 + hosts[0][1].numel() * 4
        e2e = {"value": N * B * args.steps / (e_ms / 1000.0), "unit": UNIT, "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": 4}

    traffic = _traffic(args, N)

    def rooflines(a, res):
        """Lookup (HBM) and DCN GEMM (tensor) rooflines + the iteration roofline."""
        ph_ = res["ph"]
        look_bytes, nnz, bags = a.lookup_bytes()
        n_look = max(1, a.eager_timers.count("lookup_fwd") // args.steps)
        look_ms = ph_.get("lookup_fwd", 0.0) / n_look
        look_gbs = look_bytes / (look_ms * 1e-3) / 1e9 if look_ms else 0.0
        tl = traffic.get("pooled_fwd", {}) if a.dtype == dtype else {}
        roof_lookup = {"bound": "hbm", "achieved": look_gbs, "peak": hbm, "unit": "GB/s", "frac": look_gbs / hbm,
                       "traffic": tl.get("dram_bytes_per_launch"), "traffic_source": tl.get("source"),
                       "kernel": "dmt::pooled_fwd_kernel", "algorithmic_bytes": look_bytes, "launch_ms": look_ms,
                       "peak_source": peak_src}
        U = a.unique_rows()
        bwd_bytes = a.bwd_bytes(nnz, bags, U)
        bwd_ms = ph_.get("lookup_bwd", 0.0)
        roof_bwd = {"bound": "hbm", "achieved": bwd_bytes / (bwd_ms * 1e-3) / 1e9 if bwd_ms else 0.0, "peak": hbm,
                    "unit": "GB/s", "algorithmic_bytes": bwd_bytes, "unique_rows": U, "ms": bwd_ms,
                    "kernel": "embedding backward apply (fused SGD); prepare/sort overlapped on a side stream",
                    "bytes_formula": "bags*N*s (grad rows) + nnz*4 (indices) + 2*U*N*s (row read+write)"}
        roof_bwd["frac"] = roof_bwd["achieved"] / hbm
        fl = a.tm_flops()
        tm_ms = ph_.get("tm_fwd", 0.0) + ph_.get("tm_bwd", 0.0) + ph_.get("top_fwd", 0.0) + ph_.get("top_bwd", 0.0)
        roof = roof_lookup
        if fl and tm_ms > look_ms:
            ach = fl / (tm_ms * 1e-3) / 1e12
            tg = traffic.get("gemm_dcn_step", {}) if a.dtype == dtype else {}
            nl = tg.get("launches")
            roof = {"bound": "tensor", "achieved": ach, "peak": tf_burst, "unit": "TFLOP/s", "frac": ach / tf_burst,
                    "frac_of_sustained": ach / tf_sust if tf_sust else None, "peak_sustained": tf_sust,
                    "traffic": tg.get("dram_bytes_per_launch"), "traffic_source": tg.get("source"),
                    "kernel": "dmt::gemm::gemm_kernel (the DCN fwd+bwd GEMMs of one step)",
                    "launches_per_step": nl, "algorithmic_flops": fl,
                    "algorithmic_flops_per_launch": fl / nl if nl else None, "ms": tm_ms,
                    "ms_note": "tm_fwd + tm_bwd phases (CUDA events): GEMMs plus the small column-sum / copy "
                               "kernels between them, so achieved is a lower bound",
                    "peak_source": peak_src + " bf16 dense, burst (the timed region is short and ran at "
                                              "1.8-1.97 GHz; frac_of_sustained divides by the 4 s sustained figure)"}
        ex_bytes, ex_parts = a.exchange_bytes()
        hbm_ms = (look_bytes + bwd_bytes) / (hbm * 1e9) * 1e3
        tensor_ms = fl / (tf_burst * 1e12) * 1e3
        it = {"hbm_bytes": look_bytes + bwd_bytes, "hbm_ms": hbm_ms, "exchange_bytes": ex_bytes,
              "exchange_parts": ex_parts, "tensor_flops": fl, "tensor_ms": tensor_ms}
        return roof, roof_lookup, roof_bwd, it

    _log("rooflines")
    roof, roof_lookup, roof_bwd, iteration = rooflines(arm, r)
    result = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": N, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": args.dtype, "data": "synthetic (uniform random rows, random-init tables and TM weights)",
        "config": _config(args, N), "roofline": roof, "roofline_lookup": roof_lookup, "roofline_lookup_bwd": roof_bwd,
        "lookup_hbm_gbs": roof_lookup["achieved"], "phases_ms_per_step": ph, "phases_source": r["ph_source"],
        "cuda_graph": r["graph_ok"], "eager_ms_per_step": r["eager_ms_step"],
        "exposed_comm_ms_per_step": ph.get("exchange", 0.0), "clocks": r["clocks"], "e2e": e2e,
        "gpu_launches": r["calls"] * args.steps,
        "gpu_launches_note": "libdmt entry-point calls per step x steps (each >= 1 kernel; replayed from a CUDA graph)",
    }
    if not r["graph_ok"]:
        result["cuda_graph_error"] = r["graph_err"]

    # ---- bucketing (step a) kernel: HBM GB/s on this batch ---------------------
    _log("bucketing")
    result["bucketing"] = bucketing_gbs(torch, K, arm, rank, hbm)

    # ---- NVLink bus bandwidth (NCCL all-to-all) for the exchange roofline ------
    busbw = nvlink_busbw(torch, dist, dev, N) if N > 1 else None
    iteration["nvlink_busbw_gbs"] = busbw
    iteration["nvlink_ms"] = iteration["exchange_bytes"] / (busbw * 1e9) * 1e3 if busbw else 0.0
    iteration["bound_ms"] = max(iteration["hbm_ms"], iteration["nvlink_ms"])
    iteration["frac"] = iteration["bound_ms"] / ms_step
    iteration["bound_with_tm_ms"] = max(iteration["hbm_ms"] + iteration["tensor_ms"], iteration["nvlink_ms"])
    iteration["frac_with_tm"] = iteration["bound_with_tm_ms"] / ms_step
    iteration["note"] = ("north-star roofline = max(lookup fwd+bwd HBM bytes / HBM, exchange bytes / NVLink busbw); "
                         "bound_with_tm adds the DCN GEMMs at the burst tensor peak to the HBM leg (they are "
                         "serially dependent), the exchange can overlap")
    result["iteration_roofline"] = iteration

    # ---- flat all-to-all baseline alongside (N > 1) ----------------------------
    if N > 1 and not args.no_flat:
        del arm
        torch.cuda.empty_cache()
        flat = Arm(dtype, mode="flat")
        fr = flat.measure(args.steps, args.warmup)
        fex, fparts = flat.exchange_bytes()
        result["flat_baseline"] = {"value": N * B * args.steps / (fr["total_ms"] / 1000.0),
                                   "ms_per_step": fr["ms_step"], "exposed_comm_ms_per_step": fr["ph"].get("exchange", 0.0),
                                   "phases_ms_per_step": fr["ph"], "exchange_bytes": fex, "exchange_parts": fparts,
                                   "fabric": "nvlink peer stores + barrier" if args.fabric == "peer" else "nccl all-to-all"}
        del flat
    else:
        del arm
    torch.cuda.empty_cache()

    # ---- N = 1: the fp32 C2 record (the dtype with bit-exact lookup parity) ----
    if N == 1 and not args.no_fp32 and dtype != torch.float32 and args.pool_dist == "fixed":
        _log("fp32 arm")
        a32 = Arm(torch.float32)
        r32 = a32.measure(args.steps, args.warmup)
        rf, rl, rb, it32 = rooflines(a32, r32)
        result["fp32"] = {"value": N * B * args.steps / (r32["total_ms"] / 1000.0), "ms_per_step": r32["ms_step"],
                          "cuda_graph": r32["graph_ok"], "phases_ms_per_step": r32["ph"],
                          "roofline_lookup": {k: rl[k] for k in ("achieved", "peak", "frac", "unit", "launch_ms")},
                          "roofline_lookup_bwd": {k: rb[k] for k in ("achieved", "frac", "unit", "ms")},
                          "tm_tflops": rf["achieved"] if rf.get("bound") == "tensor" else None,
                          "tm_note": "fp32 TM = 3xTF32 on tcgen05 (kind::tf32, 3 MMAs per product) with chunked "
                                     "accumulation; no fp32 tensor peak to divide by",
                          "lookup_target_gbs_baseline_md": 4580}
        del a32
        torch.cuda.empty_cache()

    # ---- N = 1: C1 through the reference-compatible API on this GPU -----------
    if N == 1 and not args.no_c1:
        _log("c1")
        try:
            result["c1_api"] = dict(c1_time(P), impl="paper_2403_00877_b200 (loopback: 8 simulated ranks on "
                                                     "this GPU), host numpy in / out per call",
                                   workload="C1 (BASELINE configs[0]), the same harness as the reference arm's "
                                            "reference_c1")
        except Exception as ex:
            result["c1_api"] = {"error": repr(ex)[:200]}

    if rank == 0 and N == 1 and not args.no_cpu:
        _log("cpu baseline")
        result["cpu_baseline"] = cpu_baseline(args)
    if rank == 0:
        print(json.dumps(result), flush=True)
    if world > 1:
        dist.destroy_process_group()


def bucketing_gbs(torch, K, arm, rank, hbm) -> dict:
    """dmt_kjt_bucketize (step a) on this rank's batch: read lengths + offsets +
    values, write the bucketed lengths + values; 20 launches, CUDA events."""
    p = arm.model.plan
    kj = arm.batches[0][rank]
    if not p.a_slots:
        return {}
    dev = kj.values.device
    offs = K.lengths_to_offsets(kj.lengths)
    slot_offs = p.a_slot_value_offsets(kj.nnz_per_feature)
    so = K.device_ints(slot_offs, torch.int64, dev)
    sf = arm.model.engine.slot_feature
    out_len = torch.empty(len(p.a_slots) * p.B, dtype=torch.int32, device=dev)
    out_val = torch.empty(max(1, slot_offs[-1]), dtype=torch.int32, device=dev)
    for _ in range(3):
        K.kjt_bucketize(kj.lengths, offs, kj.values, p.B, sf, so, out_len, out_val)
    n = 20
    s_, e_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s_.record()
    for _ in range(n):
        K.kjt_bucketize(kj.lengths, offs, kj.values, p.B, sf, so, out_len, out_val)
    e_.record()
    torch.cuda.synchronize()
    ms = s_.elapsed_time(e_) / n
    nbytes = kj.lengths.numel() * 4 + offs.numel() * 8 + kj.values.numel() * 4 + out_len.numel() * 4 + \
        int(slot_offs[-1]) * 4
    gbs = nbytes / (ms * 1e-3) / 1e9
    return {"kernel": "dmt::kjt bucketize (step a)", "launch_ms": ms, "algorithmic_bytes": nbytes, "achieved": gbs,
            "unit": "GB/s", "peak": hbm, "frac": gbs / hbm,
            "note": "inputs L2-resident after the first launch (the KJT is 17 MB), so frac can exceed the HBM line; "
                    "timed standalone: at one rank whose slots are the features in order the training step skips "
                    "it (the input KJT is already the bucketized KJT)"}


def nvlink_busbw(torch, dist, dev, N) -> float:
    """NCCL all-to-all bus bandwidth (GB/s, nccl-tests convention: algbw x
    (N-1)/N) with 256 MiB per rank, device-timed, max over ranks."""
    nbytes = 256 << 20
    x = torch.empty(nbytes // 2, dtype=torch.bfloat16, device=dev)
    y = torch.empty_like(x)
    for _ in range(3):
        dist.all_to_all_single(y, x)
    torch.cuda.synchronize()
    dist.barrier()
    s_, e_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s_.record()
    for _ in range(10):
        dist.all_to_all_single(y, x)
    e_.record()
    torch.cuda.synchronize()
    t = torch.tensor([s_.elapsed_time(e_) / 10], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    algbw = nbytes / (float(t.item()) * 1e-3) / 1e9
    return algbw * (N - 1) / N


if __name__ == "__main__":
    main()
