"""GPU parity of the individual libdmt kernels against the CPU oracle / golden
fixtures (bit-exact for integer and routing work, toleranced for float GEMMs)."""

from __future__ import annotations

import numpy as np
import pytest
import torch

from conftest import golden_meta, golden_npz

pytestmark = pytest.mark.gpu

from oracle import bf16_round, pool, route_step_a  # noqa: E402


def dev():
    return torch.device("cuda")


def test_lengths_to_offsets_matches_cumsum():
    from paper_2403_00877_b200 import kernels as K

    rng = np.random.default_rng(0)
    for n in (0, 1, 7, 1023, 8192, 8193, 212_992, 1_000_003):
        lens = rng.integers(0, 40, size=n).astype(np.int32)
        got = K.lengths_to_offsets(torch.from_numpy(lens).to(dev())).cpu().numpy()
        want = np.concatenate([[0], np.cumsum(lens, dtype=np.int64)])
        assert np.array_equal(got, want), n


def test_bucketize_matches_golden_step_a():
    from paper_2403_00877_b200 import kernels as K

    m = golden_meta()["worked_2x4"]
    arr = golden_npz("worked_2x4")
    shards = [(a, b, c, tuple(d), tuple(e)) for a, b, c, d, e in m["placement"]]
    G, F, B = arr["lengths"].shape
    routed = route_step_a(arr["lengths"], arr["values"], list(range(F)), shards, G)
    offs_all = np.concatenate([[0], np.cumsum(arr["lengths"].reshape(-1))])
    slots = [(o, sid) for o in range(G) for sid, s in enumerate(shards) if s[1] == o]
    slot_feature = [shards[sid][0] for _, sid in slots]
    for src in range(G):
        lens = arr["lengths"][src].reshape(-1).astype(np.int32)
        vals = arr["values"][offs_all[src * F * B]:offs_all[(src + 1) * F * B]].astype(np.int32)
        nnz = [int(lens[f * B:(f + 1) * B].sum()) for f in range(F)]
        slot_off = np.concatenate([[0], np.cumsum([nnz[f] for f in slot_feature])]).astype(np.int64)
        L = torch.from_numpy(lens).to(dev())
        O = K.lengths_to_offsets(L)
        V = torch.from_numpy(vals).to(dev())
        out_len = torch.empty(len(slots) * B, dtype=torch.int32, device=dev())
        out_val = torch.empty(max(1, int(slot_off[-1])), dtype=torch.int32, device=dev())
        K.kjt_bucketize(L, O, V, B, torch.tensor(slot_feature, dtype=torch.int32, device=dev()),
                        torch.from_numpy(slot_off).to(dev()), out_len, out_val)
        ol, ov = out_len.cpu().numpy(), out_val.cpu().numpy()
        for s, (owner, sid) in enumerate(slots):
            bundle = {x[0]: x for x in routed[(src, owner)]}
            _, want_len, want_idx = bundle[sid]
            assert np.array_equal(ol[s * B:(s + 1) * B], want_len)
            assert np.array_equal(ov[slot_off[s]:slot_off[s + 1]], want_idx)


def _lookup_gpu(table, lens, idx, mode, out_dtype=None, row_begin=0, row_filter=False):
    from paper_2403_00877_b200 import _lib as L
    from paper_2403_00877_b200 import kernels as K

    w = table if isinstance(table, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(table)).to(dev())
    n = len(lens)
    out = torch.zeros((n, w.shape[1]), dtype=w.dtype, device=dev())
    L_ = torch.from_numpy(np.asarray(lens, dtype=np.int32)).to(dev())
    offs = K.lengths_to_offsets(L_)
    I = torch.from_numpy(np.asarray(idx, dtype=np.int32)).to(dev())
    seg = K.Segment(weights=w, out=out, out_offset=0, out_ld=w.shape[1], bag_begin=0, nbags=n,
                    pooling=L.POOL_CODE[mode], row_begin=row_begin, row_filter=row_filter)
    err = torch.zeros(1, dtype=torch.int32, device=dev())
    K.pooled_lookup_fwd(K.SegmentTable([seg], dev()), offs, I, err)
    return out, int(err.item())


def test_lookup_golden_long_bags_bit_exact():
    g = golden_npz("lookup_order")
    lens = np.diff(g["offsets"])
    out, err = _lookup_gpu(g["table"], lens, g["values"], "sum")
    assert err == 0
    assert np.array_equal(out.double().cpu().numpy(), g["out"])


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("width", [1, 3, 8, 16, 64, 128, 200, 256, 512])
@pytest.mark.parametrize("mode", ["sum", "mean", "none"])
def test_lookup_widths_modes_bit_exact(dtype, width, mode):
    rng = np.random.default_rng(width)
    rows = 777
    table = rng.uniform(-1, 1, (rows, width)).astype(dtype)
    n = 300
    lens = np.ones(n, np.int64) if mode == "none" else rng.integers(0, 33, size=n)
    idx = rng.integers(0, rows, size=int(lens.sum()))
    out, err = _lookup_gpu(table, lens, idx, mode)
    assert err == 0
    want = pool(table, lens, idx, mode)
    assert np.array_equal(out.double().cpu().numpy(), want)


@pytest.mark.parametrize("width", [8, 64, 128, 256])
def test_lookup_bf16_matches_fp32_accumulate_then_round(width):
    rng = np.random.default_rng(3)
    rows = 1000
    t32 = bf16_round(rng.uniform(-1, 1, (rows, width)).astype(np.float32))
    lens = rng.integers(0, 40, size=200)
    idx = rng.integers(0, rows, size=int(lens.sum()))
    w = torch.from_numpy(t32).to(dev()).to(torch.bfloat16)
    out, err = _lookup_gpu(w, lens, idx, "sum")
    want = bf16_round(pool(t32, lens, idx, "sum").astype(np.float32))
    assert np.array_equal(out.float().cpu().numpy(), want)


def test_lookup_row_filter_and_errors():
    rng = np.random.default_rng(5)
    table = rng.uniform(-1, 1, (100, 16)).astype(np.float32)
    lens = rng.integers(0, 10, size=50)
    idx = rng.integers(0, 100, size=int(lens.sum()))
    shard = torch.from_numpy(table[40:70]).to(dev())
    out, err = _lookup_gpu(shard, lens, idx, "sum", row_begin=40, row_filter=True)
    assert err == 0
    keep = (idx >= 40) & (idx < 70)
    bag = np.repeat(np.arange(50), lens)
    nl = np.bincount(bag[keep], minlength=50)
    want = pool(table[40:70], nl, idx[keep] - 40, "sum")
    assert np.array_equal(out.double().cpu().numpy(), want)
    # out-of-range index on a non-filtered shard / bad bag length flag errors
    _, err = _lookup_gpu(table, [2], [0, 100], "sum")
    assert err & 1
    _, err = _lookup_gpu(table, [2], [0, 1], "none")
    assert err & 2


@pytest.mark.parametrize("m,n,k", [(128, 64, 64), (300, 100, 72), (1000, 256, 128), (4096, 512, 1024),
                                   (7, 5, 8), (129, 257, 200)])
@pytest.mark.parametrize("dt", [torch.bfloat16, torch.float32])
def test_gemm_bias_vs_torch(m, n, k, dt):
    from paper_2403_00877_b200 import _lib as L
    from paper_2403_00877_b200 import kernels as K

    g = torch.Generator(device="cuda").manual_seed(m * 7 + n)
    a = torch.randn(m, k, device="cuda", generator=g).to(dt)
    b = torch.randn(n, k, device="cuda", generator=g).to(dt)
    bias = torch.randn(n, device="cuda", generator=g)
    out = torch.empty(m, n, device="cuda", dtype=torch.float32)
    K.gemm(a, b, out, bias=bias, epilogue=L.EPI_BIAS)
    want = a.double() @ b.double().T + bias.double()
    tol = 1e-5 if dt == torch.float32 else 1e-2
    scale = (a.double().abs() @ b.double().abs().T).max().item()
    err = (out.double() - want).abs().max().item()
    assert err <= tol * scale, (err, scale)


@pytest.mark.parametrize("dt", [torch.bfloat16, torch.float32])
def test_gemm_cross_epilogue_vs_torch(dt):
    from paper_2403_00877_b200 import _lib as L
    from paper_2403_00877_b200 import kernels as K

    g = torch.Generator(device="cuda").manual_seed(11)
    m, M = 513, 192
    x0 = torch.randn(m, M, device="cuda", generator=g).to(dt)
    xl = torch.randn(m, M, device="cuda", generator=g).to(dt)
    w = (torch.randn(M, M, device="cuda", generator=g) / M ** 0.5).to(dt)
    b = torch.randn(M, device="cuda", generator=g)
    out = torch.empty(m, M, device="cuda", dtype=dt)
    u = torch.empty(m, M, device="cuda", dtype=dt)
    K.gemm(xl, w, out, bias=b, epilogue=L.EPI_CROSS, x0=x0, xl=xl, aux=u)
    uu = xl.double() @ w.double().T + b.double()
    want = x0.double() * uu + xl.double()
    tol = 1e-5 if dt == torch.float32 else 2e-2
    assert (u.double() - uu).abs().max().item() <= tol * max(1.0, uu.abs().max().item())
    assert (out.double() - want).abs().max().item() <= tol * max(1.0, want.abs().max().item())


def test_gemm_grouped_rows_output():
    """DLRM per-feature projection written straight into the tower output."""
    from paper_2403_00877_b200 import _lib as L
    from paper_2403_00877_b200 import kernels as K

    g = torch.Generator(device="cuda").manual_seed(2)
    rows, F, N, cD, pD = 70, 5, 32, 16, 8
    O = pD + F * cD
    x = torch.randn(rows, F * N, device="cuda", generator=g)
    w = torch.randn(cD, N, device="cuda", generator=g)
    bias = torch.randn(cD, device="cuda", generator=g)
    y = torch.zeros(rows, O, device="cuda")
    K.gemm(x.view(rows * F, N), w, y.view(-1)[pD:], bias=bias, epilogue=L.EPI_BIAS, rows_per_group=F,
           ld_group=O, ld_d=cD)
    want = (x.double().view(rows, F, N) @ w.double().T + bias.double()).reshape(rows, F * cD)
    assert torch.allclose(y[:, pD:].double(), want, rtol=1e-5, atol=1e-5)
    assert (y[:, :pD] == 0).all()


@pytest.mark.parametrize("ta,tb", [(True, False), (False, True), (True, True)])
@pytest.mark.parametrize("dt", [torch.bfloat16, torch.float32])
@pytest.mark.parametrize("m,n,k", [(128, 128, 64), (300, 200, 136), (3328 // 4, 512, 1024), (70, 90, 8)])
def test_gemm_mn_major_operands(ta, tb, dt, m, n, k):
    """A / B read MN-major straight from (k, m) / (k, n) storage -- no transpose."""
    from paper_2403_00877_b200 import kernels as K

    g = torch.Generator(device="cuda").manual_seed(m + n + k)
    A = torch.randn(m, k, device="cuda", generator=g).to(dt)
    Bm = torch.randn(n, k, device="cuda", generator=g).to(dt)
    a = A.t().contiguous() if ta else A
    b = Bm.t().contiguous() if tb else Bm
    out = torch.empty(m, n, device="cuda", dtype=torch.float32)
    K.gemm(a, b, out, trans_a=ta, trans_b=tb)
    want = A.double() @ Bm.double().T
    tol = 1e-5 if dt == torch.float32 else 1e-2
    scale = (A.double().abs() @ Bm.double().abs().T).max().item()
    assert (out.double() - want).abs().max().item() <= tol * scale


@pytest.mark.parametrize("epi", ["cross", "dcn_bwd", "dcn_final", "sgd", "plain_mn"])
@pytest.mark.parametrize("m,n,k,bn", [(8192, 3328, 3328, 0), (16384, 1664, 1664, 0), (300, 512, 200, 4),
                                      (4096, 2560, 192, 3), (1000, 200, 72, 4)])
def test_gemm_cta_pair_matches_single_cta(epi, m, n, k, bn):
    """cta_group::2 pairs (one 256 x BN MMA stream per CTA pair, each CTA
    staging half of B) are bit-identical to the single-CTA kernel: same
    per-element K order.  Covers the C2 shapes, an odd 128-row tile count
    (the peer CTA's rows past m), BN 192 / 256, K-major and MN-major operands
    and the CROSS / DCN_BWD / DCN_FINAL / fused-SGD epilogues."""
    from paper_2403_00877_b200 import _lib as L
    from paper_2403_00877_b200 import kernels as K

    dt = torch.bfloat16
    g = torch.Generator(device="cuda").manual_seed(m + n + k)
    A = torch.randn(m, k, device="cuda", generator=g).to(dt)
    Bm = (torch.randn(n, k, device="cuda", generator=g) / k ** 0.5).to(dt)
    x0 = torch.randn(m, n, device="cuda", generator=g).to(dt)
    u = torch.randn(m, n, device="cuda", generator=g).to(dt)
    bias = torch.randn(n, device="cuda", generator=g)
    flags0 = bn << L.GEMM_BN_SHIFT
    outs = []
    for fl in (flags0 | L.GEMM_SINGLE_CTA, flags0 | L.GEMM_CLUSTER):
        if epi == "cross":
            o = torch.empty(m, n, device="cuda", dtype=dt)
            aux = torch.empty(m, n, device="cuda", dtype=dt)
            K.gemm(A, Bm, o, bias=bias, epilogue=L.EPI_CROSS, x0=x0, xl=u, aux=aux, tune_flags=fl)
            outs.append((o, aux))
        elif epi == "dcn_bwd":  # dX-side: B read MN-major
            Bt = Bm.t().contiguous()
            o = x0.clone()
            gu = torch.empty(m, n, device="cuda", dtype=dt)
            dx0 = torch.ones(m, n, device="cuda", dtype=torch.float32)
            K.gemm(A, Bt, o, trans_b=True, epilogue=L.EPI_DCN_BWD, c=o, beta=1.0, x0=x0, xl=u, aux=gu, aux2=dx0,
                   aux2_accum=True, tune_flags=fl)
            outs.append((o, gu, dx0))
        elif epi == "dcn_final":
            Bt = Bm.t().contiguous()
            o = torch.empty(m, n, device="cuda", dtype=dt)
            dx0 = torch.randn(m, n, device="cuda", generator=torch.Generator(device="cuda").manual_seed(1))
            K.gemm(A, Bt, o, trans_b=True, epilogue=L.EPI_DCN_FINAL, c=x0, beta=1.0, aux2=dx0, tune_flags=fl)
            outs.append((o,))
        elif epi == "sgd":  # W -= lr * A^T B (MN-major A and B, K = m)
            At = A[: min(m, 4096)]
            Bk = x0[: min(m, 4096)]
            W = torch.ones(k, n, device="cuda", dtype=dt)
            K.gemm(At, Bk, W, trans_a=True, trans_b=True, epilogue=L.EPI_ACC, beta=1.0, alpha=-1e-3, tune_flags=fl)
            outs.append((W,))
        else:  # plain, fp32 out, MN-major A
            At = A.t().contiguous()
            o = torch.empty(m, n, device="cuda", dtype=torch.float32)
            K.gemm(At, Bm, o, trans_a=True, tune_flags=fl)
            outs.append((o,))
    torch.cuda.synchronize()
    for a, b in zip(*outs):
        assert torch.equal(a, b)


@pytest.mark.parametrize("rows,cols", [(8192, 3328), (1000, 256), (77, 64), (3, 8), (4096, 100)])
@pytest.mark.parametrize("dt", [torch.bfloat16, torch.float32])
def test_column_sum_vs_fp64(rows, cols, dt):
    """Bias-gradient column sums (DCN backward): fp32 partials folded into
    fp64 every 32 rows, fixed-order final reduction -- deterministic."""
    from paper_2403_00877_b200 import kernels as K

    g = torch.Generator(device="cuda").manual_seed(rows + cols)
    x = torch.randn(rows, cols, device="cuda", generator=g).to(dt)
    got = K.column_sum(x)
    again = K.column_sum(x)
    want = x.double().sum(0)
    torch.cuda.synchronize()
    assert torch.equal(got, again)
    assert (got.double() - want).abs().max().item() <= 1e-5 * (x.double().abs().sum(0).max().item() + 1)


@pytest.mark.parametrize("rows,cols,nl", [(8192, 3328, 3), (1000, 256, 2), (77, 64, 1), (130, 1664, 4)])
@pytest.mark.parametrize("dt", [torch.bfloat16, torch.float16])
def test_dcn_side_fused_matches_separate_kernels(rows, cols, nl, dt):
    """The fused crossnet-backward tail (dx0 = sum_{l=L-1..0} g_l u_l and the
    bias column sums of gu_l, one pass) is bit-identical to the per-layer
    dmt_dcn_dx0_term sequence plus dmt_column_sum (the DMT_DCN_SIDE=split form)
    and within fp32 rounding of a float64 reference."""
    from paper_2403_00877_b200 import kernels as K

    g = torch.Generator(device="cuda").manual_seed(rows * 7 + nl)
    mk = lambda: torch.randn(rows, cols, device="cuda", generator=g).to(dt)  # noqa: E731
    gs, us, gus = [mk() for _ in range(nl)], [mk() for _ in range(nl)], [mk() for _ in range(nl)]
    dx0 = torch.full((rows, cols), float("nan"), device="cuda")
    sums = [torch.full((cols,), float("nan"), device="cuda") for _ in range(nl)]
    K.dcn_side_fused(gs, us, gus, dx0, sums)
    want = torch.empty(rows, cols, device="cuda")
    for l in range(nl - 1, -1, -1):
        K.dcn_dx0_term(gs[l], us[l], want, accumulate=l != nl - 1)
    torch.cuda.synchronize()
    assert torch.equal(dx0, want)
    for l in range(nl):
        assert torch.equal(sums[l], K.column_sum(gus[l]))
    ref = sum(gs[l].double() * us[l].double() for l in range(nl))
    assert (dx0.double() - ref).abs().max().item() <= 1e-6 * (ref.abs().max().item() + 1)
    only = torch.full((rows, cols), float("nan"), device="cuda")
    K.dcn_side_fused(gs, us, None, only, None)  # dx0 only (DMT_DCN_TAIL=main)
    torch.cuda.synchronize()
    assert torch.equal(only, want)


@pytest.mark.parametrize("dt", [torch.float32, torch.bfloat16])
@pytest.mark.parametrize("nsrc,n", [(1, 5), (2, 1664 * 1664 + 3), (3, 4096), (4, 832)])
def test_peer_sum_sgd_matches_rank_order_sum(dt, nsrc, n):
    """dmt_peer_sum_sgd (tower all-reduce + SGD over peer memory) == the
    loopback engine's rank-order fp32 sum followed by dmt_sgd_dense, bit for
    bit (local buffers stand in for the IPC-mapped peers)."""
    from paper_2403_00877_b200 import kernels as K
    from paper_2403_00877_b200.errors import DomainError

    gen = torch.Generator(device="cpu").manual_seed(n + nsrc)
    w0 = torch.randn(n, generator=gen).to(dev(), dt)
    gs = [torch.randn(n, generator=gen).to(dev()) for _ in range(nsrc)]
    want = w0.clone()
    acc = gs[0].clone()
    for g in gs[1:]:
        acc.add_(g)
    K.sgd_dense(want, acc, 0.05)
    got = w0.clone()
    K.peer_sum_sgd(got, gs, 0.05)
    assert torch.equal(got, want)
    with pytest.raises(DomainError):
        K.peer_sum_sgd(got, [g.to(torch.bfloat16) for g in gs], 0.05)


@pytest.mark.parametrize("dt", [torch.bfloat16, torch.float32])
@pytest.mark.parametrize("m,n,k", [(64, 128, 212_992), (256, 512, 8192), (1, 256, 8192), (416, 512, 8192),
                                   (128, 64, 30_000)])
def test_gemm_splitk_weight_grads(dt, m, n, k):
    """Split-K (few output tiles, long K: the DLRM tower-module dW_feat over
    T*B*F rows, MLP dW over the batch): A^T B from MN-major operands vs
    float64, deterministic (fixed split order), and the fused-SGD ACC form."""
    from paper_2403_00877_b200 import _lib as L
    from paper_2403_00877_b200 import kernels as K

    assert K.splitk_factor(m, n, k, 2 if dt == torch.bfloat16 else 4) > 1
    g = torch.Generator(device="cuda").manual_seed(m + n)
    a = (torch.randn(k, m, device="cuda", generator=g) * 0.1).to(dt)  # stored (k, m): A = a^T
    b = (torch.randn(k, n, device="cuda", generator=g) * 0.1).to(dt)
    out = torch.empty(m, n, device="cuda", dtype=torch.float32)
    K.gemm(a, b, out, trans_a=True, trans_b=True)
    again = torch.empty_like(out)
    K.gemm(a, b, again, trans_a=True, trans_b=True)
    want = a.double().T @ b.double()
    tol = 1e-5 if dt == torch.float32 else 1e-2
    mag = a.double().abs().T @ b.double().abs()
    torch.cuda.synchronize()
    assert ((out.double() - want).abs() <= tol * mag).all()
    assert torch.equal(out, again)
    w = torch.ones(m, n, device="cuda", dtype=dt)
    K.gemm(a, b, w, trans_a=True, trans_b=True, epilogue=L.EPI_ACC, beta=1.0, alpha=-1e-3)
    ww = 1.0 - 1e-3 * want
    ulp = 2.0 ** -8 if dt == torch.bfloat16 else 2.0 ** -23
    assert ((w.double() - ww).abs() <= ulp + tol * 1e-3 * mag).all()


@pytest.mark.parametrize("pair", [False, True])
def test_gemm_scattered_row_and_column_groups(pair):
    """Output scatter used to fuse the exchanges into the tower-module GEMMs:
    row blocks to separate buffers (step f from the projection) and column
    blocks to separate buffers with their own row strides (d^-1 from the
    final dX GEMM) -- bit-identical to the plain GEMM's output blocks."""
    from paper_2403_00877_b200 import _lib as L
    from paper_2403_00877_b200 import kernels as K

    dt = torch.bfloat16
    g = torch.Generator(device="cuda").manual_seed(9)
    m, n, k, rpg = 1024, 512, 256, 256
    a = torch.randn(m, k, device="cuda", generator=g).to(dt)
    b = (torch.randn(n, k, device="cuda", generator=g) / 16).to(dt)
    bias = torch.randn(n, device="cuda", generator=g)
    fl = L.GEMM_CLUSTER if pair else L.GEMM_SINGLE_CTA
    want = torch.empty(m, n, device="cuda", dtype=dt)
    K.gemm(a, b, want, bias=bias, epilogue=L.EPI_BIAS, tune_flags=fl)
    rows = [torch.zeros(rpg + 3, n, device="cuda", dtype=dt) for _ in range(m // rpg)]
    K.gemm(a, b, want, bias=bias, epilogue=L.EPI_BIAS, tune_flags=fl, rows_per_group=rpg, ld_d=n,
           out_groups=[t.data_ptr() + 3 * n * 2 for t in rows])
    cols = [torch.zeros(m, 128 + 64 * j, device="cuda", dtype=dt) for j in range(n // 128)]
    x0 = torch.randn(m, n, device="cuda", generator=g).to(dt)
    d0 = torch.randn(m, n, device="cuda", generator=g)
    want2 = torch.empty(m, n, device="cuda", dtype=dt)
    K.gemm(a, b, want2, epilogue=L.EPI_DCN_FINAL, c=x0, beta=1.0, aux2=d0, tune_flags=fl)
    K.gemm(a, b, want2.clone(), epilogue=L.EPI_DCN_FINAL, c=x0, beta=1.0, aux2=d0, tune_flags=fl,
           col_groups=[(t.data_ptr(), t.stride(0)) for t in cols], col_group_width=128)
    torch.cuda.synchronize()
    for j, t in enumerate(rows):
        assert torch.equal(t[3:], want[j * rpg:(j + 1) * rpg])
    for j, t in enumerate(cols):
        assert torch.equal(t[:, :128], want2[:, j * 128:(j + 1) * 128])
