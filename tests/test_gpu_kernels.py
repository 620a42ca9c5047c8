"""Kernel-level parity on the B200: each sm_100a kernel against a plain torch
fp32 computation over the SAME bf16 operands (so the comparison isolates the
kernel's accumulation / epilogue error from bf16 input rounding)."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def lib():
    from paper_2207_06667_b200 import _lib
    return _lib


def _s():
    return torch.cuda.current_stream().cuda_stream


def _bf(x):
    return x.to(torch.bfloat16)


def _rand(*shape, scale=1.0, seed=0):
    g = torch.Generator(device="cpu").manual_seed(seed)
    return (torch.randn(*shape, generator=g) * scale).cuda()


def _padded(t, rows, cols, dtype=torch.bfloat16):
    out = torch.zeros(rows, cols, dtype=dtype, device=t.device)
    out[:t.shape[0], :t.shape[1]] = t.to(dtype)
    return out


GEMM_SHAPES = [(37, 16, 16), (128, 64, 64), (300, 208, 112), (513, 320, 1000), (1024, 1024, 2048),
               (256, 2304, 512)]
# shapes with >= one wave of 256-row tiles take the CTA-pair kernel
# (capi.cu pick_pair_bn): full tiles, ragged M / N where rank 1's A rows or B
# columns run off the end (partly or wholly), M < 256, and the bn=128 pair tile
PAIR_SHAPES = [(4096, 2048, 3072), (3000, 2000, 1000), (1000, 4100, 520), (200, 20000, 64),
               (300, 19000, 64)]


@pytest.mark.parametrize("M,N,K", GEMM_SHAPES + PAIR_SHAPES)
@pytest.mark.parametrize("act", [0, 1])
def test_linear_fwd(lib, M, N, K, act):
    Kp, Np = (K + 15) // 16 * 16, (N + 15) // 16 * 16
    x = _padded(_rand(M, K, seed=1), M, Kp)
    w = _padded(_rand(N, K, scale=K ** -0.5, seed=2), Np, Kp)
    b = torch.zeros(Np, device="cuda")
    b[:N] = _rand(N, seed=3) * 0.1
    ref = x.float() @ w.float().T + b
    if act == 1:
        y = torch.empty(M, Np, dtype=torch.bfloat16, device="cuda")
        ref = torch.tanh(ref)
    else:
        y = torch.empty(M, Np, dtype=torch.float32, device="cuda")
    lib.call("edl_linear_fwd", x.data_ptr(), Kp, w.data_ptr(), Kp, b.data_ptr(), y.data_ptr(), Np,
             M, Np, Kp, act, _s())
    torch.cuda.synchronize()
    err = (y.float() - ref).abs().max().item()
    tol = 2e-2 if act == 1 else 1e-3 * max(1.0, ref.abs().max().item())
    assert err < tol, (err, tol)


@pytest.mark.parametrize("M,N,K", GEMM_SHAPES)
def test_linear_bwd_data(lib, M, N, K):
    # dX[M,K] = (dY[M,N] @ W[N,K]) * (1 - H^2)
    Kp, Np = (K + 15) // 16 * 16, (N + 15) // 16 * 16
    dy = _padded(_rand(M, N, seed=4), M, Np)
    w = _padded(_rand(N, K, scale=N ** -0.5, seed=5), Np, Kp)
    h = _padded(torch.tanh(_rand(M, K, seed=6)), M, Kp)
    dx = torch.empty(M, Kp, dtype=torch.bfloat16, device="cuda")
    lib.call("edl_linear_bwd_data", dy.data_ptr(), Np, w.data_ptr(), Kp, h.data_ptr(), Kp,
             dx.data_ptr(), Kp, M, Np, Kp, _s())
    torch.cuda.synchronize()
    ref = (dy.float() @ w.float()) * (1 - h.float() ** 2)
    err = (dx.float() - ref).abs().max().item()
    assert err < 2e-2 * max(1.0, ref.abs().max().item()), err


@pytest.mark.parametrize("M,N,K", GEMM_SHAPES)
def test_linear_bwd_weight(lib, M, N, K):
    # dW[N,K] = s * dY[M,N]^T @ X[M,K];  db = s * colsum(dY)
    Kp, Np = (K + 15) // 16 * 16, (N + 15) // 16 * 16
    dy = _padded(_rand(M, N, seed=7), M, Np)
    x = _padded(_rand(M, K, seed=8), M, Kp)
    dw = torch.full((Np, Kp), float("nan"), device="cuda")
    db = torch.full((Np,), float("nan"), device="cuda")
    ws = torch.empty(int(lib.load().edl_colsum_workspace_floats(M, Np)), device="cuda")
    lib.call("edl_linear_bwd_weight", dy.data_ptr(), Np, x.data_ptr(), Kp, dw.data_ptr(), Kp,
             db.data_ptr(), ws.data_ptr(), M, Np, Kp, 0.5, _s())
    torch.cuda.synchronize()
    ref = 0.5 * dy.float().T @ x.float()
    refb = 0.5 * dy.float().sum(0)
    scale = max(1.0, ref.abs().max().item())
    assert (dw - ref).abs().max().item() < 1e-3 * scale
    assert (db - refb).abs().max().item() < 1e-3 * max(1.0, refb.abs().max().item())


@pytest.mark.parametrize("B,H,K,k", [(32, 256, 10, 10), (32, 256, 10, 4), (200, 512, 100, 16),
                                     (256, 1024, 1000, 16), (130, 2048, 1000, 32),
                                     (64, 256, 2000, 8), (4096, 512, 1000, 16), (300, 256, 3000, 16)])
@pytest.mark.parametrize("pair", [False, True])
def test_teacher_head_softmax_topk(lib, B, H, K, k, pair):
    """The fused head (edl/nnkit.py:193-208 + top-k) against fp64 on the same
    bf16 operands: the single-CTA cluster kernel and the CTA-pair kernel with
    the class-chunk merge through global memory (any class count)."""
    T = 2.0
    Hp, Kp = (H + 15) // 16 * 16, (K + 15) // 16 * 16
    if not pair and (Kp + 255) // 256 > 8:
        pytest.skip("the cluster head spans at most 8 x 256 classes")
    h = _padded(torch.tanh(_rand(B, H, seed=9)), B, Hp)
    w = _padded(_rand(K, H, scale=3 * H ** -0.5, seed=10), Kp, Hp)
    b = torch.zeros(Kp, device="cuda")
    b[:K] = _rand(K, seed=11) * 0.1
    vals = torch.empty(B, k, device="cuda")
    idx = torch.empty(B, k, dtype=torch.int32, device="cuda")
    if pair:
        nb = int(lib.load().edl_teacher_head_workspace_bytes(B, K, k))
        ws = torch.zeros(nb, dtype=torch.uint8, device="cuda")
        for _ in range(2):      # the tickets must come back to zero for the next launch
            lib.call("edl_teacher_head_softmax_topk_ws", h.data_ptr(), Hp, w.data_ptr(), Hp, b.data_ptr(), B, K,
                     Hp, T, k, vals.data_ptr(), idx.data_ptr(), ws.data_ptr(), nb, _s())
        torch.cuda.synchronize()
        tick = ws[-((B + 127) // 128 + 1) * 4:].view(torch.int32)
        assert (tick == 0).all()
    else:
        lib.call("edl_teacher_head_softmax_topk", h.data_ptr(), Hp, w.data_ptr(), Hp, b.data_ptr(), B, K,
                 Hp, T, k, vals.data_ptr(), idx.data_ptr(), _s())
    torch.cuda.synchronize()
    z = (h.double() @ w.double().T + b.double())[:, :K]
    p = torch.softmax(z / T, dim=1)
    order = torch.from_numpy(np.argsort(-p.cpu().numpy(), axis=1, kind="stable")[:, :k]).cuda()
    # index parity where the k-th / (k+1)-th gap exceeds fp32 accumulation noise
    sp = torch.sort(z, dim=1, descending=True).values
    gap = (sp[:, k - 1] - sp[:, k]) if k < K else torch.full((B,), 1e9, device="cuda", dtype=sp.dtype)
    safe = gap > 1e-3
    assert safe.float().mean() > 0.5
    assert torch.equal(idx[safe].long(), order[safe])
    pv = torch.gather(p, 1, idx.long())
    assert (vals.double() - pv).abs().max().item() < 1e-5


def test_teacher_head_pair_equals_cluster_head(lib):
    """cfg3's head shape: the pair kernel and the cluster kernel agree (same
    per-chunk states, same chunk-order merge)."""
    B, H, K, k, T = 4096, 8192, 1000, 16, 2.0
    Kp = 1008
    h = _padded(torch.tanh(_rand(B, H, seed=19)), B, H)
    w = _padded(_rand(K, H, scale=3 * H ** -0.5, seed=20), Kp, H)
    b = torch.zeros(Kp, device="cuda")
    outs = []
    for pair in (False, True):
        vals = torch.empty(B, k, device="cuda")
        idx = torch.empty(B, k, dtype=torch.int32, device="cuda")
        if pair:
            nb = int(lib.load().edl_teacher_head_workspace_bytes(B, K, k))
            ws = torch.zeros(nb, dtype=torch.uint8, device="cuda")
            lib.call("edl_teacher_head_softmax_topk_ws", h.data_ptr(), H, w.data_ptr(), H, b.data_ptr(), B, K, H, T, k,
                     vals.data_ptr(), idx.data_ptr(), ws.data_ptr(), nb, _s())
        else:
            lib.call("edl_teacher_head_softmax_topk", h.data_ptr(), H, w.data_ptr(), H, b.data_ptr(), B, K, H, T, k,
                     vals.data_ptr(), idx.data_ptr(), _s())
        torch.cuda.synchronize()
        outs.append((vals, idx))
    (v0, i0), (v1, i1) = outs
    same = (i0 == i1).all(1)
    assert same.float().mean() > 0.99
    assert (v0 - v1).abs().max().item() <= 1e-6 * v0.abs().max().item()


def _run_head_pair(B, H, K, k, seed, out_path=None):
    from paper_2207_06667_b200 import _lib
    Hp, Kp = (H + 15) // 16 * 16, (K + 15) // 16 * 16
    h = _padded(torch.tanh(_rand(B, H, seed=seed)), B, Hp)
    w = _padded(_rand(K, H, scale=3 * H ** -0.5, seed=seed + 1), Kp, Hp)
    b = torch.zeros(Kp, device="cuda")
    b[:K] = _rand(K, seed=seed + 2) * 0.1
    vals = torch.empty(B, k, device="cuda")
    idx = torch.empty(B, k, dtype=torch.int32, device="cuda")
    nb = int(_lib.load().edl_teacher_head_workspace_bytes(B, K, k))
    ws = torch.zeros(nb, dtype=torch.uint8, device="cuda")
    _lib.call("edl_teacher_head_softmax_topk_ws", h.data_ptr(), Hp, w.data_ptr(), Hp, b.data_ptr(), B, K, Hp, 2.0,
              k, vals.data_ptr(), idx.data_ptr(), ws.data_ptr(), nb, _s())
    torch.cuda.synchronize()
    out = (vals.cpu(), idx.cpu())
    if out_path:
        torch.save(out, out_path)
    return out


@pytest.mark.parametrize("B,H,K,k", [(1024, 2048, 1000, 16), (512, 512, 3000, 32), (4096, 1024, 1000, 16),
                                     (900, 256, 100, 8)])
def test_teacher_head_multicast_bitwise(lib, B, H, K, k, tmp_path):
    """With an even number of 256-row blocks the pair head runs in 4-CTA
    clusters sharing each B tile through a 2-SM TMA multicast: bitwise equal
    to the 2-CTA pair head (EDL_HEAD_MC=0 in a subprocess; same MMAs per tile,
    same chunk-order merge)."""
    import os
    import subprocess
    import sys
    got = _run_head_pair(B, H, K, k, seed=B + K)
    ref_path = str(tmp_path / "head.pt")
    code = ("import sys, torch; sys.path.insert(0, '.'); sys.path.insert(0, 'tests');"
            "import test_gpu_kernels as t;"
            f"t._run_head_pair({B}, {H}, {K}, {k}, {B + K}, {ref_path!r})")
    env = dict(os.environ, EDL_HEAD_MC="0")
    subprocess.run([sys.executable, "-c", code], check=True, env=env, timeout=300)
    want = torch.load(ref_path)
    assert torch.equal(got[1], want[1])
    assert torch.equal(got[0], want[0])


@pytest.mark.parametrize("B,K,k,alpha,beta,T", [(32, 10, 10, 0.5, 0.5, 2.0), (32, 10, 4, 1.0, 0.0, 2.0),
                                                (300, 1000, 16, 0.5, 0.5, 2.0), (64, 100, 100, 0.0, 1.0, 3.0),
                                                (4096, 1000, 16, 0.7, 0.3, 0.5)])
def test_kd_loss(lib, B, K, k, alpha, beta, T):
    Kp = (K + 15) // 16 * 16
    z = torch.zeros(B, Kp, device="cuda")
    z[:, :K] = _rand(B, K, scale=3.0, seed=12)
    y = torch.randint(0, K, (B,), generator=torch.Generator().manual_seed(1)).cuda()
    q = torch.rand(B, K, generator=torch.Generator().manual_seed(2)).cuda() + 0.05
    qv, qi = torch.topk(q, k, dim=1)
    qi = qi.int()
    qv = qv.contiguous()
    row = torch.empty(B, device="cuda")
    loss = torch.zeros(1, device="cuda")
    ticket = torch.zeros(1, dtype=torch.int32, device="cuda")
    status = torch.zeros(1, dtype=torch.int32, device="cuda")
    dz = torch.full((B, Kp), 7.0, dtype=torch.bfloat16, device="cuda")
    lib.call("edl_kd_loss_fwd_bwd", z.data_ptr(), Kp, y.data_ptr(), qv.data_ptr(), qi.data_ptr(), B, K, k,
             alpha, beta, T, row.data_ptr(), loss.data_ptr(), ticket.data_ptr(), dz.data_ptr(), Kp,
             status.data_ptr(), _s())
    torch.cuda.synchronize()
    zz = z[:, :K].double()
    qd = torch.zeros(B, K, device="cuda", dtype=torch.float64).scatter_(1, qi.long(), qv.double())
    qd = qd / qd.sum(1, keepdim=True)
    logp = torch.log_softmax(zz, 1)
    logpt = torch.log_softmax(zz / T, 1)
    ref = 0.0
    dref = torch.zeros_like(zz)
    if alpha > 0:
        ref += alpha * (-logp[torch.arange(B), y]).mean()
        dref += alpha / B * (logp.exp() - torch.nn.functional.one_hot(y, K))
    if beta > 0:
        ref += beta * T * T * (-(qd * logpt).sum(1)).mean()
        dref += beta * T / B * (logpt.exp() - qd)
    assert status.item() == 0 and ticket.item() == 0
    assert abs(loss.item() - float(ref)) < 1e-4 * max(1.0, abs(float(ref)))
    assert (dz[:, :K].double() - dref).abs().max().item() < 1e-2 * dref.abs().max().item() + 1e-6
    assert (dz[:, K:] == 0).all()


def _kd_reference(zz, y, qv, qi, alpha, beta, T):
    """loss and dlogits in fp64 (edl/nnkit.py:283-299) on fp64 logits."""
    B, K = zz.shape
    logp = torch.log_softmax(zz, 1)
    logpt = torch.log_softmax(zz / T, 1)
    ref = 0.0
    dref = torch.zeros_like(zz)
    if alpha > 0:
        ref += alpha * (-logp[torch.arange(B), y]).mean()
        dref += alpha / B * (logp.exp() - torch.nn.functional.one_hot(y, K))
    if beta > 0:
        qd = torch.zeros(B, K, device="cuda", dtype=torch.float64).scatter_(1, qi.long(), qv.double())
        qd = qd / qd.sum(1, keepdim=True)
        ref += beta * T * T * (-(qd * logpt).sum(1)).mean()
        dref += beta * T / B * (logpt.exp() - qd)
    return float(ref), dref, logp.exp(), logpt.exp()


# (B, hidden D, classes K, k, alpha, beta, T): one CTA / cluster of 2..8 along
# the classes, ragged B and K, every KMAX instance, T == 2 (one exp per
# element) and T != 2, hard-only and soft-only
KD_HEAD_CASES = [(32, 64, 10, 10, 0.5, 0.5, 2.0), (300, 128, 1000, 16, 0.5, 0.5, 2.0),
                 (4096, 1024, 1000, 16, 0.5, 0.5, 2.0), (129, 64, 300, 8, 1.0, 0.0, 2.0),
                 (200, 192, 513, 32, 0.0, 1.0, 3.0), (64, 80, 2048, 4, 0.7, 0.3, 0.5),
                 (1000, 512, 777, 20, 0.5, 0.5, 1.0)]


@pytest.mark.parametrize("B,D,K,k,alpha,beta,T", KD_HEAD_CASES)
def test_linear_kd_loss_fused(lib, B, D, K, k, alpha, beta, T):
    """edl_linear_kd_loss_fwd_bwd (logit GEMM + KD loss + dlogits in one
    epilogue) against fp64 over the SAME bf16 operands: logits error model
    |dz - ref| <= one bf16 ulp + the softmax's sensitivity to an fp32
    accumulation error of (D / 16) 2^-24 sum|h w| per logit."""
    Dp, Kp = (D + 15) // 16 * 16, (K + 15) // 16 * 16
    h = _padded(torch.tanh(_rand(B, D, seed=3)), B, Dp)
    w = _padded(_rand(K, D, scale=1.0 / D ** 0.5 * 3, seed=4), Kp, Dp)
    bias = torch.zeros(Kp, device="cuda")
    bias[:K] = _rand(K, scale=0.1, seed=5)
    y = torch.randint(0, K, (B,), generator=torch.Generator().manual_seed(6)).cuda()
    q = torch.rand(B, K, generator=torch.Generator().manual_seed(7)).cuda() + 0.01
    qv, qi = torch.topk(q, k, dim=1)
    qv, qi = (qv / q.sum(1, keepdim=True)).contiguous(), qi.int().contiguous()
    row = torch.empty(B, device="cuda")
    loss = torch.zeros(1, device="cuda")
    status = torch.zeros(1, dtype=torch.int32, device="cuda")
    dz = torch.full((B, Kp), 7.0, dtype=torch.bfloat16, device="cuda")
    lib.call("edl_linear_kd_loss_fwd_bwd", h.data_ptr(), Dp, w.data_ptr(), Dp, bias.data_ptr(), y.data_ptr(),
             qv.data_ptr(), qi.data_ptr(), B, K, Dp, k if beta > 0 else 0, alpha, beta, T, row.data_ptr(),
             loss.data_ptr(), dz.data_ptr(), Kp, status.data_ptr(), _s())
    torch.cuda.synchronize()
    assert status.item() == 0
    hd, wd = h.double(), w[:K].double()
    zz = hd @ wd.T + bias[:K].double()
    ref, dref, p1, pT = _kd_reference(zz, y, qv, qi, alpha, beta, T)
    eps = ((Dp + 15) // 16 * 2.0 ** -24) * (hd.abs() @ wd.abs().T).max(1, keepdim=True).values
    assert abs(loss.item() - ref) <= 1e-5 * max(1.0, abs(ref))
    d = dz[:, :K].double()
    a = dref.abs()
    ulp = torch.where(a > 0, torch.exp2(torch.floor(torch.log2(torch.where(a > 0, a, torch.ones_like(a)))) - 7),
                      torch.zeros_like(a))
    bound = ulp + 2 * eps * (alpha / B * p1 + beta * T / B * pT / T) + 2.0 ** -20 * (alpha + beta * T) / B
    assert ((d - dref).abs() / bound).max().item() <= 1.0
    assert (dz[:, K:] == 0).all()
    assert torch.isfinite(row).all()
    # the same numbers as the unfused path (logit GEMM + separate loss kernel)
    z = torch.zeros(B, Kp, device="cuda")
    lib.call("edl_linear_fwd", h.data_ptr(), Dp, w.data_ptr(), Dp, bias.data_ptr(), z.data_ptr(), Kp, B, Kp, Dp, 0, _s())
    row2, loss2 = torch.empty(B, device="cuda"), torch.zeros(1, device="cuda")
    ticket = torch.zeros(1, dtype=torch.int32, device="cuda")
    dz2 = torch.full((B, Kp), 7.0, dtype=torch.bfloat16, device="cuda")
    lib.call("edl_kd_loss_fwd_bwd", z.data_ptr(), Kp, y.data_ptr(), qv.data_ptr(), qi.data_ptr(), B, K,
             k if beta > 0 else 0, alpha, beta, T, row2.data_ptr(), loss2.data_ptr(), ticket.data_ptr(),
             dz2.data_ptr(), Kp, status.data_ptr(), _s())
    torch.cuda.synchronize()
    assert abs(loss.item() - loss2.item()) <= 1e-5 * max(1.0, abs(loss2.item()))
    assert ((dz[:, :K].double() - dz2[:, :K].double()).abs() <= 2 * bound).all()


def test_linear_kd_loss_bad_labels_set_status(lib):
    B, D, K, k = 64, 64, 100, 4
    h = _padded(torch.tanh(_rand(B, D, seed=3)), B, D)
    w = _padded(_rand(K, D, seed=4), 112, D)
    bias = torch.zeros(112, device="cuda")
    y = torch.zeros(B, dtype=torch.int64, device="cuda")
    y[5] = K                                   # out of range
    qv = torch.full((B, k), 0.25, device="cuda")
    qi = torch.arange(k, dtype=torch.int32, device="cuda").repeat(B, 1).contiguous()
    qi[7, 1] = 5000                            # soft class out of range
    row, loss = torch.empty(B, device="cuda"), torch.zeros(1, device="cuda")
    status = torch.zeros(1, dtype=torch.int32, device="cuda")
    dz = torch.zeros(B, 112, dtype=torch.bfloat16, device="cuda")
    lib.call("edl_linear_kd_loss_fwd_bwd", h.data_ptr(), D, w.data_ptr(), D, bias.data_ptr(), y.data_ptr(),
             qv.data_ptr(), qi.data_ptr(), B, K, D, k, 0.5, 0.5, 2.0, row.data_ptr(), loss.data_ptr(),
             dz.data_ptr(), 112, status.data_ptr(), _s())
    torch.cuda.synchronize()
    assert status.item() == -1
    with pytest.raises(Exception):
        lib.call("edl_linear_kd_loss_fwd_bwd", h.data_ptr(), D, w.data_ptr(), D, bias.data_ptr(), y.data_ptr(),
                 qv.data_ptr(), qi.data_ptr(), B, 4000, D, k, 0.5, 0.5, 2.0, row.data_ptr(), loss.data_ptr(),
                 dz.data_ptr(), 4000, status.data_ptr(), _s())     # > 2048 classes: the unfused path's job


def test_sgd_and_cast(lib):
    n = 1003
    p = _rand(n, seed=13)
    g = _rand(n, seed=14)
    pb = torch.empty(n, dtype=torch.bfloat16, device="cuda")
    ref = p - 0.25 * g
    lib.call("edl_sgd_step", p.data_ptr(), pb.data_ptr(), g.data_ptr(), n, 0.25, _s())
    torch.cuda.synchronize()
    assert torch.equal(p, ref)
    assert torch.equal(pb, ref.to(torch.bfloat16))


def test_gather_rows(lib):
    src = _bf(_rand(100, 48, seed=15))
    idx = torch.tensor([5, 99, 0, 5, 42], dtype=torch.int64, device="cuda")
    dst = torch.empty(5, 48, dtype=torch.bfloat16, device="cuda")
    lab = torch.arange(100, dtype=torch.int64, device="cuda") * 3
    dlab = torch.empty(5, dtype=torch.int64, device="cuda")
    lib.call("edl_gather_rows", src.data_ptr(), 48, idx.data_ptr(), dst.data_ptr(), 48, 5, 48, None, None, _s())
    torch.cuda.synchronize()
    assert torch.equal(dst, src[idx])
    dst.zero_()
    lib.call("edl_gather_rows", src.data_ptr(), 48, idx.data_ptr(), dst.data_ptr(), 48, 5, 48, lab.data_ptr(),
             dlab.data_ptr(), _s())
    torch.cuda.synchronize()
    assert torch.equal(dst, src[idx]) and torch.equal(dlab, lab[idx])


def test_topk_hits_tie_rule(lib):
    z = torch.zeros(4, 16, device="cuda")
    y = torch.tensor([0, 1, 3, 2], dtype=torch.int64, device="cuda")
    hits = torch.zeros(1, dtype=torch.int32, device="cuda")
    lib.call("edl_topk_hits", z.data_ptr(), 16, y.data_ptr(), 4, 10, 1, hits.data_ptr(), _s())
    torch.cuda.synchronize()
    assert hits.item() == 1   # constant logits: only class 0 ranks first


@pytest.mark.parametrize("B,shapes", [
    (300, [(208, 112), (64, 208), (16, 64)]),                    # single-CTA tiles
    (4096, [(2048, 3072), (1024, 2048), (1008, 1024)]),          # cfg3 student: CTA-pair tiles
    (4000, [(2000, 3008), (1008, 1984), (528, 1008)]),           # pair tiles, every dim ragged
])
def test_linear_bwd_weight_grouped_matches_reference(lib, B, shapes):
    # three student-like layers of different shapes in one launch
    dys = [_padded(_rand(B, n, seed=20 + i), B, n) for i, (n, k) in enumerate(shapes)]
    xs = [_padded(_rand(B, k, seed=30 + i), B, k) for i, (n, k) in enumerate(shapes)]
    dws = [torch.full((n, k), float("nan"), device="cuda") for n, k in shapes]
    dbs = [torch.full((n,), float("nan"), device="cuda") for n, k in shapes]
    ws = torch.empty(lib.colsum_group_workspace_floats([B] * 3, [n for n, _ in shapes]), device="cuda")
    lib.bwd_weight_grouped(dys, xs, dws, dbs, ws, [B] * 3, [n for n, _ in shapes], [k for _, k in shapes], 1.0,
                           _s())
    torch.cuda.synchronize()
    for dy, x, dw, db in zip(dys, xs, dws, dbs):
        ref = dy.float().T @ x.float()
        assert (dw - ref).abs().max().item() < 1e-3 * max(1.0, ref.abs().max().item())
        assert (db - dy.float().sum(0)).abs().max().item() < 1e-3 * max(1.0, db.abs().max().item())
