"""Halo-tiled 3x3 convolution (csrc/halo.cu): the staged-patch layout and
the row-shifted no-swizzle UMMA operand, then the full convolution against
torch (conv2d on the same bf16 operands, fp32 accumulate)."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _patch(x, n, h0, W):
    """rows h0-1 .. h0+2 of image n, columns -1 .. W, zero outside: [4*(W+2)][64]."""
    N, H, _, C = x.shape
    p = torch.zeros(4, W + 2, C)
    for i in range(4):
        h = h0 - 1 + i
        if 0 <= h < H:
            p[i, 1:W + 1] = x[n, h].float()
    return p.reshape(-1, C)


@pytest.mark.parametrize("h0,off", [(0, 0), (27, 1), (27, 59), (54, 118), (10, 61)])
def test_halo_probe_row_shifted_operand(h0, off):
    from paper_2207_06667_b200 import _lib
    N, H, W, C = 2, 56, 56, 64
    g = torch.Generator().manual_seed(h0 * 7 + off)
    x = torch.randn(N, H, W, C, generator=g).to(torch.bfloat16)
    w = torch.randn(64, 64, generator=g).to(torch.bfloat16)
    xd, wd = x.cuda(), w.cuda()
    p = _patch(x, 1, h0, W)
    p = torch.cat([p, torch.zeros(256, C)])            # rows past the patch: not compared
    want = p[off:off + 128] @ w.float().T
    valid = min(128, 4 * (W + 2) - off)
    res = {}
    for mode in (0, 1, 2):
        out = torch.zeros(128 * 64 + 1, device="cuda")
        _lib.call("edl_halo_probe", xd.data_ptr(), N, H, W, 1, h0, off, wd.data_ptr(), mode, 0, 0, out.data_ptr(),
                  torch.cuda.current_stream().cuda_stream)
        torch.cuda.synchronize()
        res[mode] = (out.cpu()[:128 * 64].view(128, 64)[:valid] - want[:valid]).abs().max().item()
    print("probe", h0, off, res)
    assert res[0] < 1e-2 and res[2] < 1e-2, res     # the base-offset field must stay 0 (mode 1 is wrong)


@pytest.mark.parametrize("off,delta", [(0, 1), (3, 56), (10, 59), (2, 118)])
def test_halo_probe_mn_major_stacked_views(off, delta):
    """Mode 4: an MN-major A operand whose two 64-wide M halves are the patch
    viewed at rows off and off + delta (LBO = delta rows of 128 B), B the
    weight tile read MN-major: the halo weight-gradient layout (two filter
    taps per 128-row UMMA)."""
    from paper_2207_06667_b200 import _lib
    N, H, W = 1, 56, 56
    g = torch.Generator().manual_seed(off * 131 + delta)
    x = torch.randn(N, H, W, 64, generator=g).to(torch.bfloat16)
    w = torch.randn(64, 64, generator=g).to(torch.bfloat16)
    p = torch.cat([_patch(x, 0, 20, W), torch.zeros(256, 64)])
    out = torch.zeros(128 * 64 + 2, device="cuda")
    _lib.call("edl_halo_probe", x.cuda().data_ptr(), N, H, W, 0, 20, off, w.cuda().data_ptr(), 4, delta, 0,
              out.data_ptr(), torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    got = out[:128 * 64].view(128, 64).cpu()
    want = torch.cat([p[off:off + 64].T @ w.float(), p[off + delta:off + delta + 64].T @ w.float()])
    err = (got - want).abs().max().item()
    print("mn-stacked", off, delta, err)
    assert err < 1e-2, err


def test_halo_probe_mma_throughput():
    """Cycles for 9 taps x 4 UMMAs (128 x 64 x 16) x reps from the staged
    patch: the no-swizzle chunk-plane layout vs SWIZZLE_128B rows."""
    from paper_2207_06667_b200 import _lib
    N, H, W = 1, 56, 56
    x = torch.randn(N, H, W, 64, device="cuda").to(torch.bfloat16)
    w = torch.randn(64, 64, device="cuda").to(torch.bfloat16)
    cyc = {}
    for mode in (0, 2):
        out = torch.zeros(128 * 64 + 1, device="cuda")
        _lib.call("edl_halo_probe", x.data_ptr(), N, H, W, 0, 10, 0, w.data_ptr(), mode, 200, 0, out.data_ptr(),
                  torch.cuda.current_stream().cuda_stream)
        torch.cuda.synchronize()
        cyc[mode] = out[128 * 64].item() / (200 * 36)
    out = torch.zeros(128 * 64 + 1, device="cuda")       # reps > 1000: the same on all 148 SMs at once
    _lib.call("edl_halo_probe", x.data_ptr(), N, H, W, 0, 10, 0, w.data_ptr(), 2, 1200, 0, out.data_ptr(),
              torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    cyc["all_sms"] = out[128 * 64].item() / (200 * 36)
    w9 = torch.randn(64, 576, device="cuda").to(torch.bfloat16)   # 9 tap tiles, alternating accumulators
    out = torch.zeros(128 * 64 + 1, device="cuda")
    _lib.call("edl_halo_probe", x.data_ptr(), N, H, W, 0, 10, 0, w9.data_ptr(), 3, 2200, 0, out.data_ptr(),
              torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    cyc["9_taps_2_acc"] = out[128 * 64].item() / (200 * 36)
    for kb in (106, 112, 114, 116, 120, 140, 170, 200):   # dynamic shared memory of the CTA
        out = torch.zeros(128 * 64 + 2, device="cuda")
        _lib.call("edl_halo_probe", x.data_ptr(), N, H, W, 0, 10, 0, w.data_ptr(), 2, 200, kb, out.data_ptr(),
                  torch.cuda.current_stream().cuda_stream)
        torch.cuda.synchronize()
        cyc[f"smem_{kb}KB"] = out[128 * 64].item() / (200 * 36)
    print("cycles per 128x64x16 UMMA:", cyc)

_CASES = [  # N, H, W, residual / add, relu / mask
    (2, 14, 14, True, True),
    (3, 17, 17, False, True),       # R = 6 rows per tile, H % R != 0
    (1, 9, 62, True, False),        # R = 2 with W + 2 = 64 (the widest halo tile)
    (1, 5, 90, True, True),         # W > 62: the im2col GEMM path (dispatch boundary)
    (2, 56, 56, True, True),        # stage-1 shape (R = 2, 116 of 128 tile rows live)
    (5, 7, 30, False, False),
]


def _run_convs(case, seed, out_path=None):
    """Forward (bias, optional residual, ReLU) and data gradient (optional add
    and mask) through the C-ABI; returns the two outputs on the CPU."""
    from paper_2207_06667_b200 import _lib
    N, H, W, extra, flag = case
    g = torch.Generator().manual_seed(seed)
    x = torch.randn(N, H, W, 64, generator=g).to(torch.bfloat16).cuda()
    w = (torch.randn(64, 576, generator=g) * 0.06).to(torch.bfloat16).cuda()
    b = (torch.randn(64, generator=g) * 0.1).cuda()
    r = torch.randn(N, H, W, 64, generator=g).to(torch.bfloat16).cuda()
    m = torch.randn(N, H, W, 64, generator=g).to(torch.bfloat16).cuda()
    s = torch.cuda.current_stream().cuda_stream
    y = torch.empty(N, H, W, 64, dtype=torch.bfloat16, device="cuda")
    act = _lib.EDL_ACT_RELU if (flag or extra) else _lib.EDL_ACT_IDENT
    _lib.call("edl_conv_fwd_nhwc", x.data_ptr(), N, H, W, 64, w.data_ptr(), 576, b.data_ptr(), 64, 3, 3, 1, 1,
              r.data_ptr() if extra else None, 64, y.data_ptr(), 64, act, s)
    wf = torch.empty(64, 576, dtype=torch.bfloat16, device="cuda")
    _lib.call("edl_conv_flip_weights", w.data_ptr(), 576, 64, 64, 3, 3, wf.data_ptr(), 576, s)
    dx = torch.empty_like(y)
    _lib.call("edl_conv_dgrad_nhwc", x.data_ptr(), N, H, W, 64, wf.data_ptr(), 576, 64, 3, 3, 1,
              r.data_ptr() if extra else None, m.data_ptr() if flag else None, dx.data_ptr(), s)
    torch.cuda.synchronize()
    out = (y.cpu(), dx.cpu(), x.cpu(), w.cpu(), b.cpu(), r.cpu(), m.cpu())
    if out_path:
        torch.save(out[:2], out_path)
    return out


@pytest.mark.parametrize("case", _CASES)
def test_halo_conv_bitwise_vs_im2col_gemm_and_torch(case, tmp_path):
    """The halo conv (dispatched by edl_conv_fwd_nhwc / edl_conv_dgrad_nhwc
    for 64 -> 64 3x3 stride-1 layers) is bitwise equal to the TMA-im2col GEMM
    path (EDL_HALO=0 in a subprocess: same tap-major K order, same UMMA
    shapes, same epilogue arithmetic) and within 1e-2 of torch conv2d."""
    import subprocess
    import sys

    import torch.nn.functional as F
    seed = sum(case[:3]) * 13 + int(case[3]) + 2 * int(case[4])
    y, dx, x, w, b, r, m = _run_convs(case, seed)
    ref_path = str(tmp_path / "ref.pt")
    code = ("import sys, torch; sys.path.insert(0, '.'); sys.path.insert(0, 'tests');"
            "import test_gpu_halo as t;"
            f"t._run_convs({case!r}, {seed}, {ref_path!r})")
    env = dict(__import__("os").environ, EDL_HALO="0")
    subprocess.run([sys.executable, "-c", code], check=True, env=env, timeout=300)
    y0, dx0 = torch.load(ref_path)
    assert torch.equal(y, y0)
    assert torch.equal(dx, dx0)
    N, H, W, extra, flag = case
    xt = x.float().permute(0, 3, 1, 2)
    wt = w.float().reshape(64, 3, 3, 64).permute(0, 3, 1, 2)
    want = F.conv2d(xt, wt, b, padding=1) + (r.float().permute(0, 3, 1, 2) if extra else 0)
    if flag or extra:
        want = torch.relu(want)
    got = y.float().permute(0, 3, 1, 2)
    assert ((got - want).norm() / want.norm()).item() < 1e-2


def _run_wgrad(case, seed, out_path=None):
    from paper_2207_06667_b200 import _lib
    N, H, W = case
    g = torch.Generator().manual_seed(seed)
    x = torch.randn(N, H, W, 64, generator=g).to(torch.bfloat16).cuda()
    dz = (torch.randn(N, H, W, 64, generator=g) * 0.1).to(torch.bfloat16).cuda()
    s = torch.cuda.current_stream().cuda_stream
    ws = torch.empty(int(_lib.load().edl_bwd_weight_workspace_floats(N * H * W, 64, 576)), device="cuda")
    outs = []
    for _ in range(2):   # determinism: two runs
        dw = torch.full((64, 576), float("nan"), device="cuda")
        _lib.call("edl_conv_bwd_weight_nhwc", x.data_ptr(), N, H, W, 64, 3, 3, 1, 1, dz.data_ptr(), 64, 64,
                  dw.data_ptr(), 576, None, ws.data_ptr(), ws.numel(), 0.5, s)
        torch.cuda.synchronize()
        outs.append(dw.cpu())
    if out_path:
        torch.save(outs[0], out_path)
    return outs, x.cpu(), dz.cpu()


@pytest.mark.parametrize("case", [(2, 14, 14), (3, 17, 17), (1, 9, 62), (8, 56, 56), (2, 7, 30)])
def test_halo_wgrad_vs_im2col_and_torch(case, tmp_path):
    """The halo weight gradient (edl_conv_bwd_weight_nhwc for 64 -> 64 3x3
    stride-1 layers without db) against the im2col split-K path (EDL_HALO=0 in
    a subprocess; fp32 sums in another order: <= 1e-5 relative) and torch's
    fp32 dz^T im2col(x) (<= 1e-3); deterministic (two runs bitwise equal)."""
    import subprocess
    import sys

    import torch.nn.functional as F
    seed = sum(case) * 7
    (a, b), x, dz = _run_wgrad(case, seed)
    assert torch.equal(a, b)
    assert torch.isfinite(a).all()
    ref_path = str(tmp_path / "ref.pt")
    code = ("import sys, torch; sys.path.insert(0, '.'); sys.path.insert(0, 'tests');"
            "import test_gpu_halo as t;"
            f"t._run_wgrad({case!r}, {seed}, {ref_path!r})")
    env = dict(__import__("os").environ, EDL_HALO="0")
    subprocess.run([sys.executable, "-c", code], check=True, env=env, timeout=300)
    ref = torch.load(ref_path)
    assert ((a - ref).norm() / ref.norm()).item() < 1e-5
    N, H, W = case
    cols = F.unfold(x.float().permute(0, 3, 1, 2), 3, padding=1)          # [N][C*9][HW], (c, r, s) order
    cols = cols.view(N, 64, 9, H * W).permute(0, 3, 2, 1).reshape(N * H * W, 576)   # -> (r, s, c)
    want = 0.5 * dz.float().reshape(-1, 64).T @ cols
    assert ((a - want).norm() / want.norm()).item() < 1e-3
