"""Per-kernel timing at the cfg3 (wide MLP) shapes: CUDA events on the launch
stream, warm-up first, inputs larger than L2 rotated between iterations.

    python scripts/microbench.py [--batch 4096] [--iters 20]
"""

import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2207_06667_b200 import _lib  # noqa: E402


def timeit(fn, iters, warm=3):
    for _ in range(warm):
        fn(0)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for i in range(iters):
        fn(i)
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters * 1e-3


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=4096)
    ap.add_argument("--iters", type=int, default=20)
    a = ap.parse_args()
    B = a.batch
    st = torch.cuda.current_stream().cuda_stream
    bf = torch.bfloat16
    res = {}
    peak = 1389.5
    # forward GEMMs: (M=B, N, K)
    for name, N, K, act in [("t_fwd1", 8192, 3072, 1), ("t_fwd2", 8192, 8192, 1), ("s_fwd1", 2048, 3072, 1),
                            ("s_fwd2", 1024, 2048, 1), ("s_fwd3", 1008, 1024, 0)]:
        xs = [torch.randn(B, K, device="cuda").to(bf) for _ in range(2)]
        w = (torch.randn(N, K, device="cuda") * K ** -0.5).to(bf)
        b = torch.zeros(N, device="cuda")
        y = torch.empty(B, N, device="cuda", dtype=bf if act else torch.float32)
        t = timeit(lambda i: _lib.call("edl_linear_fwd", xs[i % 2].data_ptr(), K, w.data_ptr(), K, b.data_ptr(),
                                       y.data_ptr(), N, B, N, K, act, st), a.iters)
        res[name] = dict(us=t * 1e6, tflops=2 * B * N * K / t / 1e12)
    # backward data: dX[B,K] = dY[B,N] W[N,K]
    for name, N, K in [("s_bwd_data2", 1024, 2048), ("s_bwd_data3", 1008, 1024)]:
        dy = torch.randn(B, N, device="cuda").to(bf)
        w = torch.randn(N, K, device="cuda").to(bf)
        h = torch.randn(B, K, device="cuda").to(bf)
        dx = torch.empty(B, K, device="cuda", dtype=bf)
        t = timeit(lambda i: _lib.call("edl_linear_bwd_data", dy.data_ptr(), N, w.data_ptr(), K, h.data_ptr(), K,
                                       dx.data_ptr(), K, B, N, K, st), a.iters)
        res[name] = dict(us=t * 1e6, tflops=2 * B * N * K / t / 1e12)
    # backward weight: dW[N,K] = dY^T X, + db
    for name, N, K in [("s_bwd_w1", 2048, 3072), ("s_bwd_w2", 1024, 2048), ("s_bwd_w3", 1008, 1024)]:
        dy = torch.randn(B, N, device="cuda").to(bf)
        x = torch.randn(B, K, device="cuda").to(bf)
        dw = torch.empty(N, K, device="cuda")
        db = torch.empty(N, device="cuda")
        ws = torch.empty(int(_lib.load().edl_colsum_workspace_floats(B, N)), device="cuda")
        t = timeit(lambda i: _lib.call("edl_linear_bwd_weight", dy.data_ptr(), N, x.data_ptr(), K, dw.data_ptr(), K,
                                       db.data_ptr(), ws.data_ptr(), B, N, K, 1.0, st), a.iters)
        res[name] = dict(us=t * 1e6, tflops=2 * B * N * K / t / 1e12)
    # operand-major experiment: the dW1 problem (M=2048, N=3072, K=4096) with
    # K-major operands through the forward kernel, vs. MN-major (s_bwd_w1)
    xa = torch.randn(2048, B, device="cuda").to(bf)
    xb = torch.randn(3072, B, device="cuda").to(bf)
    yo = torch.empty(2048, 3072, device="cuda")
    t = timeit(lambda i: _lib.call("edl_linear_fwd", xa.data_ptr(), B, xb.data_ptr(), B, None, yo.data_ptr(), 3072,
                                   2048, 3072, B, 0, st), a.iters)
    res["dw1_shape_kmajor"] = dict(us=t * 1e6, tflops=2 * B * 2048 * 3072 / t / 1e12)
    # the three student dW in one grouped launch (what the backward pass issues)
    shapes = [(2048, 3072), (1024, 2048), (1008, 1024)]
    dys = [torch.randn(B, n, device="cuda").to(bf) for n, _ in shapes]
    xs = [torch.randn(B, kk, device="cuda").to(bf) for _, kk in shapes]
    dws = [torch.empty(n, kk, device="cuda") for n, kk in shapes]
    dbs = [torch.empty(n, device="cuda") for n, _ in shapes]
    ws = torch.empty(max(int(_lib.load().edl_colsum_workspace_floats(B, n)) for n, _ in shapes), device="cuda")
    t = timeit(lambda i: _lib.bwd_weight_grouped(dys, xs, dws, dbs, ws, [B] * 3, [n for n, _ in shapes],
                                                 [kk for _, kk in shapes], 1.0, st), a.iters)
    fl = sum(2 * B * n * kk for n, kk in shapes)
    res["s_bwd_w_grouped"] = dict(us=t * 1e6, tflops=fl / t / 1e12)
    # teacher head
    H, C, k = 8192, 1000, 16
    hs = [torch.randn(B, H, device="cuda").to(bf) for _ in range(2)]
    w = (torch.randn(1008, H, device="cuda") * H ** -0.5).to(bf)
    b = torch.zeros(1008, device="cuda")
    vals = torch.empty(B, k, device="cuda")
    idx = torch.empty(B, k, device="cuda", dtype=torch.int32)
    t = timeit(lambda i: _lib.call("edl_teacher_head_softmax_topk", hs[i % 2].data_ptr(), H, w.data_ptr(), H,
                                   b.data_ptr(), B, C, H, 2.0, k, vals.data_ptr(), idx.data_ptr(), st), a.iters)
    res["t_head"] = dict(us=t * 1e6, tflops=2 * B * C * H / t / 1e12)
    # kd loss (HBM bound): reads z fp32 B x 1000, writes dz bf16
    z = torch.randn(B, 1008, device="cuda")
    y = torch.randint(0, 1000, (B,), device="cuda")
    qv = torch.rand(B, k, device="cuda")
    qi = torch.randint(0, 1000, (B, k), device="cuda", dtype=torch.int32)
    row = torch.empty(B, device="cuda")
    loss = torch.empty(1, device="cuda")
    ticket = torch.zeros(1, dtype=torch.int32, device="cuda")
    status = torch.zeros(1, dtype=torch.int32, device="cuda")
    dz = torch.empty(B, 1008, device="cuda", dtype=bf)
    t = timeit(lambda i: _lib.call("edl_kd_loss_fwd_bwd", z.data_ptr(), 1008, y.data_ptr(), qv.data_ptr(),
                                   qi.data_ptr(), B, 1000, k, 0.5, 0.5, 2.0, row.data_ptr(), loss.data_ptr(),
                                   ticket.data_ptr(), dz.data_ptr(), 1008, status.data_ptr(), st), a.iters)
    byts = B * (1000 * 4 + 1008 * 2 + k * 8 + 8 + 4)
    res["kd_loss"] = dict(us=t * 1e6, gbs=byts / t / 1e9)
    # sgd over the student's 9.4M params
    n = 9_430_000
    p = torch.randn(n, device="cuda")
    pb = torch.empty(n, device="cuda", dtype=bf)
    g = torch.randn(n, device="cuda")
    t = timeit(lambda i: _lib.call("edl_sgd_step", p.data_ptr(), pb.data_ptr(), g.data_ptr(), n, 1e-6, st), a.iters)
    res["sgd"] = dict(us=t * 1e6, gbs=n * 14 / t / 1e9)
    for k_, v in res.items():
        if "tflops" in v:
            v["frac"] = v["tflops"] / peak
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
