"""Per-kernel timing at the cfg3 (wide MLP) shapes: CUDA events on the launch
stream, warm-up first, two input buffers alternated between iterations.

    python scripts/microbench.py [--batch 4096] [--iters 20] [--only t_fwd2,kd_loss]
"""

import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2207_06667_b200 import _lib  # noqa: E402

PEAK = 1389.5  # MEASURED_PEAKS.json bf16_tflops_sustained


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
    ap.add_argument("--only", default="", help="comma-separated entries to run (default: all)")
    a = ap.parse_args()
    only = set(filter(None, a.only.split(",")))
    B = a.batch
    st = torch.cuda.current_stream().cuda_stream
    bf = torch.bfloat16
    res = {}

    def want(name):
        return not only or name in only

    def rec(name, t, flop=None, byts=None):
        r = {"us": round(t * 1e6, 2)}
        if flop:
            r["tflops"] = round(flop / t / 1e12, 1)
            r["frac"] = round(flop / t / 1e12 / PEAK, 4)
        if byts:
            r["gbs"] = round(byts / t / 1e9, 1)
        res[name] = r

    # forward GEMMs (M=B, N, K)
    for name, N, K, act in [("t_fwd1", 8192, 3072, 1), ("t_fwd2", 8192, 8192, 1), ("s_fwd1", 2048, 3072, 1),
                            ("s_fwd2", 1024, 2048, 1), ("s_fwd3", 1008, 1024, 0)]:
        if not want(name):
            continue
        xs = [torch.randn(B, K, device="cuda").to(bf) for _ in range(2)]
        w = (torch.randn(N, K, device="cuda") * K ** -0.5).to(bf)
        b = torch.zeros(N, device="cuda")
        y = torch.empty(B, N, device="cuda", dtype=bf if act else torch.float32)
        t = timeit(lambda i: _lib.call("edl_linear_fwd", xs[i % 2].data_ptr(), K, w.data_ptr(), K, b.data_ptr(),
                                       y.data_ptr(), N, B, N, K, act, st), a.iters)
        rec(name, t, 2 * B * N * K)
    # backward data: dX[B,K] = dY[B,N] W[N,K] * (1 - H^2)
    for name, N, K in [("s_bwd_data2", 1024, 2048), ("s_bwd_data3", 1008, 1024)]:
        if not want(name):
            continue
        dy = torch.randn(B, N, device="cuda").to(bf)
        w = torch.randn(N, K, device="cuda").to(bf)
        h = torch.randn(B, K, device="cuda").to(bf)
        dx = torch.empty(B, K, device="cuda", dtype=bf)
        t = timeit(lambda i: _lib.call("edl_linear_bwd_data", dy.data_ptr(), N, w.data_ptr(), K, h.data_ptr(), K,
                                       dx.data_ptr(), K, B, N, K, st), a.iters)
        rec(name, t, 2 * B * N * K)
    # backward weight, per layer: dW[N,K] = dY^T X (+ db when with_db)
    for name, N, K in [("s_bwd_w1", 2048, 3072), ("s_bwd_w2", 1024, 2048), ("s_bwd_w3", 1008, 1024)]:
        if not want(name):
            continue
        dy = torch.randn(B, N, device="cuda").to(bf)
        x = torch.randn(B, K, device="cuda").to(bf)
        dw = torch.empty(N, K, device="cuda")
        t = timeit(lambda i: _lib.call("edl_linear_bwd_weight", dy.data_ptr(), N, x.data_ptr(), K, dw.data_ptr(), K,
                                       None, None, B, N, K, 1.0, st), a.iters)
        rec(name, t, 2 * B * N * K)
    # the three student dW in one grouped launch, with and without the db column sums
    shapes = [(2048, 3072), (1024, 2048), (1008, 1024)]
    if want("s_bwd_w_grouped") or want("s_bwd_w_grouped_db"):
        dys = [torch.randn(B, n, device="cuda").to(bf) for n, _ in shapes]
        xs = [torch.randn(B, kk, device="cuda").to(bf) for _, kk in shapes]
        dws = [torch.empty(n, kk, device="cuda") for n, kk in shapes]
        dbs = [torch.empty(n, device="cuda") for n, _ in shapes]
        ws = torch.empty(_lib.colsum_group_workspace_floats([B] * 3, [n for n, _ in shapes]), device="cuda")
        fl = sum(2 * B * n * kk for n, kk in shapes)
        P = _lib.c_void_p * 3
        nodb = P(None, None, None)
        L = _lib.load()

        def grouped(with_db):
            def f(i):
                if with_db:
                    _lib.bwd_weight_grouped(dys, xs, dws, dbs, ws, [B] * 3, [n for n, _ in shapes],
                                            [kk for _, kk in shapes], 1.0, st)
                else:
                    I3 = _lib.c_int * 3
                    LL3 = _lib.c_ll * 3
                    _lib.check(L.edl_linear_bwd_weight_grouped(
                        3, P(*[t.data_ptr() for t in dys]), LL3(*[t.stride(0) for t in dys]),
                        P(*[t.data_ptr() for t in xs]), LL3(*[t.stride(0) for t in xs]),
                        P(*[t.data_ptr() for t in dws]), LL3(*[kk for _, kk in shapes]), nodb, None,
                        I3(B, B, B), I3(*[n for n, _ in shapes]), I3(*[kk for _, kk in shapes]), 1.0, st), "grouped")
            return f
        rec("s_bwd_w_grouped", timeit(grouped(False), a.iters), fl)
        rec("s_bwd_w_grouped_db", timeit(grouped(True), a.iters), fl)
    # teacher head: GEMM + fused tempered softmax + top-16
    if want("t_head"):
        H, C, k = 8192, 1000, 16
        hs = [torch.randn(B, H, device="cuda").to(bf) for _ in range(2)]
        w = (torch.randn(1008, H, device="cuda") * H ** -0.5).to(bf)
        b = torch.zeros(1008, device="cuda")
        vals = torch.empty(B, k, device="cuda")
        idx = torch.empty(B, k, device="cuda", dtype=torch.int32)
        t = timeit(lambda i: _lib.call("edl_teacher_head_softmax_topk", hs[i % 2].data_ptr(), H, w.data_ptr(), H,
                                       b.data_ptr(), B, C, H, 2.0, k, vals.data_ptr(), idx.data_ptr(), st), a.iters)
        rec("t_head", t, 2 * B * C * H)
    # kd loss (HBM bound): reads z fp32 B x 1000, writes dz bf16
    if want("kd_loss"):
        k = 16
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
        rec("kd_loss", t, byts=B * (1000 * 4 + 1008 * 2 + k * 8 + 8 + 4))
    # sgd over the student's 9.4M params (fp32 p r+w, g r, bf16 copy w)
    if want("sgd"):
        n = 9_430_000
        p = torch.randn(n, device="cuda")
        pb = torch.empty(n, device="cuda", dtype=bf)
        g = torch.randn(n, device="cuda")
        t = timeit(lambda i: _lib.call("edl_sgd_step", p.data_ptr(), pb.data_ptr(), g.data_ptr(), n, 1e-6, st),
                   a.iters)
        rec("sgd", t, byts=n * 14)
    # batch gather (B rows of 3072 bf16 from a 32768-row shard)
    if want("gather"):
        src = torch.randn(32768, 3072, device="cuda").to(bf)
        idx = torch.randperm(32768, device="cuda")[:B].contiguous()
        dst = torch.empty(B, 3072, device="cuda", dtype=bf)
        t = timeit(lambda i: _lib.call("edl_gather_rows", src.data_ptr(), 3072, idx.data_ptr(), dst.data_ptr(),
                                       3072, B, 3072, None, None, st), a.iters)
        rec("gather", t, byts=2 * B * 3072 * 2)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
