"""Same-process timing of the student's logit layer + KD loss at cfg3
(B=4096, D=1024, K=1000, k=16): the fused edl_linear_kd_loss_fwd_bwd vs the
logit GEMM (edl_linear_fwd) + edl_kd_loss_fwd_bwd.

    python scripts/kd_head_bench.py [--iters 200]
"""

import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2207_06667_b200 import _lib  # noqa: E402


def timeit(fn, iters, warm=10):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters * 1e3


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=200)
    ap.add_argument("--B", type=int, default=4096)
    a = ap.parse_args()
    torch.cuda.set_device(0)
    B, D, K, Kp, k = a.B, 1024, 1000, 1008, 16
    g = torch.Generator(device="cpu").manual_seed(0)
    h = torch.tanh(torch.randn(B, D, generator=g)).to(torch.bfloat16).cuda()
    w = torch.zeros(Kp, D, dtype=torch.bfloat16, device="cuda")
    w[:K] = (torch.randn(K, D, generator=g) * 0.05).to(torch.bfloat16).cuda()
    bias = torch.zeros(Kp, device="cuda")
    y = torch.randint(0, K, (B,), generator=g).cuda()
    qv = torch.softmax(torch.randn(B, k, generator=g), 1).cuda()
    qi = torch.randint(0, K, (B, k), generator=g).int().cuda()
    row, loss = torch.empty(B, device="cuda"), torch.zeros(1, device="cuda")
    ticket = torch.zeros(1, dtype=torch.int32, device="cuda")
    status = torch.zeros(1, dtype=torch.int32, device="cuda")
    dz = torch.zeros(B, Kp, dtype=torch.bfloat16, device="cuda")
    z = torch.zeros(B, Kp, device="cuda")
    s = torch.cuda.current_stream().cuda_stream

    def fused():
        _lib.call("edl_linear_kd_loss_fwd_bwd", h.data_ptr(), D, w.data_ptr(), D, bias.data_ptr(), y.data_ptr(),
                  qv.data_ptr(), qi.data_ptr(), B, K, D, k, 0.5, 0.5, 2.0, row.data_ptr(), loss.data_ptr(),
                  dz.data_ptr(), Kp, status.data_ptr(), s)

    def gemm():
        _lib.call("edl_linear_fwd", h.data_ptr(), D, w.data_ptr(), D, bias.data_ptr(), z.data_ptr(), Kp, B, Kp, D,
                  0, s)

    def loss_kernel():
        _lib.call("edl_kd_loss_fwd_bwd", z.data_ptr(), Kp, y.data_ptr(), qv.data_ptr(), qi.data_ptr(), B, K, k,
                  0.5, 0.5, 2.0, row.data_ptr(), loss.data_ptr(), ticket.data_ptr(), dz.data_ptr(), Kp,
                  status.data_ptr(), s)

    res = {"fused_us": timeit(fused, a.iters), "gemm_us": timeit(gemm, a.iters),
           "loss_us": timeit(loss_kernel, a.iters)}
    res["unfused_us"] = timeit(lambda: (gemm(), loss_kernel()), a.iters)
    res["fused_again_us"] = timeit(fused, a.iters)
    print(json.dumps({kk: round(v, 2) for kk, v in res.items()}))


if __name__ == "__main__":
    main()
