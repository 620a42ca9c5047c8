"""The cfg4 teacher's stage-1 1x1 expansion (256 x 56 x 56 pixels, 64 -> 256
channels, bias + residual + ReLU) through edl_linear_fwd_residual: CUDA-event
time and algorithmic bytes (x, residual in; y out); NCU=1 runs it once."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2207_06667_b200 import _lib  # noqa: E402


def main(M=802816, K=64, N=256, iters=20):
    torch.cuda.set_device(0)
    x = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    w = (torch.randn(N, K, device="cuda") * 0.1).to(torch.bfloat16)
    b = torch.zeros(N, device="cuda")
    r = torch.randn(M, N, device="cuda").to(torch.bfloat16)
    y = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    s = torch.cuda.current_stream().cuda_stream

    mode = os.environ.get("EXP_MODE", "res")

    def run():
        if mode == "res":
            _lib.call("edl_linear_fwd_residual", x.data_ptr(), K, w.data_ptr(), K, b.data_ptr(), r.data_ptr(), N,
                      y.data_ptr(), N, M, N, K, s)
        else:   # "relu" / "ident": the same GEMM without the residual
            _lib.call("edl_linear_fwd", x.data_ptr(), K, w.data_ptr(), K, b.data_ptr(), y.data_ptr(), N, M, N, K,
                      _lib.EDL_ACT_RELU if mode == "relu" else _lib.EDL_ACT_IDENT, s)
    if os.environ.get("NCU"):
        run()
        torch.cuda.synchronize()
        return
    for _ in range(3):
        run()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        run()
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / iters * 1e3
    nbytes = M * K * 2 + (2 if mode == "res" else 1) * M * N * 2
    print(json.dumps({"mode": mode, "env": {k: v for k, v in os.environ.items() if k.startswith("EDL_")},
                      "us": round(us, 1),
                      "GB_per_s": round(nbytes / us / 1e3, 1)}))


if __name__ == "__main__":
    main()
