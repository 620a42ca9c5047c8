"""One 64 -> 64 3x3 stride-1 conv (cfg4 stage 1: 256 x 56 x 56) forward,
data gradient and weight gradient through the C-ABI, CUDA-event timed (or once under ncu with
NCU=1). EDL_HALO=0 selects the TMA-im2col GEMM path instead of the halo conv.
    python scripts/conv64_bench.py [--N 256] [--H 56]"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2207_06667_b200 import _lib  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--N", type=int, default=256)
    ap.add_argument("--H", type=int, default=56)
    ap.add_argument("--iters", type=int, default=20)
    a = ap.parse_args()
    N, H = a.N, a.H
    torch.cuda.set_device(0)
    x = torch.randn(N, H, H, 64, device="cuda").to(torch.bfloat16)
    w = (torch.randn(64, 576, device="cuda") * 0.06).to(torch.bfloat16)
    b = torch.zeros(64, device="cuda")
    y = torch.empty_like(x)
    wf = torch.empty_like(w)
    dx = torch.empty_like(x)
    s = torch.cuda.current_stream().cuda_stream
    _lib.call("edl_conv_flip_weights", w.data_ptr(), 576, 64, 64, 3, 3, wf.data_ptr(), 576, s)

    def fwd():
        _lib.call("edl_conv_fwd_nhwc", x.data_ptr(), N, H, H, 64, w.data_ptr(), 576, b.data_ptr(), 64, 3, 3, 1, 1,
                  None, 64, y.data_ptr(), 64, _lib.EDL_ACT_IDENT, s)

    def dgrad():
        _lib.call("edl_conv_dgrad_nhwc", x.data_ptr(), N, H, H, 64, wf.data_ptr(), 576, 64, 3, 3, 1, None,
                  y.data_ptr(), dx.data_ptr(), s)

    ws = torch.empty(int(_lib.load().edl_bwd_weight_workspace_floats(N * H * H, 64, 576)), device="cuda")
    dw = torch.empty(64, 576, device="cuda")

    def wgrad():
        _lib.call("edl_conv_bwd_weight_nhwc", x.data_ptr(), N, H, H, 64, 3, 3, 1, 1, y.data_ptr(), 64, 64,
                  dw.data_ptr(), 576, None, ws.data_ptr(), ws.numel(), 1.0, s)
    if os.environ.get("NCU"):
        fwd()
        dgrad()
        wgrad()
        torch.cuda.synchronize()
        return
    flop = 2.0 * N * H * H * 64 * 576
    res = {"halo": os.environ.get("EDL_HALO", "1")}
    for name, fn in (("fwd", fwd), ("dgrad", dgrad), ("wgrad", wgrad)):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.iters):
            fn()
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) / a.iters * 1e3
        res[name] = {"us": round(us, 1), "tflops": round(flop / us / 1e6, 1)}
    print(json.dumps(res))


if __name__ == "__main__":
    main()
