"""Teacher layer 2 (4096 x 8192 x 8192, tanh) alone: CUDA-event time of the
pair GEMM under the current EDL_RASTER / EDL_L2HINT environment (raster
group and L2 eviction policies; one setting per process).

    EDL_RASTER=16 EDL_L2HINT=1 python scripts/layer2_raster.py
"""

import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2207_06667_b200 import _lib  # noqa: E402


def main():
    torch.cuda.set_device(0)
    M, N, K = (int(v) for v in os.environ.get("SHAPE", "4096,8192,8192").split(","))
    g = torch.Generator(device="cpu").manual_seed(0)
    x = torch.tanh(torch.randn(M, K, generator=g)).to(torch.bfloat16).cuda()
    w = (torch.randn(N, K, generator=g) * 0.01).to(torch.bfloat16).cuda()
    b = torch.zeros(N, device="cuda")
    y = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    iters = int(os.environ.get("ITERS", "30"))

    def run():
        _lib.call("edl_linear_fwd", x.data_ptr(), K, w.data_ptr(), K, b.data_ptr(), y.data_ptr(), N, M, N, K, 1, s)
    for _ in range(5):
        run()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        run()
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / iters * 1e3
    print(json.dumps({"shape": [M, N, K], "raster": os.environ.get("EDL_RASTER", "default"), "l2hint": os.environ.get("EDL_L2HINT", "0"),
                      "us": round(us, 2), "tflops": round(2.0 * M * N * K / us / 1e6, 1)}))


if __name__ == "__main__":
    main()
