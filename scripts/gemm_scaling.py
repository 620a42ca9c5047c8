"""Fixed vs per-k-block cost of a one-wave GEMM: time edl_linear_fwd at one
(M, N) over a range of K and fit T = a + b * K (a = launch + prologue +
epilogue + drain, b = main-loop cost per unit K).

    python scripts/gemm_scaling.py [--M 4096] [--N 1008] [--act 0]
"""

import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2207_06667_b200 import _lib  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--M", type=int, default=4096)
    ap.add_argument("--N", type=int, default=1008)
    ap.add_argument("--act", type=int, default=0)
    ap.add_argument("--iters", type=int, default=50)
    a = ap.parse_args()
    st = torch.cuda.current_stream().cuda_stream
    res = {}
    for K in (64, 256, 512, 1024, 2048, 4096):
        x = [torch.randn(a.M, K, device="cuda").to(torch.bfloat16) for _ in range(2)]
        w = (torch.randn(a.N, K, device="cuda") * K ** -0.5).to(torch.bfloat16)
        b = torch.zeros(a.N, device="cuda")
        y = torch.empty(a.M, a.N, device="cuda", dtype=torch.float32 if a.act == 0 else torch.bfloat16)

        def run(i):
            _lib.call("edl_linear_fwd", x[i % 2].data_ptr(), K, w.data_ptr(), K, b.data_ptr(), y.data_ptr(), a.N,
                      a.M, a.N, K, a.act, st)
        for i in range(5):
            run(i)
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for i in range(a.iters):
            run(i)
        e.record()
        torch.cuda.synchronize()
        res[K] = s.elapsed_time(e) / a.iters * 1e3
    Ks = np.array(sorted(res))
    Ts = np.array([res[k] for k in Ks])
    slope, icept = np.polyfit(Ks, Ts, 1)
    print(json.dumps({"M": a.M, "N": a.N, "us_by_K": {int(k): round(res[k], 2) for k in Ks},
                      "fit_fixed_us": round(float(icept), 2), "fit_us_per_1024K": round(float(slope) * 1024, 2)}))


if __name__ == "__main__":
    main()
