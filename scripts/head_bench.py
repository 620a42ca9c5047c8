"""Same-process timing of the cfg3 teacher head (B=4096, H=8192, K=1000,
k=16): the single-CTA cluster head vs the CTA-pair head.

    python scripts/head_bench.py [--iters 100]
"""

import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2207_06667_b200 import _lib  # noqa: E402


def timeit(fn, iters, warm=5):
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
    ap.add_argument("--iters", type=int, default=100)
    a = ap.parse_args()
    torch.cuda.set_device(0)
    B, H, K, Kp, k = 4096, 8192, 1000, 1008, 16
    g = torch.Generator(device="cpu").manual_seed(0)
    h = torch.tanh(torch.randn(B, H, generator=g)).to(torch.bfloat16).cuda()
    w = torch.zeros(Kp, H, dtype=torch.bfloat16, device="cuda")
    w[:K] = (torch.randn(K, H, generator=g) * 0.03).to(torch.bfloat16).cuda()
    b = torch.zeros(Kp, device="cuda")
    vals = torch.empty(B, k, device="cuda")
    idx = torch.empty(B, k, dtype=torch.int32, device="cuda")
    nb = int(_lib.load().edl_teacher_head_workspace_bytes(B, K, k))
    ws = torch.zeros(nb, dtype=torch.uint8, device="cuda")
    s = torch.cuda.current_stream().cuda_stream

    def cluster():
        _lib.call("edl_teacher_head_softmax_topk", h.data_ptr(), H, w.data_ptr(), H, b.data_ptr(), B, K, H, 2.0, k,
                  vals.data_ptr(), idx.data_ptr(), s)

    def pair():
        _lib.call("edl_teacher_head_softmax_topk_ws", h.data_ptr(), H, w.data_ptr(), H, b.data_ptr(), B, K, H, 2.0,
                  k, vals.data_ptr(), idx.data_ptr(), ws.data_ptr(), nb, s)

    res = {"cluster_us": timeit(cluster, a.iters), "pair_us": timeit(pair, a.iters),
           "cluster_again_us": timeit(cluster, a.iters), "pair_again_us": timeit(pair, a.iters)}
    flop = 2.0 * B * K * H
    res["pair_tflops"] = flop / res["pair_us"] / 1e6
    print(json.dumps({kk: round(v, 2) for kk, v in res.items()}))


if __name__ == "__main__":
    main()
