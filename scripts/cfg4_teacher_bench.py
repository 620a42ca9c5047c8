"""cfg4 teacher inference timing (ResNet-50-style, 224^2, top-16 head) at
batch 256: CUDA events over a few batches (A/B runs via env switches).
    python scripts/cfg4_teacher_bench.py"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2207_06667_b200.resnet import ResNetConfig, ResNetTeacher, init_resnet, to_nhwc  # noqa: E402


def main(B=256, iters=8):
    te = ResNetTeacher(init_resnet(ResNetConfig(), 1), "cuda", B)
    x = to_nhwc(np.random.default_rng(0).normal(size=(B, 3, 224, 224)).astype(np.float32), "cuda")
    for _ in range(2):
        te.soft_labels(x, 2.0, 16)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters):
        out = te.soft_labels(x, 2.0, 16)
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / iters
    print(json.dumps({"env": {k: v for k, v in os.environ.items() if k.startswith("EDL_")}, "ms_per_batch": round(ms, 3),
                      "images_per_s": round(B / ms * 1e3, 1),
                      "tflops": round(B * te.flops_per_sample() / ms / 1e9, 1),
                      "top1_class_sum": int(out.classes[:, 0].sum().item())}))


if __name__ == "__main__":
    main()
