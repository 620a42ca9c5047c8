"""One cfg4 teacher batch (ResNet-50 style, 224^2) for kernel-level profiling:
    ncu --metrics gpu__time_duration.sum --csv python scripts/cfg4_profile.py
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2207_06667_b200.resnet import ResNetConfig, ResNetTeacher, init_resnet, to_nhwc  # noqa: E402

B = int(os.environ.get("CFG4_BATCH", "64"))
teacher = ResNetTeacher(init_resnet(ResNetConfig(), 1), "cuda", B)
x = to_nhwc(np.random.default_rng(0).normal(size=(B, 3, 224, 224)).astype(np.float32), "cuda")
for _ in range(2):
    teacher.soft_labels(x, 2.0, 16)
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("cfg4_batch")
teacher.soft_labels(x, 2.0, 16)
torch.cuda.nvtx.range_pop()
torch.cuda.synchronize()
print("ok")
