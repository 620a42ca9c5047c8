"""cfg4 student timing: the ResNet-18-style KD step (training-mode BN;
CFG4_BN=0 for the BN-free variant) alone and the
co-located (online) teacher ResNet-50 -> student step, at a few batch sizes.

    python scripts/cfg4_student_bench.py                 # timings
    CFG4_PROFILE=1 CFG4_BATCH=128 ncu --metrics gpu__time_duration.sum --csv \
        python scripts/cfg4_student_bench.py              # one step for a launch list
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2207_06667_b200.resnet import (ResNetConfig, ResNetStudent, ResNetTeacher,  # noqa: E402
                                          StudentResNetConfig, init_resnet, init_student_resnet, to_nhwc)


def run(B, iters=6, warmup=2, with_teacher=False, profile=False):
    bn = os.environ.get("CFG4_BN", "1") != "0"
    st = ResNetStudent(init_student_resnet(StudentResNetConfig(bn=bn), 0), "cuda", B)
    te = ResNetTeacher(init_resnet(ResNetConfig(), 1), "cuda", B) if with_teacher else None
    rng = np.random.default_rng(0)
    xs = [to_nhwc(rng.normal(size=(B, 3, 224, 224)).astype(np.float32), "cuda") for _ in range(2)]
    ys = [torch.from_numpy(rng.integers(0, 1000, size=B)).cuda() for _ in range(2)]

    def step(i):
        soft = te.soft_labels(xs[i % 2], 2.0, 16) if te is not None else None
        return st.train_step(xs[i % 2], ys[i % 2], soft, 0.5, 0.5 if te is not None else 0.0, 2.0, 1e-3)

    for i in range(warmup):
        step(i)
    torch.cuda.synchronize()
    if profile:
        step(0)
        torch.cuda.synchronize()
        return None
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for i in range(iters):
        loss = step(i)
    e.record()
    torch.cuda.synchronize()
    t = s.elapsed_time(e) / 1e3 / iters
    flop = st.flops_per_sample() + (te.flops_per_sample() if te is not None else 0.0)
    return {"B": B, "bn": bn, "teacher": with_teacher, "samples_per_s": round(B / t, 1), "ms": round(t * 1e3, 3),
            "tflops": round(B * flop / t / 1e12, 1), "gflop_per_sample": round(flop / 1e9, 3),
            "loss": round(float(loss.item()), 4)}


if __name__ == "__main__":
    if os.environ.get("CFG4_PROFILE"):
        run(int(os.environ.get("CFG4_BATCH", "128")), with_teacher=bool(os.environ.get("CFG4_TEACHER")),
            profile=True)
        print("ok")
    else:
        for B in (64, 128, 256):
            print(run(B), flush=True)
        for B in (128, 256):
            print(run(B, with_teacher=True), flush=True)
