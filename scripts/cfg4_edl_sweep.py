"""cfg4 on one GPU: online (one stream) vs EDL two-stream decoupling at several teacher SM reserves."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2207_06667_b200.resnet import (ResNetConfig, ResNetStudent, ResNetTeacher,  # noqa: E402
                                          StudentResNetConfig, init_resnet, init_student_resnet, to_nhwc)

B = int(os.environ.get("CFG4_BATCH", "256"))
st = ResNetStudent(init_student_resnet(StudentResNetConfig(), 0), "cuda", B)
te = ResNetTeacher(init_resnet(ResNetConfig(), 1), "cuda", B)
rng = np.random.default_rng(0)
xs = [to_nhwc(rng.normal(size=(B, 3, 224, 224)).astype(np.float32), "cuda") for _ in range(2)]
ys = [torch.from_numpy(rng.integers(0, 1000, size=B)).cuda() for _ in range(2)]
for reserve in (0, 20, 40, 60, 80):
    print(reserve, bench._cfg4_edl_streams(st, te, xs, ys, B, 8, 2, 1389.5, reserve=reserve), flush=True)
