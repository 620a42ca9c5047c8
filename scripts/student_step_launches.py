"""A few cfg3 student steps (B=4096, fused SGD) and one teacher batch, for an
ncu launch list of every kernel they run:

    ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv \\
        python scripts/student_step_launches.py
"""

import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2207_06667_b200 import formats, nnkit  # noqa: E402
from paper_2207_06667_b200.data import DeviceDataset, DeviceShardSampler  # noqa: E402
from paper_2207_06667_b200.student import StudentStep  # noqa: E402


def main():
    torch.cuda.set_device(0)
    B = 4096
    data = DeviceDataset(formats.make_blobs(0, 16384, 3072, 1000, 1.0))
    sampler = DeviceShardSampler(data, 1, 0, B, seed=0)
    teacher = nnkit.Model.from_host(formats.init_model((3072, 8192, 8192, 1000), 1))
    cfg = nnkit.TrainConfig(eta=0.05, alpha=0.5, beta=0.5, temperature=2.0, batch_size=B)
    eng = StudentStep(nnkit.Model.from_host(formats.init_model((3072, 2048, 1024, 1000), 0)), cfg, B, 1)
    tws = nnkit.Workspace(teacher, B)
    for it in range(3):
        b = sampler.batch_for(it, out=eng.batch)
        soft = nnkit.teacher_soft_labels(teacher, b.inputs, 2.0, 16, ws=tws)
        eng.step(b, soft)
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
