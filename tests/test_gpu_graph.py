"""StudentStep(graph=True): the whole training step replayed as one CUDA
graph (for host-bound loops such as a split placement's student) gives the
same parameters and losses, bit for bit, as the eager step (B200 only)."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("beta", [0.5, 0.0])
def test_graph_step_equals_eager_step(beta):
    from paper_2207_06667_b200 import formats, nnkit
    from paper_2207_06667_b200.data import DeviceDataset, DeviceShardSampler
    from paper_2207_06667_b200.student import StudentStep
    B = 64
    data = DeviceDataset(formats.make_blobs(0, 1024, 48, 10, 1.0))
    teacher = nnkit.Model.from_host(formats.init_model((48, 96, 10), 1))
    host = formats.init_model((48, 80, 32, 10), 2)
    cfg = nnkit.TrainConfig(eta=0.05, alpha=0.5, beta=beta, temperature=2.0, batch_size=B)
    engines = [StudentStep(nnkit.Model.from_host(host), cfg, B, 1, max_steps=16, graph=g) for g in (False, True)]
    for eng in engines:
        sampler = DeviceShardSampler(data, 1, 0, B, seed=0)
        for it in range(8):
            b = sampler.batch_for(it, out=eng.batch if eng._use_graph else None)
            soft = nnkit.teacher_soft_labels(teacher, b.inputs, 2.0, 4) if beta > 0 else None
            eng.step(b, soft)
        eng.check_status()
    torch.cuda.synchronize()
    assert engines[1]._graph is not None
    assert torch.equal(engines[0].model.flat, engines[1].model.flat)
    assert torch.equal(engines[0].model.flat_bf16, engines[1].model.flat_bf16)
    assert np.array_equal(engines[0].loss_values(), engines[1].loss_values())
