"""Parity at the full cfg3 sizes (teacher [3072,8192,8192,1000], student
[3072,2048,1024,1000], B=4096, k=16) through properties that do not need the
fp64 oracle to finish: the fused head's top-k equals the top-k of the dense
device path and of a torch fp32 recomputation over the same bf16 operands;
the student's loss and gradients match torch fp32 autograd over the same
bf16 inputs/weights; training reduces the loss. Tolerances as in
test_gpu_nnkit.py (fp32 accumulate, bf16 storage)."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

B, D, K, k, T = 4096, 3072, 1000, 16, 2.0


@pytest.fixture(scope="module")
def setup():
    from paper_2207_06667_b200 import formats, nnkit
    from paper_2207_06667_b200.data import DeviceDataset, DeviceShardSampler
    data = DeviceDataset(formats.make_blobs(0, 8192, D, K, 1.0))
    sampler = DeviceShardSampler(data, 1, 0, B, seed=0)
    teacher = nnkit.Model.from_host(formats.init_model((D, 8192, 8192, K), 1))
    student_h = formats.init_model((D, 2048, 1024, K), 0)
    return nnkit, sampler, teacher, student_h


def test_fused_head_topk_equals_dense_path_full_size(setup):
    nk, sampler, teacher, _ = setup
    batch = sampler.batch_for(0)
    soft = nk.teacher_soft_labels(teacher, batch.inputs, T, k)
    z = nk.forward(teacher, batch.inputs)                    # device dense path (fp32 logits)
    p = nk.tempered_softmax(z, T)
    torch.cuda.synchronize()
    # probabilities of the fused head == dense softmax at the chosen classes
    got = torch.gather(p, 1, soft.classes.long())
    assert (soft.probs - got).abs().max().item() < 1e-5
    # class ids == stable top-k of the dense path where the k-th / (k+1)-th gap
    # exceeds fp32 accumulation-order noise
    zs, order = torch.sort(z, dim=1, descending=True, stable=True)
    safe = (zs[:, k - 1] - zs[:, k]) > 1e-3
    assert safe.float().mean().item() > 0.9
    assert torch.equal(soft.classes[safe].long(), order[safe, :k])
    # simplex properties: sorted descending, probabilities in (0, 1], mass <= 1
    assert (soft.probs[:, :-1] >= soft.probs[:, 1:]).all()
    assert (soft.probs > 0).all() and (soft.probs.sum(1) <= 1 + 1e-5).all()
    # torch fp32 recomputation of the logits from the same bf16 hidden state
    # (layer-2 output is bf16 in both) agrees on the winners
    w = teacher.w_bf16(2)[:K].float()
    h = nk.workspace_for(teacher, B).acts[2].float()
    zt = h @ w.T + teacher.b(2)[:K]
    assert (zt - z).abs().max().item() < 1e-2 * max(1.0, zt.abs().max().item())


def test_student_step_full_size_vs_torch_autograd(setup):
    nk, sampler, teacher, student_h = setup
    batch = sampler.batch_for(1)
    soft = nk.teacher_soft_labels(teacher, batch.inputs, T, k)
    student = nk.Model.from_host(student_h)
    cfg = nk.TrainConfig(eta=0.05, alpha=0.5, beta=0.5, temperature=T, batch_size=B)
    loss, grads = nk.kd_loss(student, batch, soft, cfg)
    lv = float(loss)
    # torch fp32 autograd over the SAME bf16 operands (inputs, weight copies)
    L = student.layout
    x = batch.inputs.float()[:, :D]
    ws = [student.w_bf16(l)[:student.layer_dims[l + 1], :student.layer_dims[l]].float().requires_grad_()
          for l in range(L.layers)]
    bs = [student.b(l)[:student.layer_dims[l + 1]].clone().requires_grad_() for l in range(L.layers)]
    h = x
    for l in range(L.layers):
        z = h @ ws[l].T + bs[l]
        h = z if l == L.layers - 1 else torch.tanh(z)
    q = torch.zeros(B, K, device="cuda").scatter_(1, soft.classes.long(), soft.probs)
    q = q / q.sum(1, keepdim=True)
    y = batch.hard_labels
    ref = 0.5 * torch.nn.functional.cross_entropy(h, y) + \
        0.5 * T * T * (-(q * torch.log_softmax(h / T, 1)).sum(1)).mean()
    ref.backward()
    assert abs(lv - ref.item()) <= 1e-3 * abs(ref.item())
    g = grads.flat
    for l in range(L.layers):
        dw = g[L.w_off[l]:L.w_off[l] + L.dims_p[l + 1] * L.dims_p[l]].view(L.dims_p[l + 1], L.dims_p[l])
        dw = dw[:student.layer_dims[l + 1], :student.layer_dims[l]]
        rel = ((dw - ws[l].grad).norm() / ws[l].grad.norm()).item()
        assert rel < 2e-2, (l, rel)
        db = g[L.b_off[l]:L.b_off[l] + student.layer_dims[l + 1]]
        relb = ((db - bs[l].grad).norm() / bs[l].grad.norm()).item()
        assert relb < 2e-2, (l, relb)


def test_training_reduces_loss_full_size(setup):
    from paper_2207_06667_b200.student import StudentStep
    nk, sampler, teacher, student_h = setup
    cfg = nk.TrainConfig(eta=0.05, alpha=0.5, beta=0.5, temperature=T, batch_size=B)
    eng = StudentStep(nk.Model.from_host(student_h), cfg, B, 1, max_steps=16)
    for it in range(12):
        b = sampler.batch_for(it % 2)
        soft = nk.teacher_soft_labels(teacher, b.inputs, T, k)
        eng.step(b, soft)
    losses = eng.loss_values()
    assert np.isfinite(losses).all()
    assert np.mean(losses[-3:]) < np.mean(losses[:3])
