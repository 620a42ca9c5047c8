"""Device path vs. the reference, through the nnkit mirror (B200 only).

Tolerances (north_star: fp32 accumulate, <= 1e-3 relative for bf16 inputs):
  * vs. the oracle run with the device's bf16 storage points emulated
    (inputs, weight copies, hidden activations, dlogits, deltas rounded to
    bf16; everything else fp64): loss rel <= 1e-3, gradient rel-norm <= 1e-2;
  * vs. the plain fp64 reference golden: loss rel <= 2e-2, gradients
    rel-norm <= 5e-2 (bf16 rounding of 7-12-dim inputs dominates);
  * top-k class indices bit-exact wherever the reference gap between the k-th
    and (k+1)-th logit exceeds the bf16 error bound (1e-2 here).
"""

import os

import numpy as np
import pytest
import torch

from oracle import nnkit_ref as ref

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")
DIMS = (12, 24, 16, 7)


def g(name):
    return np.load(os.path.join(GOLD, name + ".npz"))


@pytest.fixture(scope="module")
def nk():
    from paper_2207_06667_b200 import nnkit
    return nnkit


def host_model(flat, dims):
    from paper_2207_06667_b200.formats import HostModel
    ws, bs = ref.unflatten(flat, dims)
    return HostModel(tuple(dims), tuple(ws), tuple(bs))


def dense_soft(nk, probs, t):
    B, K = probs.shape
    return nk.SoftLabels(torch.tensor(probs, dtype=torch.float32, device="cuda"),
                         torch.arange(K, dtype=torch.int32, device="cuda").repeat(B, 1).contiguous(), t)


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


@pytest.mark.parametrize("ci", range(5))
def test_kd_loss_and_grads_vs_reference(nk, ci):
    d = g("kd_loss")
    flat = d[f"c{ci}_params"]
    alpha, beta, t = (float(v) for v in d[f"c{ci}_cfg"])
    x, y, probs = d[f"c{ci}_x"], d[f"c{ci}_y"], d[f"c{ci}_probs"]
    model = nk.Model.from_host(host_model(flat, DIMS))
    batch = nk.make_batch(x, y)
    soft = dense_soft(nk, probs, t) if beta > 0 else None
    cfg = nk.TrainConfig(eta=0.1, alpha=alpha, beta=beta, temperature=t, batch_size=9)
    loss, grads = nk.kd_loss(model, batch, soft, cfg)
    lv = float(loss)
    gdev = nk.flatten_grads(grads)
    ws, bs = ref.unflatten(flat, DIMS)
    l16, gw, gb = ref.kd_loss_bf16_storage(ws, bs, x, y, probs if beta > 0 else None, alpha, beta, t)
    assert abs(lv - l16) <= 1e-3 * abs(l16)
    assert rel(gdev, ref.flatten(gw, gb)) <= 1e-2
    assert abs(lv - float(d[f"c{ci}_loss"])) <= 2e-2 * abs(float(d[f"c{ci}_loss"]))
    assert rel(gdev, d[f"c{ci}_grads"]) <= 5e-2
    # SGD on the fp32 master: p - eta * g exactly as the device computes it
    before = nk.flatten_params(model)
    nk.sgd_step(model, grads, 0.1)
    after = nk.flatten_params(model)
    np.testing.assert_allclose(after, (before.astype(np.float32) - np.float32(0.1) * gdev.astype(np.float32)),
                               rtol=0, atol=1e-6)
    assert rel(after, d[f"c{ci}_after_sgd"]) <= 2e-2


@pytest.mark.parametrize("k", [3, 7])
def test_topk_soft_labels_and_kd_loss_vs_reference(nk, k):
    d = g("kd_loss")
    teacher = nk.Model.from_host(host_model(d["topk_teacher"], (12, 32, 7)))
    x = d["topk_x"]
    batch = nk.make_batch(x, d["topk_y"])
    soft = nk.teacher_soft_labels(teacher, batch.inputs, 2.0, k)
    idx = soft.classes.cpu().numpy()
    vals = soft.probs.cpu().numpy()
    tw, tb = ref.unflatten(d["topk_teacher"], (12, 32, 7))
    z = ref.forward(tw, tb, x)
    zs = np.sort(z, axis=1)[:, ::-1]
    safe = (zs[:, k - 1] - zs[:, k]) > 1e-2 if k < 7 else np.ones(len(x), bool)
    assert safe.mean() > 0.5
    assert np.array_equal(idx[safe], d[f"topk{k}_idx"][safe])
    p16 = ref.tempered_softmax(ref.forward_bf16_storage(tw, tb, x), 2.0)
    np.testing.assert_allclose(vals, np.take_along_axis(p16, idx.astype(np.int64), axis=1), atol=2e-5, rtol=1e-3)
    np.testing.assert_allclose(vals[safe], d[f"topk{k}_vals"][safe], atol=2e-2)
    student = nk.Model.from_host(host_model(d["topk_params"], DIMS))
    cfg = nk.TrainConfig(eta=0.1, alpha=0.5, beta=0.5, temperature=2.0, batch_size=9)
    loss, grads = nk.kd_loss(student, batch, soft, cfg)
    assert abs(float(loss) - float(d[f"topk{k}_loss"])) <= 2e-2 * abs(float(d[f"topk{k}_loss"]))
    assert rel(nk.flatten_grads(grads), d[f"topk{k}_grads"]) <= 5e-2


def test_teacher_soft_labels_cfg1_dense_and_topk(nk):
    """cfg1 (the reference CPU default): pretrained [16,256,256,10] teacher;
    k = K = 10 reproduces the reference's dense INFER_REPLY probs."""
    d = g("cfg1")
    teacher_h = host_model(d["teacher"], (16, 256, 256, 10))
    teacher = nk.Model.from_host(teacher_h)
    x = d["b0_x"]
    batch = nk.make_batch(x, d["b0_y"])
    dense = nk.teacher_soft_labels(teacher, batch.inputs, 2.0, 10)
    p = dense.probs.cpu().numpy()
    c = dense.classes.cpu().numpy().astype(np.int64)
    full = np.zeros_like(p)
    np.put_along_axis(full, c, p, axis=1)
    np.testing.assert_allclose(full.sum(axis=1), 1.0, atol=1e-5)
    np.testing.assert_allclose(full, d["b0_probs"], atol=3e-2)
    tw, tb = ref.unflatten(d["teacher"], (16, 256, 256, 10))
    p16 = ref.tempered_softmax(ref.forward_bf16_storage(tw, tb, x), 2.0)
    np.testing.assert_allclose(full, p16, atol=3e-4)   # tanh.approx + fp32 accumulation
    # top-4: class ids bit-exact where the fp64 logit gap is above the bf16 bound
    top4 = nk.teacher_soft_labels(teacher, batch.inputs, 2.0, 4)
    z = ref.forward(tw, tb, x)
    zs = np.sort(z, axis=1)[:, ::-1]
    safe = (zs[:, 3] - zs[:, 4]) > 1e-2
    order = np.argsort(-d["b0_probs"], axis=1, kind="stable")[:, :4]
    assert safe.mean() > 0.8
    assert np.array_equal(top4.classes.cpu().numpy()[safe], order[safe])
    # the dense device API (forward + tempered_softmax) agrees too
    pt = nk.tempered_softmax(nk.forward(teacher, batch.inputs), 2.0).cpu().numpy()
    np.testing.assert_allclose(pt, p16, atol=3e-4)


def test_cfg1_distillation_trajectory_and_accuracy(nk):
    """40 EDL steps at cfg1 through the device path vs. the reference's own
    trajectory (golden, fp64): parameters, per-step loss and holdout top-1
    within a stated margin."""
    from paper_2207_06667_b200.data import DeviceDataset, DeviceShardSampler
    from paper_2207_06667_b200.formats import make_blobs
    d = g("cfg1")
    data = make_blobs(0, 2048, 16, 10, 1.0)
    assert data.id == str(d["data_id"])
    dd = DeviceDataset(data)
    sampler = DeviceShardSampler(dd, 1, 0, 32, seed=0)
    teacher = nk.Model.from_host(host_model(d["teacher"], (16, 256, 256, 10)))
    student = nk.Model.from_host(host_model(d["student0"], (16, 64, 10)))
    cfg = nk.TrainConfig(eta=0.05, alpha=0.5, beta=0.5, temperature=2.0, batch_size=32)
    losses = []
    for it in range(int(d["steps"])):
        b = sampler.batch_for(it)
        soft = nk.teacher_soft_labels(teacher, b.inputs, 2.0, 10)
        loss, grads = nk.kd_loss(student, b, soft, cfg)
        losses.append(float(loss))
        nk.sgd_step(student, grads, cfg.eta)
    np.testing.assert_allclose(losses, d["losses"], rtol=2e-2)
    assert rel(nk.flatten_params(student), d["student_final"]) <= 2e-2
    hold = make_blobs(0, 3048, 16, 10, 1.0)
    acc = nk.evaluate(student, hold.samples[2048:], hold.labels[2048:], 1)
    assert abs(acc - float(d["holdout_top1_student"])) <= 0.02


def test_edld_teacher_ingest_and_checkpoint_write_back(nk, tmp_path):
    """A reference-written EDLD teacher (the cfg1 pretrained teacher, golden)
    loads onto the device (f64 -> fp32 master + bf16) and serves the same soft
    labels; a device model written back is a valid EDLD file whose f64 params
    are the fp32 masters exactly."""
    from paper_2207_06667_b200 import formats
    d = g("cfg1")
    host = host_model(d["teacher"], (16, 256, 256, 10))
    p = tmp_path / "teacher.edld"
    p.write_bytes(formats.serialize_model(host, 7))
    dev, it = nk.load_model(str(p))
    assert it == 7 and dev.layer_dims == (16, 256, 256, 10)
    np.testing.assert_array_equal(nk.flatten_params(dev), d["teacher"].astype(np.float32).astype(np.float64))
    x = nk.make_batch(d["b0_x"], d["b0_y"]).inputs
    direct = nk.teacher_soft_labels(nk.Model.from_host(host), x, 2.0, 4)
    loaded = nk.teacher_soft_labels(dev, x, 2.0, 4)
    assert torch.equal(direct.probs, loaded.probs) and torch.equal(direct.classes, loaded.classes)
    q = tmp_path / "ckpt.edld"
    nk.save_model(str(q), dev, 123)
    back, it2 = formats.deserialize_model(q.read_bytes())
    assert it2 == 123
    np.testing.assert_array_equal(ref.flatten(list(back.weights), list(back.biases)), nk.flatten_params(dev))


def test_fused_sgd_step_matches_kd_loss_then_sgd(nk):
    """kd_loss(..., fused_sgd_eta) (dW/db + SGD in the GEMM / column-sum
    epilogues) == kd_loss + sgd_step, on the fp32 masters and the bf16 copies."""
    from paper_2207_06667_b200 import formats
    host = formats.init_model((40, 96, 48, 30), 4)
    data = formats.make_blobs(2, 300, 40, 30, 1.0)
    batch = nk.make_batch(data.samples, data.labels)
    teacher = nk.Model.from_host(formats.init_model((40, 64, 30), 5))
    soft = nk.teacher_soft_labels(teacher, batch.inputs, 2.0, 8)
    cfg = nk.TrainConfig(eta=0.07, alpha=0.6, beta=0.4, temperature=2.0, batch_size=300)
    a = nk.Model.from_host(host)
    b = nk.Model.from_host(host)
    for _ in range(3):
        la, ga = nk.kd_loss(a, batch, soft, cfg, ws=nk.Workspace(a, 300))
        nk.sgd_step(a, ga, cfg.eta)
        lb, gb = nk.kd_loss(b, batch, soft, cfg, ws=nk.Workspace(b, 300), fused_sgd_eta=cfg.eta)
        assert gb is None
        assert float(la) == float(lb)
    torch.cuda.synchronize()
    assert (a.flat - b.flat).abs().max().item() <= 1e-6 * max(1.0, a.flat.abs().max().item())
    assert (a.flat_bf16.float() - b.flat_bf16.float()).abs().max().item() <= 1e-2


def test_error_mapping(nk):
    model = nk.Model((8, 16, 4))
    batch = nk.make_batch(np.zeros((3, 8)), np.array([0, 1, 9]))
    with pytest.raises(nk.ShapeError):
        float(nk.kd_loss(model, batch, None, nk.TrainConfig(alpha=1.0, beta=0.0, batch_size=3))[0])
    with pytest.raises(ValueError):
        nk.tempered_softmax(torch.zeros(2, 4, device="cuda"), 0.0)
    with pytest.raises(nk.ShapeError):
        nk.forward(model, torch.zeros(3, 32, dtype=torch.bfloat16, device="cuda"))
