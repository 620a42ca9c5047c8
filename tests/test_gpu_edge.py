"""Edge cases on the device path, mirroring the reference's error behaviour
(edl/nnkit.py:31-36,120-131,200-204,265-297) and its boundary shapes: a single
row, ragged (non-multiple-of-16) dims, k = 1, two classes, the largest class
count / k the fused head supports, non-finite inputs, bad class ids."""

import numpy as np
import pytest
import torch

from oracle import nnkit_ref as ref

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def nk():
    from paper_2207_06667_b200 import nnkit
    return nnkit


def _model(nk, dims, seed):
    from paper_2207_06667_b200 import formats
    h = formats.init_model(dims, seed)
    return nk.Model.from_host(h), h


@pytest.mark.parametrize("dims,B,k", [((5, 7, 2), 1, 1), ((5, 7, 2), 3, 2), ((13, 29, 11), 1, 3),
                                      ((21, 40, 33, 9), 130, 9), ((16, 64, 2048), 70, 32),
                                      ((16, 48, 1000), 257, 1)])
def test_head_and_loss_ragged_shapes_vs_oracle(nk, dims, B, k):
    teacher, th = _model(nk, dims, 1)
    x = np.random.default_rng(B).normal(size=(B, dims[0]))
    y = np.random.default_rng(B + 1).integers(0, dims[-1], size=B)
    batch = nk.make_batch(x, y)
    soft = nk.teacher_soft_labels(teacher, batch.inputs, 2.0, k)
    p16 = ref.tempered_softmax(ref.forward_bf16_storage(list(th.weights), list(th.biases), x), 2.0)
    idx = soft.classes.cpu().numpy().astype(np.int64)
    np.testing.assert_allclose(soft.probs.cpu().numpy(), np.take_along_axis(p16, idx, axis=1), atol=3e-4)
    z = ref.forward(list(th.weights), list(th.biases), x)
    zs = np.sort(z, axis=1)[:, ::-1]
    # output is rank-ordered: every adjacent gap among the compared ranks
    # (and the k-th vs (k+1)-th) must clear bf16 storage noise
    gaps = zs[:, :min(k + 1, dims[-1])]
    safe = (gaps[:, :-1] - gaps[:, 1:]).min(axis=1) > 1e-2 if gaps.shape[1] > 1 else np.ones(B, bool)
    order = np.argsort(-z, axis=1, kind="stable")[:, :k]
    assert np.array_equal(idx[safe], order[safe])
    # the student consumes them: loss vs the bf16-storage oracle
    student, sh = _model(nk, dims, 2)
    cfg = nk.TrainConfig(eta=0.1, alpha=0.5, beta=0.5, temperature=2.0, batch_size=B)
    loss, _ = nk.kd_loss(student, batch, soft, cfg)
    q = ref.topk_dense(soft.probs.cpu().numpy().astype(np.float64), idx, dims[-1])
    l16, _, _ = ref.kd_loss_bf16_storage(list(sh.weights), list(sh.biases), x, y, q, 0.5, 0.5, 2.0)
    assert abs(float(loss) - l16) <= 2e-3 * max(1.0, abs(l16))


def test_constant_logits_tie_rule_lower_class_first(nk):
    """All-equal logits (zero weights): top-k must be classes 0..k-1, the
    reference's stable-argsort tie rule (edl/nnkit.py:333)."""
    from paper_2207_06667_b200.formats import HostModel
    dims = (8, 12, 40)
    h = HostModel(dims, (np.zeros((12, 8)), np.zeros((40, 12))), (np.zeros(12), np.zeros(40)))
    m = nk.Model.from_host(h)
    batch = nk.make_batch(np.random.default_rng(0).normal(size=(33, 8)), np.zeros(33, dtype=np.int64))
    soft = nk.teacher_soft_labels(m, batch.inputs, 3.0, 7)
    assert (soft.classes.cpu().numpy() == np.arange(7)).all()
    np.testing.assert_allclose(soft.probs.cpu().numpy(), 1 / 40, rtol=1e-5)
    assert nk.evaluate(m, np.zeros((50, 8)), np.arange(50) % 40, k=1) == pytest.approx(2 / 50)


def test_nonfinite_inputs_raise_numeric_error(nk):
    student, _ = _model(nk, (6, 10, 4), 0)
    x = np.ones((5, 6))
    x[2, 3] = np.inf
    batch = nk.make_batch(x, np.array([0, 1, 2, 3, 0]))
    with pytest.raises(nk.NumericError):
        float(nk.kd_loss(student, batch, None, nk.TrainConfig(alpha=1.0, beta=0.0, batch_size=5))[0])


def test_bad_soft_label_class_raises_shape_error(nk):
    student, _ = _model(nk, (6, 10, 4), 0)
    batch = nk.make_batch(np.zeros((3, 6)), np.array([0, 1, 2]))
    soft = nk.SoftLabels(torch.full((3, 2), 0.5, device="cuda"),
                         torch.tensor([[0, 1], [2, 9], [1, 3]], dtype=torch.int32, device="cuda"), 2.0)
    with pytest.raises(nk.ShapeError):
        float(nk.kd_loss(student, batch, soft, nk.TrainConfig(alpha=0.5, beta=0.5, batch_size=3))[0])


def test_argument_validation_mirrors_reference(nk):
    student, _ = _model(nk, (6, 10, 4), 0)
    batch = nk.make_batch(np.zeros((3, 6)), np.array([0, 1, 2]))
    soft = nk.teacher_soft_labels(student, batch.inputs, 2.0, 2)
    with pytest.raises(nk.ShapeError):            # beta > 0 without soft labels
        nk.kd_loss(student, batch, None, nk.TrainConfig(alpha=0.5, beta=0.5, batch_size=3))
    with pytest.raises(ValueError):               # temperature disagreement
        nk.kd_loss(student, batch, soft, nk.TrainConfig(alpha=0.5, beta=0.5, temperature=3.0, batch_size=3))
    with pytest.raises(ValueError):
        nk.teacher_soft_labels(student, batch.inputs, -1.0, 2)
    with pytest.raises(ValueError):               # k beyond the class count
        nk.teacher_soft_labels(student, batch.inputs, 2.0, 5)
    with pytest.raises(nk.ShapeError):
        nk.make_batch(np.zeros((0, 6)), np.zeros(0))
    with pytest.raises(ValueError):
        nk.TrainConfig(alpha=0.0, beta=0.0)


def test_large_batch_and_width(nk):
    """B = 8192, D = 8192: the GEMMs tile past one wave in every dimension."""
    from paper_2207_06667_b200 import _lib
    B, D, N = 8192, 8192, 1024
    g = torch.Generator(device="cpu").manual_seed(0)
    x = torch.randn(B, D, generator=g).cuda().to(torch.bfloat16)
    w = (torch.randn(N, D, generator=g) * D ** -0.5).cuda().to(torch.bfloat16)
    b = torch.zeros(N, device="cuda")
    y = torch.empty(B, N, device="cuda")
    _lib.call("edl_linear_fwd", x.data_ptr(), D, w.data_ptr(), D, b.data_ptr(), y.data_ptr(), N, B, N, D, 0,
              torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    ref_ = x.float() @ w.float().T
    assert (y - ref_).abs().max().item() < 1e-3 * ref_.abs().max().item()
