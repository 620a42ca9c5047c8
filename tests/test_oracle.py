"""Pin the CPU oracle to the reference: every oracle function against golden
vectors produced by the real reference (oracle/gen_golden.py) and against the
reference's own known-answer tests. CPU only."""

import os

import numpy as np
import pytest

from oracle import nnkit_ref as ref

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def g(name):
    return np.load(os.path.join(GOLD, name + ".npz"))


def test_softmax_reference_kat():
    # frozen 60-digit mpmath values from tests/test_nnkit.py:42-46
    expected = np.array([0.18632372322584757702, 0.30719588571849839707, 0.5064803910556540259])
    np.testing.assert_allclose(ref.tempered_softmax(np.array([1.0, 2, 3]), 2.0), expected, rtol=1e-14)
    d = g("softmax")
    assert np.array_equal(ref.tempered_softmax(d["kat_in"], 2.0), d["kat_out"])


def test_softmax_golden_sweep_bitwise():
    d = g("softmax")
    for i, t in enumerate(d["t"]):
        assert np.array_equal(ref.tempered_softmax(d["z"], float(t)), d["p"][i])


def test_softmax_properties():
    rng = np.random.default_rng(0)
    z = rng.normal(scale=50.0, size=(10_000, 10))
    assert np.abs(ref.tempered_softmax(z, 3.0).sum(axis=1) - 1.0).max() <= 1e-12
    with pytest.raises(ValueError):
        ref.tempered_softmax(np.array([1.0, np.inf]), 1.0)
    with pytest.raises(ValueError):
        ref.tempered_softmax(np.array([1.0, 2.0]), 0.0)


DIMS = (12, 24, 16, 7)


@pytest.mark.parametrize("ci", range(5))
def test_kd_loss_matches_reference(ci):
    d = g("kd_loss")
    ws, bs = ref.unflatten(d[f"c{ci}_params"], DIMS)
    alpha, beta, t = d[f"c{ci}_cfg"]
    x, y, probs = d[f"c{ci}_x"], d[f"c{ci}_y"], d[f"c{ci}_probs"]
    assert np.array_equal(ref.forward(ws, bs, x), d[f"c{ci}_logits"])
    loss, gw, gb = ref.kd_loss(ws, bs, x, y, probs if beta > 0 else None, alpha, beta, t)
    assert loss == float(d[f"c{ci}_loss"])
    assert np.array_equal(ref.flatten(gw, gb), d[f"c{ci}_grads"])
    w2, b2 = ref.sgd_step(ws, bs, gw, gb, 0.1)
    assert np.array_equal(ref.flatten(w2, b2), d[f"c{ci}_after_sgd"])


@pytest.mark.parametrize("k", [3, 7])
def test_topk_soft_labels_match_reference(k):
    d = g("kd_loss")
    tw, tb = ref.unflatten(d["topk_teacher"], (12, 32, 7))
    vals, idx = ref.teacher_soft(tw, tb, d["topk_x"], 2.0, k)
    assert np.array_equal(idx, d[f"topk{k}_idx"])
    assert np.array_equal(vals, d[f"topk{k}_vals"])
    ws, bs = ref.unflatten(d["topk_params"], DIMS)
    q = ref.topk_dense(vals, idx, 7)
    loss, gw, gb = ref.kd_loss(ws, bs, d["topk_x"], d["topk_y"], q, 0.5, 0.5, 2.0)
    assert loss == float(d[f"topk{k}_loss"])
    assert np.array_equal(ref.flatten(gw, gb), d[f"topk{k}_grads"])


def test_topk_equals_dense_at_k_equals_K():
    d = g("kd_loss")
    ws, bs = ref.unflatten(d["topk_params"], DIMS)
    p = d["topk_p"]
    dense = ref.kd_loss(ws, bs, d["topk_x"], d["topk_y"], p, 0.5, 0.5, 2.0)
    full = ref.kd_loss(ws, bs, d["topk_x"], d["topk_y"], ref.topk_dense(*ref.topk(p, 7), 7), 0.5, 0.5, 2.0)
    assert abs(dense[0] - full[0]) < 1e-14
    assert np.abs(ref.flatten(dense[1], dense[2]) - ref.flatten(full[1], full[2])).max() < 1e-14


def test_topk_tie_rule_lower_index_first():
    p = np.array([[0.2, 0.3, 0.2, 0.3]])
    _, idx = ref.topk(p, 3)
    assert idx.tolist() == [[1, 3, 0]]


def test_data_plumbing():
    d = g("data")
    s, l = ref.make_blobs(42, 100, 5, 4, 1.5)
    assert np.array_equal(s, d["blobs_samples"]) and np.array_equal(l, d["blobs_labels"])
    assert np.array_equal(ref.epoch_order(0, 0, 0, 100), d["order"])
    assert np.array_equal(ref.epoch_order(3, 1, 2, 50), d["order_e1"])
    samples, _ = ref.make_blobs(0, 65, 4, 4, 1.0)
    bpe = int(d["bpe"])
    lo, hi = ref.partition_bounds(65, 2, 0)
    assert np.array_equal(samples[lo:hi][ref.batch_rows(0, 0, hi - lo, 16, bpe, 0)], d["s0_b0"])
    assert np.array_equal(samples[lo:hi][ref.batch_rows(0, 0, hi - lo, 16, bpe, 3)], d["s0_b3"])
    lo, hi = ref.partition_bounds(65, 2, 1)
    assert np.array_equal(samples[lo:hi][ref.batch_rows(0, 1, hi - lo, 16, bpe, 1)], d["s1_b1"])


@pytest.mark.parametrize("n", range(1, 6))
def test_ring_reduce_values(n):
    d = g("ring")
    out = ref.ring_reduce_values(list(d[f"n{n}_in"]))
    assert np.array_equal(out, d[f"n{n}_out"])
    np.testing.assert_allclose(out, d[f"n{n}_in"].mean(axis=0), atol=1e-12)


def test_cfg1_teacher_and_trajectory_bitwise():
    d = g("cfg1")
    samples, labels = ref.make_blobs(0, 2048, 16, 10, 1.0)
    tw, tb = ref.pretrain_teacher(samples, labels, 0.1, 32, 0, 3, (256, 256))
    assert np.array_equal(ref.flatten(tw, tb), d["teacher"])
    assert np.array_equal(ref.tempered_softmax(ref.forward(tw, tb, d["b0_x"]), 2.0), d["b0_probs"])
    s0 = ref.init_model((16, 64, 10), 0)
    assert np.array_equal(ref.flatten(*s0), d["student0"])
    (ws, bs), losses = ref.dp_distill_trajectory(s0, (tw, tb), samples, labels, 1, 32, 0, int(d["steps"]),
                                                 0.5, 0.5, 2.0, 0.05)
    assert np.array_equal(np.array(losses), d["losses"])
    assert np.array_equal(ref.flatten(ws, bs), d["student_final"])
    hs, hl = ref.make_blobs(0, 3048, 16, 10, 1.0)
    assert ref.evaluate(tw, tb, hs[2048:], hl[2048:], 1) == float(d["holdout_top1_teacher"])
    assert ref.evaluate(ws, bs, hs[2048:], hl[2048:], 1) == float(d["holdout_top1_student"])


def test_two_student_virtual_cluster_trajectory():
    """N=2 DP oracle == the reference's VirtualCluster final_params (bitwise)."""
    d = g("cfg1")
    samples, labels = ref.make_blobs(0, 2048, 16, 10, 1.0)
    teacher = ref.unflatten(d["teacher"], (16, 256, 256, 10))
    s0 = ref.init_model((16, 64, 10), 0)
    (ws, bs), _ = ref.dp_distill_trajectory(s0, teacher, samples, labels, 2, 32, 0, int(d["vc_steps"]),
                                            0.5, 0.5, 2.0, 0.05)
    assert np.array_equal(ref.flatten(ws, bs), d["vc_final"])
