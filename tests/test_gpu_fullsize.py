"""Parity at the full cfg3 sizes against the fp64 oracle (B200 only).

cfg3: teacher [3072, 8192, 8192, 1000], student [3072, 2048, 1024, 1000],
B = 4096, k = 16, T = 2, alpha = beta = 0.5.

Two levels, both against oracle/nnkit_ref.py in fp64 (numpy, the box's host
cores; ~2 s for the 256-row teacher slice, ~3 s for the full student batch):

1. Per kernel, on the device's own bf16 operands: every stage is recomputed in
   fp64 from exactly the inputs the kernel read (the device's bf16 inputs,
   activations, dlogits and deltas), so only the kernel's own arithmetic is
   under test, elementwise against the error model of fp32 accumulation:
       |dev - ref| <= ulp_bf16(ref) [bf16 outputs only] + acc(K) * sum_k |a_k b_k|
   with acc(K) = (K / 16) * 2^-24: the worst case of one fp32 rounding per
   16-deep MMA k-step of a K-long reduction (measured typical ~2^-22 at
   K = 3072, profiles/r02_stage_probe.json; the dW GEMMs, K = 4096 rows
   with mostly same-sign terms, reach ~2^-18). The ulp term
   is the store's own half-ulp rounding plus tanh.approx's 2^-11 (measured
   0.502 ulp worst). The sum term matters where the terms cancel: near-zero
   pre-activations and the backprop-data products dz W, whose rows sum to
   ~0. Weight / bias gradients also by relative norm <= 1e-5. Head
   probabilities within 2 acc sum|h w| / T relative; top-k ids bit-exact in
   order wherever every adjacent fp64 logit gap exceeds 4 acc sum|h w|.

2. End to end, against the oracle run with the device's bf16 storage points
   emulated (kd_loss_bf16_storage / forward_bf16_storage) and against the
   plain fp64 reference (north_star: fp32 accumulate, <= 1e-3 relative for
   bf16 inputs):
     * loss: <= 1e-3 relative (measured 1e-8);
     * soft-label probabilities: <= 1e-3 relative, every entry (measured
       8.3e-4 max on the 256-row slice);
     * top-k ids: bit-exact as a set where the oracle's k-th / (k+1)-th logit
       gap exceeds TAU, and position by position wherever the oracle's gaps
       to both neighbours exceed TAU; TAU = 1e-2 against the bf16-storage
       oracle and 4e-2 against fp64 (bf16 input rounding), each >= 2x the
       measured device-vs-oracle logit error (asserted);
     * per-layer gradients: <= 2.5e-3 relative norm against the bf16-storage
       oracle (measured 1.65e-3 layer 0, 8.0e-4 layer 1, 5.9e-4 layer 2;
       profiles/r02_parity_probe.json). The 1e-3 target is not met end to
       end, and not because of a kernel (level 1 holds every kernel to
       1e-5): every bf16 store rounds the kernel's fp32 value, and an fp32
       accumulation that differs from fp64 by ~1e-6 relative lands on the
       other side of a rounding boundary for ~1-5% of the activations and
       deltas; each such flip is a full bf16 ulp (2^-8 relative) and they
       compound through the three layers. The fp64 oracle cannot emulate
       them; tanhf instead of tanh.approx only moves layer 0 from 1.65e-3 to
       1.38e-3.
Measured values are written to $EDL_PARITY_OUT (JSON) when set."""

import json
import os

import numpy as np
import pytest
import torch

from oracle import nnkit_ref as ref

pytestmark = pytest.mark.gpu

B, D, K, k, T = 4096, 3072, 1000, 16, 2.0
ROWS = 256
ULP = 2.0 ** -8          # one bf16 ulp, relative (8 significand bits)


def acc(K):
    """fp32 accumulation error per unit of sum_k |a_k b_k| for a K-long
    tensor-core reduction (one rounding per 16-deep k-step, worst case)."""
    return (K + 15) // 16 * 2.0 ** -24
MEASURED: dict = {}


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def bf16_host(t: torch.Tensor) -> np.ndarray:
    return t.float().cpu().numpy().astype(np.float64)


def ulp_bf16(x):
    a = np.abs(x)
    return np.where(a > 0, np.exp2(np.floor(np.log2(np.where(a > 0, a, 1.0))) - 7), 0.0)


def worst_ratio(dev, ref64, bound):
    """max |dev - ref| / bound (<= 1: every element inside its error model)."""
    return float((np.abs(dev - ref64) / bound).max())


@pytest.fixture(scope="module")
def setup():
    from paper_2207_06667_b200 import formats, nnkit
    from paper_2207_06667_b200.data import DeviceDataset, DeviceShardSampler
    host = formats.make_blobs(0, 8192, D, K, 1.0)
    data = DeviceDataset(host)
    sampler = DeviceShardSampler(data, 1, 0, B, seed=0)
    teacher_h = formats.init_model((D, 8192, 8192, K), 1)
    teacher = nnkit.Model.from_host(teacher_h)
    student_h = formats.init_model((D, 2048, 1024, K), 0)
    yield nnkit, host, sampler, teacher, teacher_h, student_h
    out = os.environ.get("EDL_PARITY_OUT")
    if out:
        with open(out, "w") as fh:
            json.dump(MEASURED, fh, indent=1)


@pytest.fixture(scope="module")
def teacher_run(setup):
    nk, host, sampler, teacher, teacher_h, _ = setup
    batch = sampler.batch_for(0)
    ws = nk.Workspace(teacher, B)
    soft = nk.teacher_soft_labels(teacher, batch.inputs, T, k, ws=ws)
    torch.cuda.synchronize()
    rows = sampler.rows_for(0).cpu().numpy()
    return batch, ws, soft, host.samples[rows[:ROWS]]


def test_teacher_kernels_on_device_operands(setup, teacher_run):
    """Level 1: hidden tanh GEMMs and the fused head, each against fp64 on
    the bf16 operands the kernel read."""
    nk, _, _, teacher, teacher_h, _ = setup
    batch, ws, soft, _ = teacher_run
    wq = [ref.bf16(w) for w in teacher_h.weights]
    h = bf16_host(batch.inputs[:ROWS, :D])
    for l in range(2):
        z = h @ wq[l].T + teacher_h.biases[l]
        t = np.tanh(z)
        dev = bf16_host(ws.acts[l + 1][:ROWS, :teacher.layer_dims[l + 1]])
        worst = worst_ratio(dev, t, ulp_bf16(t) + acc(h.shape[1]) * (np.abs(h) @ np.abs(wq[l]).T))
        MEASURED[f"teacher_layer{l}_tanh_worst_ratio"] = worst
        assert worst <= 1.0, (l, worst)
        h = dev
    z = h @ wq[2].T + teacher_h.biases[2]
    p = ref.tempered_softmax(z, T)
    # logit error model: acc(K) * sum_k |h_k w_k| per logit; a probability moves
    # with the difference of two logits over T (+ ex2.approx's 2^-22)
    smax = acc(h.shape[1]) * (np.abs(h) @ np.abs(wq[2]).T).max(axis=1, keepdims=True)
    idx = soft.classes[:ROWS].cpu().numpy().astype(np.int64)
    vals = soft.probs[:ROWS].cpu().numpy().astype(np.float64)
    pz = np.take_along_axis(p, idx, axis=1)
    r = np.abs(vals - pz) / pz
    worst = float((r / (2 * smax / T + 2.0 ** -20)).max())
    MEASURED["teacher_head_prob_rel_max_on_device_h2"] = float(r.max())
    MEASURED["teacher_head_prob_worst_ratio"] = worst
    assert worst <= 1.0
    s_safe, pinned = _ids_checks("fp64_on_device_h2", z, idx, 4 * smax)
    assert s_safe > 0.6 and pinned > 0.6


def _ids_checks(name, z, idx, tau):
    """Set equality where the oracle's k-th / (k+1)-th gap exceeds tau, and
    position-wise equality at every 'pinned' position j of the top k (the
    oracle's logit gaps to both neighbours exceed tau): bit-exact wherever
    there is no near-tie."""
    zs = np.sort(z, axis=1)[:, ::-1]
    order = np.argsort(-z, axis=1, kind="stable")[:, :k]
    tau = np.broadcast_to(np.asarray(tau, dtype=np.float64).reshape(-1, 1), (len(z), 1))
    set_safe = (zs[:, k - 1] - zs[:, k]) > tau[:, 0]
    same_set = np.array([set(a) == set(b) for a, b in zip(idx.tolist(), order.tolist())])
    gaps = -np.diff(zs[:, :k + 1], axis=1)                    # gaps[:, j] = z_(j) - z_(j+1)
    left = np.concatenate([np.full((len(z), 1), np.inf), gaps[:, :k - 1]], axis=1)
    pinned = (left > tau) & (gaps[:, :k] > tau)
    MEASURED[f"ids_vs_{name}"] = {"tau_max": float(tau.max()), "set_safe_frac": float(set_safe.mean()),
                                  "set_exact_on_safe": float(same_set[set_safe].mean()),
                                  "set_exact_all_rows": float(same_set.mean()),
                                  "pinned_position_frac": float(pinned.mean()),
                                  "pinned_exact": float((idx == order)[pinned].mean())}
    assert same_set[set_safe].all(), name
    assert (idx == order)[pinned].all(), name
    return set_safe.mean(), pinned.mean()


def test_teacher_soft_labels_vs_oracle_slice(setup, teacher_run):
    """Level 2: the fused head's top-16 on a 256-row slice vs the
    bf16-storage oracle and the plain fp64 reference (forward +
    tempered_softmax, edl/nnkit.py:193-234; top-k with the :333 tie rule).
    The tie margins tau are 2x the measured device-vs-oracle logit error
    (dense device path, same hidden GEMMs) rounded up."""
    nk, _, _, teacher, teacher_h, _ = setup
    batch, _, soft, x = teacher_run
    tw, tb = list(teacher_h.weights), list(teacher_h.biases)
    z16 = ref.forward_bf16_storage(tw, tb, x)
    z64 = ref.forward(tw, tb, x)
    zdev = nk.forward(teacher, batch.inputs)[:ROWS].cpu().numpy().astype(np.float64)
    e16, e64 = float(np.abs(zdev - z16).max()), float(np.abs(zdev - z64).max())
    MEASURED["teacher_logit_maxabs_err"] = {"vs_bf16_oracle": e16, "vs_fp64": e64}
    tau16, tau64 = 1e-2, 4e-2
    assert 2 * e16 <= tau16 and 2 * e64 <= tau64, (e16, e64)
    idx = soft.classes[:ROWS].cpu().numpy().astype(np.int64)
    vals = soft.probs[:ROWS].cpu().numpy().astype(np.float64)
    p16 = np.take_along_axis(ref.tempered_softmax(z16, T), idx, axis=1)
    r = np.abs(vals - p16) / p16
    MEASURED["teacher_prob_rel_vs_bf16_oracle"] = {"max": float(r.max()), "mean": float(r.mean())}
    assert r.max() <= 1e-3
    p64 = np.take_along_axis(ref.tempered_softmax(z64, T), idx, axis=1)
    MEASURED["teacher_prob_rel_vs_fp64"] = {"max": float((np.abs(vals - p64) / p64).max())}
    s16, pin16 = _ids_checks("bf16_oracle", z16, idx, tau16)
    _, pin64 = _ids_checks("fp64", z64, idx, tau64)
    assert s16 > 0.4 and pin16 > 0.3 and pin64 > 0.05
    # simplex properties of the shipped pairs
    v = soft.probs
    assert (v[:, :-1] >= v[:, 1:]).all() and (v > 0).all() and (v.sum(1) <= 1 + 1e-5).all()


@pytest.fixture(scope="module")
def student_run(setup, teacher_run):
    nk, host, sampler, _, _, student_h = setup
    batch, _, soft, _ = teacher_run
    student = nk.Model.from_host(student_h)
    ws = nk.Workspace(student, B)
    cfg = nk.TrainConfig(eta=0.05, alpha=0.5, beta=0.5, temperature=T, batch_size=B)
    loss, grads = nk.kd_loss(student, batch, soft, cfg, ws=ws)
    lv = float(loss)
    rows = sampler.rows_for(0).cpu().numpy()
    return student, ws, lv, grads, host.samples[rows], host.labels[rows]


def _grad_blocks(student, g):
    L = student.layout
    out = []
    for l in range(L.layers):
        r_, c_ = student.layer_dims[l + 1], student.layer_dims[l]
        dw = g[L.w_off[l]:L.w_off[l] + L.dims_p[l + 1] * L.dims_p[l]].reshape(L.dims_p[l + 1], L.dims_p[l])
        out.append((dw[:r_, :c_], g[L.b_off[l]:L.b_off[l] + r_]))
    return out


def test_student_kernels_on_device_operands(setup, teacher_run, student_run):
    """Level 1 for the student step: forward GEMMs, the fused KD loss/dz
    kernel, the backprop-data GEMMs and the grouped dW / db, each against
    fp64 on the bf16 operands it read."""
    _, _, _, _, _, student_h = setup
    _, _, soft, _ = teacher_run
    student, ws, lv, grads, _, y = student_run
    dims = student.layer_dims
    wq = [ref.bf16(w) for w in student_h.weights]
    acts = [None] * 3
    acts[0] = bf16_host(teacher_run[0].inputs[:, :D])
    for l in range(2):
        z = acts[l] @ wq[l].T + student_h.biases[l]
        t = np.tanh(z)
        dev = bf16_host(ws.acts[l + 1][:, :dims[l + 1]])
        worst = worst_ratio(dev, t, ulp_bf16(t) + acc(acts[l].shape[1]) * (np.abs(acts[l]) @ np.abs(wq[l]).T))
        MEASURED[f"student_fwd{l}_worst_ratio"] = worst
        assert worst <= 1.0, (l, worst)
        acts[l + 1] = dev
    # the fused logit GEMM + loss + dz kernel (edl_linear_kd_loss_fwd_bwd):
    # fp64 on the device's bf16 layer-2 activations; the logit error model
    # eps = acc(D) sum_k |a_k w_k| enters the loss and, through the softmax,
    # dz (|d softmax_i| <= 2 p_i eps)
    z = acts[2] @ wq[2].T + student_h.biases[2]
    eps = acc(acts[2].shape[1]) * (np.abs(acts[2]) @ np.abs(wq[2]).T).max(axis=1, keepdims=True)
    q = ref.topk_dense(soft.probs.cpu().numpy().astype(np.float64), soft.classes.cpu().numpy(), K)
    rows = np.arange(B)
    logp = ref.log_softmax(z)
    logp_t = ref.log_softmax(z / T)
    loss = 0.5 * float(-logp[rows, y].mean()) + 0.5 * T * T * float(-(q * logp_t).sum(axis=1).mean())
    MEASURED["student_loss_rel_fused"] = abs(lv - loss) / abs(loss)
    assert abs(lv - loss) <= 1e-5 * abs(loss)
    p1, pT = np.exp(logp), np.exp(logp_t)
    p = p1.copy()
    p[rows, y] -= 1.0
    dz = (0.5 / B) * p + (0.5 * T / B) * (pT - q)
    dz_dev = bf16_host(ws.deltas[3][:, :K])
    bound = ulp_bf16(dz) + 2 * eps * (0.5 / B * p1 + 0.5 * T / B * pT / T) + 2.0 ** -20 * (0.5 + 0.5 * T) / B
    worst = worst_ratio(dz_dev, dz, bound)
    MEASURED["student_dz_worst_ratio"] = worst
    assert worst <= 1.0
    assert (bf16_host(ws.deltas[3][:, K:]) == 0).all()
    # backprop data: delta_l = bf16((delta_{l+1} W_l) * (1 - a_l^2))
    deltas = {3: dz_dev}
    for l in (2, 1):
        gate = 1.0 - acts[l] ** 2
        d = (deltas[l + 1] @ wq[l]) * gate
        dev = bf16_host(ws.deltas[l][:, :dims[l]])
        worst = worst_ratio(dev, d, ulp_bf16(d) + acc(dims[l + 1]) * (np.abs(deltas[l + 1]) @ np.abs(wq[l])) * gate + 1e-30)
        MEASURED[f"student_bwd_data{l}_worst_ratio"] = worst
        assert worst <= 1.0, (l, worst)
        deltas[l] = dev
    # grouped dW / db
    g = grads.flat.cpu().numpy().astype(np.float64)
    for l, (dw, db) in enumerate(_grad_blocks(student, g)):
        want = deltas[l + 1].T @ acts[l]
        rw = rel(dw, want)
        rb = rel(db, deltas[l + 1].sum(axis=0))
        worst = worst_ratio(dw, want, acc(B) * (np.abs(deltas[l + 1]).T @ np.abs(acts[l])) + 1e-30)
        MEASURED[f"student_dW{l}_rel_on_device_operands"] = rw
        MEASURED[f"student_db{l}_rel_on_device_operands"] = rb
        MEASURED[f"student_dW{l}_worst_ratio"] = worst
        assert rw <= 1e-5 and rb <= 1e-5 and worst <= 1.0, (l, rw, rb, worst)


def test_student_step_vs_oracle(setup, teacher_run, student_run):
    """Level 2: kd_loss (edl/nnkit.py:254-309) over the whole B = 4096 batch vs
    the bf16-storage oracle and the fp64 reference, on the same soft labels."""
    _, _, _, _, _, student_h = setup
    _, _, soft, _ = teacher_run
    student, _, lv, grads, x, y = student_run
    sw, sb = list(student_h.weights), list(student_h.biases)
    q = ref.topk_dense(soft.probs.cpu().numpy().astype(np.float64), soft.classes.cpu().numpy(), K)
    l16, gw16, gb16 = ref.kd_loss_bf16_storage(sw, sb, x, y, q, 0.5, 0.5, T)
    l64, gw64, gb64 = ref.kd_loss(sw, sb, x, y, q, 0.5, 0.5, T)
    MEASURED["loss"] = {"device": lv, "bf16_oracle": l16, "fp64": l64}
    assert abs(lv - l16) <= 1e-3 * abs(l16)
    assert abs(lv - l64) <= 1e-3 * abs(l64)
    g = grads.flat.cpu().numpy().astype(np.float64)
    for l, (dw, db) in enumerate(_grad_blocks(student, g)):
        m = {"dW_vs_bf16_oracle": rel(dw, gw16[l]), "db_vs_bf16_oracle": rel(db, gb16[l]),
             "dW_vs_fp64": rel(dw, gw64[l]), "db_vs_fp64": rel(db, gb64[l])}
        MEASURED[f"student_layer{l}_grads"] = m
        assert m["dW_vs_bf16_oracle"] <= 2.5e-3 and m["db_vs_bf16_oracle"] <= 2.5e-3, (l, m)
        assert m["dW_vs_fp64"] <= 1e-2 and m["db_vs_fp64"] <= 1e-2, (l, m)


def test_training_reduces_loss_full_size(setup):
    from paper_2207_06667_b200.student import StudentStep
    nk, _, sampler, teacher, _, student_h = setup
    cfg = nk.TrainConfig(eta=0.05, alpha=0.5, beta=0.5, temperature=T, batch_size=B)
    eng = StudentStep(nk.Model.from_host(student_h), cfg, B, 1, max_steps=16)
    for it in range(12):
        b = sampler.batch_for(it % 2)
        soft = nk.teacher_soft_labels(teacher, b.inputs, T, k)
        eng.step(b, soft)
    eng.check_status()
    losses = eng.loss_values()
    assert np.isfinite(losses).all()
    assert np.mean(losses[-3:]) < np.mean(losses[:3])
