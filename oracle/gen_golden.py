"""Generate tests/golden/*.npz by running the REAL reference (EDL-Dist,
/root/reference/pkg/src/edl) in the build container. The reference is pure
Python + numpy, so it is imported directly (read-only) — no build step.

The fixtures pin both the oracle (oracle/nnkit_ref.py, checked by
tests/test_oracle.py on CPU) and the device path (tests/test_gpu_*.py). The
GPU box never reads /root/reference; it only reads these committed files.

    PYTHONPATH=/root/reference/pkg/src python oracle/gen_golden.py
"""

from __future__ import annotations

import os
import sys
from types import SimpleNamespace

import numpy as np

REF = "/root/reference/pkg/src"
OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden")


def _flat(model):
    from edl import nnkit
    return nnkit.flatten_params(model)


def main() -> None:
    sys.path.insert(0, REF)
    from edl import allreduce, harness, nnkit
    from edl.student_node import DataSpec, ShardSampler
    os.makedirs(OUT, exist_ok=True)

    # 1. tempered softmax: the reference's own KAT input + a random sweep
    rng = np.random.default_rng(7)
    z = rng.normal(scale=5.0, size=(64, 7))
    np.savez(os.path.join(OUT, "softmax.npz"),
             kat_in=np.array([1.0, 2.0, 3.0]), kat_out=nnkit.tempered_softmax(np.array([1.0, 2, 3]), 2.0),
             z=z, t=np.array([0.5, 1.0, 3.7]),
             p=np.stack([nnkit.tempered_softmax(z, t) for t in (0.5, 1.0, 3.7)]))

    # 2. forward / kd_loss on small models, 4 (alpha, beta, T) configs of the
    #    reference FD test (tests/test_nnkit.py:148-149) + a dense and a top-k case
    cases = {}
    for ci, (alpha, beta, t) in enumerate([(1.0, 0.0, 1.0), (0.0, 1.0, 3.0), (0.7, 0.3, 2.0),
                                           (0.2, 1.5, 0.5), (0.5, 0.5, 2.0)]):
        m = nnkit.init_model([12, 24, 16, 7], seed=ci)
        r = np.random.default_rng(100 + ci)
        x = r.normal(size=(9, 12))
        y = r.integers(0, 7, size=9)
        probs = r.uniform(0.05, 1.0, size=(9, 7))
        probs /= probs.sum(axis=1, keepdims=True)
        soft = nnkit.SoftLabelBatch(probs, t) if beta > 0 else None
        cfg = nnkit.TrainConfig(eta=0.1, alpha=alpha, beta=beta, temperature=t)
        loss, g = nnkit.kd_loss(m, nnkit.Batch(x, y), soft, cfg)
        m2 = nnkit.sgd_step(m, g, 0.1)
        cases[f"c{ci}_params"] = _flat(m)
        cases[f"c{ci}_x"] = x
        cases[f"c{ci}_y"] = y
        cases[f"c{ci}_probs"] = probs
        cases[f"c{ci}_cfg"] = np.array([alpha, beta, t])
        cases[f"c{ci}_logits"] = nnkit.forward(m, x)
        cases[f"c{ci}_loss"] = np.array(loss)
        cases[f"c{ci}_grads"] = nnkit.flatten_grads(g)
        cases[f"c{ci}_after_sgd"] = _flat(m2)
    # top-k soft labels fed to the reference kd_loss through a duck-typed object
    # (the reference only reads .size/.probs/.temperature, edl/nnkit.py:265-295)
    m = nnkit.init_model([12, 24, 16, 7], seed=9)
    r = np.random.default_rng(9)
    x, y = r.normal(size=(9, 12)), r.integers(0, 7, size=9)
    teacher = nnkit.init_model([12, 32, 7], seed=10)
    p = nnkit.tempered_softmax(nnkit.forward(teacher, x), 2.0)
    for k in (3, 7):
        idx = np.argsort(-p, axis=1, kind="stable")[:, :k]
        vals = np.take_along_axis(p, idx, axis=1)
        q = np.zeros_like(p)
        np.put_along_axis(q, idx, vals / vals.sum(axis=1, keepdims=True), axis=1)
        cfg = nnkit.TrainConfig(eta=0.1, alpha=0.5, beta=0.5, temperature=2.0)
        loss, g = nnkit.kd_loss(m, nnkit.Batch(x, y), SimpleNamespace(probs=q, temperature=2.0, size=9), cfg)
        cases[f"topk{k}_idx"] = idx
        cases[f"topk{k}_vals"] = vals
        cases[f"topk{k}_loss"] = np.array(loss)
        cases[f"topk{k}_grads"] = nnkit.flatten_grads(g)
    cases["topk_params"] = _flat(m)
    cases["topk_teacher"] = _flat(teacher)
    cases["topk_x"], cases["topk_y"], cases["topk_p"] = x, y, p
    np.savez(os.path.join(OUT, "kd_loss.npz"), **cases)

    # 3. data plumbing: blobs, partition, epoch order, sampler, EDLD bytes
    d = nnkit.make_blobs(42, 100, 5, 4, 1.5)
    data = nnkit.make_blobs(0, 65, 4, 4, 1.0)
    s0 = ShardSampler(data, 2, 0, 16, seed=0)
    s1 = ShardSampler(data, 2, 1, 16, seed=0)
    small = nnkit.init_model([3, 4, 2], seed=9)
    np.savez(os.path.join(OUT, "data.npz"),
             blobs_samples=d.samples, blobs_labels=d.labels, blobs_id=np.array(d.id),
             order=nnkit.epoch_order(0, 0, 0, 100), order_e1=nnkit.epoch_order(3, 1, 2, 50),
             s0_b0=s0.batch_for(0).inputs, s0_b3=s0.batch_for(3).inputs, s1_b1=s1.batch_for(1).inputs,
             bpe=np.array(s0.batches_per_epoch),
             edld=np.frombuffer(nnkit.serialize_model(small, iteration=137), dtype=np.uint8),
             edld_params=_flat(small))

    # 4. ring all-reduce value (exact ring order), N = 1..5
    ring = {}
    for n in range(1, 6):
        vecs = [np.random.default_rng(n * 10 + r).normal(size=23) for r in range(n)]
        ring[f"n{n}_in"] = np.stack(vecs)
        ring[f"n{n}_out"] = allreduce.ring_reduce_values(vecs)
    np.savez(os.path.join(OUT, "ring.npz"), **ring)

    # 5. cfg1 (reference CPU default): pretrained teacher [16,256,256,10],
    #    student [16,64,10], T=2, alpha=beta=0.5, eta=0.05, B=32 — the
    #    harness defaults (edl/harness.py:82-88, edl/cli.py:136-147,251-252).
    spec = DataSpec(seed=0, n=2048, dim=16, classes=10, spread=1.0)
    data = spec.build()
    tcfg = nnkit.TrainConfig(eta=0.1, alpha=1.0, beta=0.0, temperature=2.0, batch_size=32, seed=0)
    teacher = nnkit.pretrain_teacher(data, tcfg, epochs=3, hidden=(256, 256))
    student0 = nnkit.init_model((16, 64, 10), 0)
    sampler = ShardSampler(data, 1, 0, 32, seed=0)
    cfg = nnkit.TrainConfig(eta=0.05, alpha=0.5, beta=0.5, temperature=2.0, batch_size=32, seed=0)
    b0 = sampler.batch_for(0)
    p0 = nnkit.tempered_softmax(nnkit.forward(teacher, b0.inputs), 2.0)
    student = student0
    losses = []
    steps = 40
    for it in range(steps):
        b = sampler.batch_for(it)
        soft = nnkit.SoftLabelBatch(nnkit.tempered_softmax(nnkit.forward(teacher, b.inputs), 2.0), 2.0)
        loss, g = nnkit.kd_loss(student, b, soft, cfg)
        student = nnkit.sgd_step(student, g, cfg.eta)
        losses.append(loss)
    holdout = nnkit.make_blobs(0, 2048 + 1000, 16, 10, 1.0)   # same centers
    hx, hy = holdout.samples[2048:], holdout.labels[2048:]
    hds = nnkit.Dataset(hx, hy)
    # N=2 data-parallel trajectory through the reference's own virtual cluster
    sc = harness.Scenario(mode=harness.EDL_DIST, students=2, teachers=2, teacher_hidden=(256, 256),
                          data=spec, max_steps=20, d_s=0.01, d_t=0.01)
    rep = harness.run_scenario(sc)
    vc_teacher = harness.build_teacher_model(sc)
    assert np.array_equal(_flat(vc_teacher), _flat(teacher)), "harness teacher differs from cfg1 teacher"
    np.savez_compressed(
        os.path.join(OUT, "cfg1.npz"),
        data_id=np.array(data.id), teacher=_flat(teacher), student0=_flat(student0),
        b0_x=b0.inputs, b0_y=b0.hard_labels, b0_probs=p0,
        student_final=_flat(student), losses=np.array(losses), steps=np.array(steps),
        holdout_top1_teacher=np.array(nnkit.evaluate(teacher, hds, 1)),
        holdout_top1_student=np.array(nnkit.evaluate(student, hds, 1)),
        holdout_top1_student0=np.array(nnkit.evaluate(student0, hds, 1)),
        vc_final=np.frombuffer(rep.final_params, dtype=np.float64), vc_steps=np.array(rep.iterations))
    print("golden fixtures written to", OUT)


if __name__ == "__main__":
    main()
