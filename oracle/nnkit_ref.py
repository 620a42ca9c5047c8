"""CPU ORACLE — test infrastructure only.

A float64 numpy restatement of the reference's hot-path arithmetic
(EDL-Dist, pkg/src/edl). Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference leg may import it, and only as the checker or
the timed CPU baseline — never as the product path (the product is
libedl_b200.so via paper_2207_06667_b200).

Parity is PINNED: tests/test_oracle.py checks every function here against
golden vectors produced by running the reference itself in the build
container (oracle/gen_golden.py -> tests/golden/*.npz) plus the reference's
own known-answer tests (tests/test_nnkit.py:40-46 softmax KAT etc.).

The reference's arithmetic lives in third-party numpy (pkg/pyproject.toml:10
pins `numpy>=1.24`; golden vectors were generated with numpy 2.3.5 /
OpenBLAS 0.3.30). Every function cites the reference lines it restates.
"""

from __future__ import annotations

import numpy as np


# ---------------------------------------------------------------- math core
def tempered_softmax(logits, temperature):
    """edl/nnkit.py:193-208."""
    if not np.isfinite(temperature) or temperature <= 0:
        raise ValueError(f"temperature must be a positive finite real, got {temperature}")
    z = np.asarray(logits, dtype=np.float64)
    if not np.isfinite(z).all():
        raise ValueError("logits must be finite")
    scaled = z / temperature
    shifted = scaled - scaled.max(axis=-1, keepdims=True)
    e = np.exp(shifted)
    return e / e.sum(axis=-1, keepdims=True)


def init_model(layer_dims, seed):
    """edl/nnkit.py:211-220 -> (weights, biases) lists."""
    rng = np.random.Generator(np.random.PCG64(np.random.SeedSequence(seed)))
    dims = tuple(int(d) for d in layer_dims)
    ws, bs = [], []
    for l in range(len(dims) - 1):
        a = np.sqrt(6.0 / (dims[l] + dims[l + 1]))
        ws.append(rng.uniform(-a, a, size=(dims[l + 1], dims[l])))
        bs.append(np.zeros(dims[l + 1]))
    return ws, bs


def forward_activations(weights, biases, x):
    """edl/nnkit.py:237-246 (forward(), :223-234, is its last element)."""
    acts = [np.asarray(x, dtype=np.float64)]
    h = acts[0]
    last = len(weights) - 1
    for l, (w, b) in enumerate(zip(weights, biases)):
        z = h @ w.T + b
        h = z if l == last else np.tanh(z)
        acts.append(h)
    return acts


def forward(weights, biases, x):
    return forward_activations(weights, biases, x)[-1]


def log_softmax(scaled):
    """edl/nnkit.py:249-251."""
    shifted = scaled - scaled.max(axis=1, keepdims=True)
    return shifted - np.log(np.exp(shifted).sum(axis=1, keepdims=True))


def kd_loss(weights, biases, x, labels, soft_probs, alpha, beta, temperature):
    """edl/nnkit.py:254-309. soft_probs is a dense B x K matrix (or None when
    beta == 0); top-k soft labels are passed densified (see topk_dense)."""
    b = x.shape[0]
    acts = forward_activations(weights, biases, x)
    logits = acts[-1]
    rows = np.arange(b)
    loss = 0.0
    dlogits = np.zeros_like(logits)
    if alpha > 0:
        logp = log_softmax(logits)
        loss += alpha * float(-logp[rows, labels].mean())
        p = np.exp(logp)
        p[rows, labels] -= 1.0
        dlogits += (alpha / b) * p
    if beta > 0:
        t = temperature
        logp_t = log_softmax(logits / t)
        loss += beta * t * t * float(-(soft_probs * logp_t).sum(axis=1).mean())
        dlogits += (beta * t / b) * (np.exp(logp_t) - soft_probs)
    if not np.isfinite(loss):
        raise ArithmeticError(f"loss is not finite: {loss}")
    gw = [None] * len(weights)
    gb = [None] * len(biases)
    delta = dlogits
    for l in range(len(weights) - 1, -1, -1):
        gw[l] = delta.T @ acts[l]
        gb[l] = delta.sum(axis=0)
        if l > 0:
            delta = (delta @ weights[l]) * (1.0 - acts[l] ** 2)
    return loss, gw, gb


def sgd_step(weights, biases, gw, gb, eta):
    """edl/nnkit.py:312-322."""
    return ([w - eta * g for w, g in zip(weights, gw)],
            [b - eta * g for b, g in zip(biases, gb)])


def evaluate(weights, biases, samples, labels, k=1):
    """edl/nnkit.py:325-335 (stable argsort: ties to the lower class)."""
    logits = forward(weights, biases, samples)
    order = np.argsort(-logits, axis=1, kind="stable")
    return float((order[:, :k] == labels[:, None]).any(axis=1).mean())


def flatten(ws, bs):
    """edl/nnkit.py:342-347 order: W0, b0, W1, b1, ..."""
    parts = []
    for w, b in zip(ws, bs):
        parts.append(w.ravel())
        parts.append(b)
    return np.concatenate(parts)


def unflatten(flat, dims):
    """edl/nnkit.py:350-360."""
    ws, bs, off = [], [], 0
    for l in range(len(dims) - 1):
        n = dims[l + 1] * dims[l]
        ws.append(flat[off:off + n].reshape(dims[l + 1], dims[l]))
        off += n
        bs.append(flat[off:off + dims[l + 1]])
        off += dims[l + 1]
    return ws, bs


# ---------------------------------------------------------------- top-k soft labels
def topk(probs, k):
    """Top-k of a dense distribution with the reference tie rule
    (np.argsort(-p, kind="stable"), edl/nnkit.py:333): probability desc,
    lower class first. Returns (vals, idx) of the RAW probabilities."""
    idx = np.argsort(-probs, axis=1, kind="stable")[:, :k]
    return np.take_along_axis(probs, idx, axis=1), idx


def topk_dense(vals, idx, num_classes):
    """Renormalised top-k densified with zeros: the soft-label
    matrix the reference kd_loss consumes; k = K reproduces the dense case."""
    q = np.zeros((vals.shape[0], num_classes))
    np.put_along_axis(q, np.asarray(idx, dtype=np.int64), vals / vals.sum(axis=1, keepdims=True), axis=1)
    return q


def teacher_soft(weights, biases, x, temperature, k):
    """soft_label_reply's math (edl/teacher_node.py:54) + top-k."""
    p = tempered_softmax(forward(weights, biases, x), temperature)
    return topk(p, k)


# ---------------------------------------------------------------- data
def make_blobs(seed, n_samples, dim, classes, spread):
    """edl/nnkit.py:371-388 -> (samples, labels)."""
    rng = np.random.Generator(np.random.PCG64(np.random.SeedSequence([seed, 0xB10B5])))
    centers = rng.normal(size=(classes, dim))
    centers *= 3.0 / np.linalg.norm(centers, axis=1, keepdims=True)
    labels = np.arange(n_samples, dtype=np.int64) % classes
    samples = centers[labels] + rng.normal(scale=spread, size=(n_samples, dim))
    return samples, labels


def partition_bounds(n, world_size, rank):
    """edl/nnkit.py:391-399."""
    return (n * rank) // world_size, (n * (rank + 1)) // world_size


def epoch_order(seed, epoch, rank, n):
    """edl/nnkit.py:402-405."""
    ss = np.random.SeedSequence([seed, epoch, rank, 0x0A7A])
    return np.random.Generator(np.random.PCG64(ss)).permutation(n)


def batch_rows(seed, rank, shard_size, batch_size, batches_per_epoch, iteration):
    """ShardSampler.batch_for row selection (edl/student_node.py:145-151)."""
    epoch, i = divmod(iteration, batches_per_epoch)
    order = epoch_order(seed, epoch, rank, shard_size)
    return order[i * batch_size:(i + 1) * batch_size]


def pretrain_teacher(samples, labels, eta, batch_size, seed, epochs, hidden):
    """edl/nnkit.py:408-426 (hard-label SGD)."""
    classes = int(labels.max()) + 1
    ws, bs = init_model((samples.shape[1], *hidden, classes), seed)
    bpe = samples.shape[0] // batch_size
    for epoch in range(epochs):
        order = epoch_order(seed, epoch, 0, samples.shape[0])
        for i in range(bpe):
            idx = order[i * batch_size:(i + 1) * batch_size]
            _, gw, gb = kd_loss(ws, bs, samples[idx], labels[idx], None, 1.0, 0.0, 1.0)
            ws, bs = sgd_step(ws, bs, gw, gb, eta)
    return ws, bs


# ---------------------------------------------------------------- collective
def chunk_bounds(length, n):
    """edl/allreduce.py:69-74."""
    base = length // n
    bounds = [(i * base, (i + 1) * base) for i in range(n - 1)]
    bounds.append(((n - 1) * base, length))
    return bounds


def ring_reduce_values(vectors):
    """edl/allreduce.py:123-144: the ring's exact summation order, then mean."""
    n = len(vectors)
    vecs = [np.ascontiguousarray(v, dtype=np.float64) for v in vectors]
    if n == 1:
        return vecs[0].copy()
    out = np.empty(vecs[0].size)
    for c, (lo, hi) in enumerate(chunk_bounds(vecs[0].size, n)):
        seg = vecs[c][lo:hi].copy()
        for k in range(1, n):
            seg = seg + vecs[(c + k) % n][lo:hi]
        out[lo:hi] = seg
    out /= n
    return out


def dp_distill_trajectory(student, teacher, samples, labels, students, batch_size, seed, steps,
                          alpha, beta, temperature, eta, k=None):
    """N-student data-parallel distillation, the VirtualCluster._commit loop
    (edl/harness.py:411-433): per student kd_loss on its shard's batch with
    the teacher's (top-k) soft labels, ring mean of the flat grads, SGD.
    Returns (final (ws, bs), per-step rank-0 losses)."""
    ws, bs = student
    tw, tb = teacher
    dims = tuple([ws[0].shape[1]] + [w.shape[0] for w in ws])
    n = samples.shape[0]
    bpe = (n // students) // batch_size
    losses = []
    for it in range(steps):
        flats = []
        for r in range(students):
            lo, hi = partition_bounds(n, students, r)
            rows = batch_rows(seed, r, hi - lo, batch_size, bpe, it)
            x, y = samples[lo:hi][rows], labels[lo:hi][rows]
            q = None
            if beta > 0:
                p = tempered_softmax(forward(tw, tb, x), temperature)
                q = p if k is None else topk_dense(*topk(p, k), p.shape[1])
            loss, gw, gb = kd_loss(ws, bs, x, y, q, alpha, beta, temperature)
            if r == 0:
                losses.append(loss)
            flats.append(flatten(gw, gb))
        avg = ring_reduce_values(flats)
        gw, gb = unflatten(avg, dims)
        ws, bs = sgd_step(ws, bs, gw, gb, eta)
    return (ws, bs), losses


# ---------------------------------------------------------------- bf16-storage emulation
def bf16(a):
    """Round-to-nearest-even to bfloat16, returned as float64 (emulates the
    device's bf16 storage points; arithmetic stays fp64)."""
    a = np.ascontiguousarray(a, dtype=np.float32)
    u = a.view(np.uint32).astype(np.uint64)
    r = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16
    return r.astype(np.uint32).view(np.float32).astype(np.float64)


def kd_loss_bf16_storage(weights, biases, x, labels, soft_probs, alpha, beta, temperature):
    """kd_loss (edl/nnkit.py:254-309) with the device path's storage points
    rounded to bf16: inputs, weight copies, hidden activations, dlogits and
    hidden deltas. Isolates the kernels' accumulation error in the parity
    tests."""
    wq = [bf16(w) for w in weights]
    b = x.shape[0]
    acts = [bf16(x)]
    h = acts[0]
    last = len(weights) - 1
    for l, (w, bb) in enumerate(zip(wq, biases)):
        z = h @ w.T + bb
        h = z if l == last else bf16(np.tanh(z))
        acts.append(h)
    logits = acts[-1]
    rows = np.arange(b)
    loss = 0.0
    dlogits = np.zeros_like(logits)
    if alpha > 0:
        logp = log_softmax(logits)
        loss += alpha * float(-logp[rows, labels].mean())
        p = np.exp(logp)
        p[rows, labels] -= 1.0
        dlogits += (alpha / b) * p
    if beta > 0:
        t = temperature
        logp_t = log_softmax(logits / t)
        loss += beta * t * t * float(-(soft_probs * logp_t).sum(axis=1).mean())
        dlogits += (beta * t / b) * (np.exp(logp_t) - soft_probs)
    gw = [None] * len(weights)
    gb = [None] * len(biases)
    delta = bf16(dlogits)
    for l in range(len(weights) - 1, -1, -1):
        gw[l] = delta.T @ acts[l]
        gb[l] = delta.sum(axis=0)
        if l > 0:
            delta = bf16((delta @ wq[l]) * (1.0 - acts[l] ** 2))
    return loss, gw, gb


def forward_bf16_storage(weights, biases, x):
    """forward() with bf16 inputs / weights / hidden activations (device storage)."""
    h = bf16(x)
    last = len(weights) - 1
    for l, (w, b) in enumerate(zip(weights, biases)):
        z = h @ bf16(w).T + b
        h = z if l == last else bf16(np.tanh(z))
    return h
