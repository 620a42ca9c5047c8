"""TEST INFRASTRUCTURE ONLY (tests/ may import this; the product never does).

cfg4 stand-in oracle: the reference has no convolutions, so the
ResNet-style teacher's parity is against torch.nn.functional on the CPU, as
SURVEY §8(f) rank 4 specifies. PARITY UNPINNED BY THE REFERENCE: there is no
reference output to pin this to. It emulates the device's storage points
(bf16 weights, activations rounded to bf16 after every layer, fp32 math) so
tests isolate accumulation-order error from storage rounding.
"""

from __future__ import annotations

import numpy as np
import torch
import torch.nn.functional as F


def _bf(t: torch.Tensor) -> torch.Tensor:
    return t.to(torch.bfloat16).to(torch.float32)


def _conv(x, c, residual=None):
    w = _bf(torch.from_numpy(c.w))
    y = F.conv2d(x, w, torch.from_numpy(c.b), stride=c.stride, padding=c.pad)
    if residual is not None:
        y = y + residual
    if c.relu or residual is not None:
        y = torch.relu(y)
    return _bf(y)


def features(net, images: np.ndarray) -> torch.Tensor:
    """NCHW images -> pooled features [N][C] (bf16-rounded, fp32 tensor)."""
    x = _bf(torch.from_numpy(np.asarray(images, dtype=np.float32)))
    x = _conv(x, net.stem)
    x = _bf(F.max_pool2d(x, 3, 2, 1))
    for blk in net.blocks:
        shortcut = _conv(x, blk.shortcut) if blk.shortcut is not None else x
        y = x
        for i, c in enumerate(blk.convs):
            y = _conv(y, c, shortcut if i == len(blk.convs) - 1 else None)
        x = y
    return _bf(x.mean(dim=(2, 3)))


def logits(net, images: np.ndarray) -> torch.Tensor:
    f = features(net, images)
    return f @ _bf(torch.from_numpy(net.fc_w)).T + torch.from_numpy(net.fc_b)


def student_loss_and_grads(net, images: np.ndarray, labels: np.ndarray, q_dense: np.ndarray, alpha: float,
                           beta: float, T: float):
    """BN-free ResNet-18-style student (resnet.init_student_resnet) trained
    with the reference's KD loss (edl/nnkit.py:283-295: alpha * CE(z, y) +
    beta * T^2 * CE(q, softmax(z / T)), batch mean) by torch autograd on the
    CPU, from bf16-rounded weights (the device's operands). Forward values
    are rounded to bf16 where the device stores them (conv / shortcut
    outputs, pooled features) by straight-through rounding, which changes
    values but not the gradient formulas; the device's bf16 deltas remain
    the only storage difference. Returns (loss,
    {"stem": (dW, db), "blocks": [((dW1, db1), (dW2, db2), sc or None)],
    "fc": (dW, db)}) in torch layout (fp32)."""
    def leaf(a):
        return _bf(torch.from_numpy(np.asarray(a, dtype=np.float32))).requires_grad_(True)

    def st(t):
        return t + (_bf(t.detach()) - t.detach())

    def conv(x, c, p, residual=None):
        y = F.conv2d(x, p[0], p[1], stride=c.stride, padding=c.pad)
        if residual is not None:
            y = y + residual
        return st(torch.relu(y) if (c.relu or residual is not None) else y)

    P = {"stem": (leaf(net.stem.w), torch.from_numpy(net.stem.b).clone().requires_grad_(True))}
    blocks = []
    for blk in net.blocks:
        p1 = (leaf(blk.convs[0].w), torch.from_numpy(blk.convs[0].b).clone().requires_grad_(True))
        p2 = (leaf(blk.convs[1].w), torch.from_numpy(blk.convs[1].b).clone().requires_grad_(True))
        ps = None
        if blk.shortcut is not None:
            ps = (leaf(blk.shortcut.w), torch.from_numpy(blk.shortcut.b).clone().requires_grad_(True))
        blocks.append((p1, p2, ps))
    fc = (leaf(net.fc_w), torch.from_numpy(net.fc_b).clone().requires_grad_(True))
    x = _bf(torch.from_numpy(np.asarray(images, dtype=np.float32)))
    x = conv(x, net.stem, P["stem"])
    x = F.max_pool2d(x, 3, 2, 1)
    for blk, (p1, p2, ps) in zip(net.blocks, blocks):
        sc = conv(x, blk.shortcut, ps) if ps is not None else x
        h = conv(x, blk.convs[0], p1)
        x = conv(h, blk.convs[1], p2, sc)
    f = st(x.mean(dim=(2, 3)))
    z = f @ fc[0].T + fc[1]
    y = torch.from_numpy(np.asarray(labels, dtype=np.int64))
    hard = -torch.log_softmax(z, dim=1)[torch.arange(z.shape[0]), y]
    q = torch.from_numpy(np.asarray(q_dense, dtype=np.float32))
    soft = -(q * torch.log_softmax(z / T, dim=1)).sum(dim=1) * T * T
    loss = (alpha * hard + beta * soft).mean()
    loss.backward()
    g = lambda p: (p[0].grad.detach(), p[1].grad.detach())  # noqa: E731
    return float(loss.detach()), {"stem": g(P["stem"]),
                         "blocks": [(g(p1), g(p2), g(ps) if ps is not None else None) for p1, p2, ps in blocks],
                         "fc": g(fc)}


class _RoundGrad(torch.autograd.Function):
    """Identity forward; the incoming gradient rounded to bf16 (the device
    stores every activation gradient in bf16)."""

    @staticmethod
    def forward(ctx, t):
        return t.view_as(t)

    @staticmethod
    def backward(ctx, g):
        return _bf(g)


def student_bn_loss_and_grads(net, images: np.ndarray, labels: np.ndarray, q_dense: np.ndarray, alpha: float,
                              beta: float, T: float, eps: float = 1e-5, round_grads: bool = False,
                              forced: dict | None = None):
    """The BatchNorm ResNet-18-style student (resnet.init_student_resnet with
    bn=True): every conv (no bias) followed by training-mode BatchNorm (batch
    statistics, biased variance, as nn.BatchNorm2d in training), ReLU after
    BN except on the shortcut projection, the residual added before the
    block's last ReLU; the reference's KD loss (edl/nnkit.py:283-295). torch
    autograd on the CPU from bf16-rounded conv / fc weights, with forward
    values rounded where the device stores bf16 (conv outputs z, BN outputs,
    pooled features) by straight-through rounding; round_grads=True also
    rounds the gradients at those points to bf16, as the device stores them.
    forced: the device's own forward values at those points (NCHW float
    tensors keyed "stem_z", "stem_y", "b{i}_z1", "b{i}_h1", "b{i}_z2",
    "b{i}_y", "b{i}_zsc", "b{i}_sc", "features"), substituted straight-through
    so autograd differentiates the device's forward: the gradient then
    differs from the device's only by the backward's own arithmetic (at
    initialisation this BN net's gradient moves ~24% for a 1e-3 relative
    perturbation of the images, so an independent forward cannot pin it).
    Returns (loss, {"stem": (dW, dgamma, dbeta), "blocks": [(c1, c2, sc or
    None)], "fc": (dW, db)})."""
    def leaf(a):
        return _bf(torch.from_numpy(np.asarray(a, dtype=np.float32))).requires_grad_(True)

    def vec(a):
        return torch.from_numpy(np.asarray(a, dtype=np.float32)).clone().requires_grad_(True)

    def st(t, key=None):
        v = forced[key] if (forced is not None and key in forced) else _bf(t.detach())
        t = t + (v - t.detach())
        return _RoundGrad.apply(t) if round_grads else t

    def conv_bn(x, c, p, relu, residual=None, zkey=None, ykey=None):
        z = st(F.conv2d(x, p[0], None, stride=c.stride, padding=c.pad), zkey)
        y = F.batch_norm(z, None, None, p[1], p[2], training=True, eps=eps)
        if residual is not None:
            y = y + residual
        return st(torch.relu(y) if relu else y, ykey)

    def params(c):
        return (leaf(c.w), vec(c.gamma), vec(c.b))

    P = {"stem": params(net.stem)}
    blocks = [(params(b.convs[0]), params(b.convs[1]), params(b.shortcut) if b.shortcut is not None else None)
              for b in net.blocks]
    fc = (leaf(net.fc_w), torch.from_numpy(net.fc_b).clone().requires_grad_(True))
    x = _bf(torch.from_numpy(np.asarray(images, dtype=np.float32)))
    x = conv_bn(x, net.stem, P["stem"], True, zkey="stem_z", ykey="stem_y")
    x = F.max_pool2d(x, 3, 2, 1)
    for bi, (blk, (p1, p2, ps)) in enumerate(zip(net.blocks, blocks)):
        sc = conv_bn(x, blk.shortcut, ps, False, zkey=f"b{bi}_zsc", ykey=f"b{bi}_sc") if ps is not None else x
        h = conv_bn(x, blk.convs[0], p1, True, zkey=f"b{bi}_z1", ykey=f"b{bi}_h1")
        x = conv_bn(h, blk.convs[1], p2, True, sc, zkey=f"b{bi}_z2", ykey=f"b{bi}_y")
    f = st(x.mean(dim=(2, 3)), "features")
    z = f @ fc[0].T + fc[1]
    y = torch.from_numpy(np.asarray(labels, dtype=np.int64))
    hard = -torch.log_softmax(z, dim=1)[torch.arange(z.shape[0]), y]
    q = torch.from_numpy(np.asarray(q_dense, dtype=np.float32))
    soft = -(q * torch.log_softmax(z / T, dim=1)).sum(dim=1) * T * T
    loss = (alpha * hard + beta * soft).mean()
    loss.backward()
    g3 = lambda p: tuple(t.grad.detach() for t in p)  # noqa: E731
    return float(loss.detach()), {"stem": g3(P["stem"]),
                                  "blocks": [(g3(p1), g3(p2), g3(ps) if ps is not None else None)
                                             for p1, p2, ps in blocks],
                                  "fc": g3(fc)}
