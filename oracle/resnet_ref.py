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
