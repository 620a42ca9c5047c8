"""cfg4 (BASELINE.json configs[3]): a ResNet-style
teacher's inference on the B200, ending in the same fused softmax + top-k head
as the MLP teachers. The reference has no convolutions; parity
is against torch.nn.functional on the CPU (oracle/resnet_ref.py, tests only).

Round-1 slice: teacher inference. Each convolution is an NHWC im2col gather
(edl_im2col_nhwc; 1x1 stride-1 convolutions need none) feeding the tcgen05
GEMM, whose TMA-store epilogue adds the folded-BN bias, the block's shortcut,
and ReLU. Stem max pool, global average pool, then
edl_teacher_head_softmax_topk on the pooled features. BatchNorm is folded
into the convolution weights and bias (inference). Activations are NHWC bf16
with channels padded to a multiple of 16.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .nnkit import SoftLabels, pad


@dataclass(frozen=True)
class ResNetConfig:
    block: str = "bottleneck"          # "bottleneck" (ResNet-50 style) or "basic" (ResNet-18/34 style)
    layers: tuple = (3, 4, 6, 3)
    width: int = 64                    # stem / first-stage width
    classes: int = 1000
    image: int = 224
    in_channels: int = 3

    @property
    def expansion(self) -> int:
        return 4 if self.block == "bottleneck" else 1


@dataclass
class HostConv:
    """Folded conv + BN: w fp32 [cout][cin][k][k], b fp32 [cout]."""
    w: np.ndarray
    b: np.ndarray
    stride: int
    pad: int
    relu: bool = True


@dataclass
class HostBlock:
    convs: list
    shortcut: HostConv | None


@dataclass
class HostResNet:
    cfg: ResNetConfig
    stem: HostConv
    blocks: list = field(default_factory=list)
    fc_w: np.ndarray | None = None     # [classes][features]
    fc_b: np.ndarray | None = None


def _conv(rng, cin, cout, k, stride, relu=True, gain=1.0):
    # He-normal weights with a random BN fold (gamma / sqrt(var + eps), beta - mean * that)
    w = rng.normal(0.0, np.sqrt(2.0 / (cin * k * k)), size=(cout, cin, k, k)) * gain
    scale = rng.uniform(0.8, 1.2, size=cout)
    shift = rng.normal(0.0, 0.05, size=cout)
    return HostConv((w * scale[:, None, None, None]).astype(np.float32), shift.astype(np.float32), stride,
                    k // 2, relu)


def init_resnet(cfg: ResNetConfig, seed: int) -> HostResNet:
    rng = np.random.default_rng(seed)
    net = HostResNet(cfg, _conv(rng, cfg.in_channels, cfg.width, 7, 2))
    net.stem.pad = 3
    cin = cfg.width
    for stage, n in enumerate(cfg.layers):
        mid = cfg.width * (2 ** stage)
        cout = mid * cfg.expansion
        for i in range(n):
            stride = 2 if (i == 0 and stage > 0) else 1
            if cfg.block == "bottleneck":
                convs = [_conv(rng, cin, mid, 1, 1), _conv(rng, mid, mid, 3, stride),
                         _conv(rng, mid, cout, 1, 1, relu=True, gain=0.5)]
            else:
                convs = [_conv(rng, cin, mid, 3, stride), _conv(rng, mid, cout, 3, 1, relu=True, gain=0.5)]
            shortcut = None
            if stride != 1 or cin != cout:
                shortcut = _conv(rng, cin, cout, 1, stride, relu=False)
                shortcut.pad = 0
            net.blocks.append(HostBlock(convs, shortcut))
            cin = cout
    net.fc_w = (rng.normal(0.0, np.sqrt(1.0 / cin), size=(cfg.classes, cin))).astype(np.float32)
    net.fc_b = np.zeros(cfg.classes, dtype=np.float32)
    return net


class _DevConv:
    """Device form: W bf16 [cout_p][kdim] in im2col (r, s, c) order, b fp32 [cout_p].
    Inputs with fewer than 8 channels (the RGB stem) use the packed im2col:
    K = k*k*cin padded to 16, instead of k*k*pad(cin)."""

    def __init__(self, c: HostConv, dev):
        cout, cin, k, _ = c.w.shape
        self.k, self.stride, self.pad, self.relu = k, c.stride, c.pad, c.relu
        self.cin, self.cin_p, self.cout_p = cin, pad(cin), pad(cout)
        self.packed = cin < 8
        wt = c.w.transpose(0, 2, 3, 1)                      # [cout][k][k][cin]
        if self.packed:
            self._kdim = pad(k * k * cin)
            w = np.zeros((self.cout_p, self._kdim), dtype=np.float32)
            w[:cout, :k * k * cin] = wt.reshape(cout, -1)
        else:
            self._kdim = k * k * self.cin_p
            w = np.zeros((self.cout_p, k, k, self.cin_p), dtype=np.float32)
            w[:cout, :, :, :cin] = wt
        self.w = torch.from_numpy(w.reshape(self.cout_p, -1)).to(dev).to(torch.bfloat16)
        b = np.zeros(self.cout_p, dtype=np.float32)
        b[:cout] = c.b
        self.b = torch.from_numpy(b).to(dev)

    def out_hw(self, h, w):
        return (h + 2 * self.pad - self.k) // self.stride + 1, (w + 2 * self.pad - self.k) // self.stride + 1

    @property
    def kdim(self):
        return self._kdim


class ResNetTeacher:
    """Device ResNet-style teacher for a fixed batch size (buffers allocated
    once; the inference path never allocates)."""

    def __init__(self, host: HostResNet, device=None, batch_size: int = 64):
        self.cfg = host.cfg
        self.device = dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.B = B = batch_size
        self.stem = _DevConv(host.stem, dev)
        self.blocks = [([_DevConv(c, dev) for c in blk.convs], _DevConv(blk.shortcut, dev) if blk.shortcut else None)
                       for blk in host.blocks]
        feat = host.fc_w.shape[1]
        self.feat_p = pad(feat)
        fc = np.zeros((host.fc_w.shape[0], self.feat_p), dtype=np.float32)
        fc[:, :feat] = host.fc_w
        self.fc_w = torch.from_numpy(fc).to(dev).to(torch.bfloat16)
        self.fc_b = torch.from_numpy(host.fc_b.astype(np.float32)).to(dev)
        self.classes = host.fc_w.shape[0]
        # shapes + buffers
        H = W = self.cfg.image
        self.in_c = pad(self.cfg.in_channels)
        h, w = self.stem.out_hw(H, W)
        col = B * h * w * self.stem.kdim
        self.x0 = torch.empty(B, h, w, self.stem.cout_p, dtype=torch.bfloat16, device=dev)
        ph, pw = (h + 2 - 3) // 2 + 1, (w + 2 - 3) // 2 + 1
        self.pool_hw = (h, w, ph, pw)
        cur = torch.empty(B, ph, pw, self.stem.cout_p, dtype=torch.bfloat16, device=dev)
        self.x1 = cur
        h, w = ph, pw
        self.buffers = []
        for convs, sc in self.blocks:
            bh, bw = h, w
            outs = []
            for c in convs:
                oh, ow = c.out_hw(bh, bw)
                col = max(col, B * oh * ow * c.kdim if (c.k > 1 or c.stride > 1) else 0)
                outs.append(torch.empty(B, oh, ow, c.cout_p, dtype=torch.bfloat16, device=dev))
                bh, bw = oh, ow
            sc_out = None
            if sc is not None:
                oh, ow = sc.out_hw(h, w)
                col = max(col, B * oh * ow * sc.kdim if sc.stride > 1 else 0)
                sc_out = torch.empty(B, oh, ow, sc.cout_p, dtype=torch.bfloat16, device=dev)
            self.buffers.append((outs, sc_out, h, w))
            h, w = bh, bw
        self.final_hw = (h, w)
        self.col = torch.empty(max(col, 16), dtype=torch.bfloat16, device=dev)
        self.features_buf = torch.empty(B, self.feat_p, dtype=torch.bfloat16, device=dev)

    # one convolution: x NHWC [B][h][w][cin_p] -> out NHWC; residual (bf16, out's shape) or None
    def _conv(self, c: _DevConv, x, h, w, out, residual, s):
        oh, ow = c.out_hw(h, w)
        M = self.B * oh * ow
        if c.k == 1 and c.stride == 1:
            a, lda = x, c.cin_p                            # NHWC already is the GEMM's A
        else:
            a, lda = self.col, c.kdim
            _lib.call("edl_im2col_nhwc", x.data_ptr(), self.B, h, w, c.cin_p, c.cin if c.packed else c.cin_p,
                      c.k, c.k, c.stride, c.pad, self.col.data_ptr(), lda, s)
        if residual is not None:
            _lib.call("edl_linear_fwd_residual", a.data_ptr(), lda, c.w.data_ptr(), c.kdim, c.b.data_ptr(),
                      residual.data_ptr(), c.cout_p, out.data_ptr(), c.cout_p, M, c.cout_p, c.kdim, s)
        else:
            act = _lib.EDL_ACT_RELU if c.relu else _lib.EDL_ACT_IDENT
            _lib.call("edl_linear_fwd", a.data_ptr(), lda, c.w.data_ptr(), c.kdim, c.b.data_ptr(), out.data_ptr(),
                      c.cout_p, M, c.cout_p, c.kdim, act, s)
        return oh, ow

    def features(self, x: torch.Tensor, stream=None) -> torch.Tensor:
        """x: NHWC bf16 [B][image][image][pad(in_channels)] -> pooled features bf16 [B][feat_p]."""
        if tuple(x.shape) != (self.B, self.cfg.image, self.cfg.image, self.in_c) or x.dtype != torch.bfloat16:
            raise ValueError(f"expected NHWC bf16 {(self.B, self.cfg.image, self.cfg.image, self.in_c)}")
        s = (stream or torch.cuda.current_stream()).cuda_stream
        H = W = self.cfg.image
        self._conv(self.stem, x, H, W, self.x0, None, s)
        h, w, ph, pw = self.pool_hw
        _lib.call("edl_maxpool_nhwc", self.x0.data_ptr(), self.B, h, w, self.stem.cout_p, 3, 2, 1,
                  self.x1.data_ptr(), s)
        cur = self.x1
        for (convs, sc), (outs, sc_out, bh, bw) in zip(self.blocks, self.buffers):
            shortcut = cur
            if sc is not None:
                self._conv(sc, cur, bh, bw, sc_out, None, s)
                shortcut = sc_out
            h, w = bh, bw
            y = cur
            for i, (c, out) in enumerate(zip(convs, outs)):
                last = i == len(convs) - 1
                h, w = self._conv(c, y, h, w, out, shortcut if last else None, s)
                y = out
            cur = y
        fh, fw = self.final_hw
        _lib.call("edl_avgpool_nhwc", cur.data_ptr(), self.B, fh * fw, cur.shape[-1], self.features_buf.data_ptr(),
                  self.feat_p, s)
        return self.features_buf

    def soft_labels(self, x: torch.Tensor, temperature: float, k: int, out: SoftLabels | None = None,
                    stream=None) -> SoftLabels:
        """Top-k soft labels of softmax(logits / T), the fused head as for the MLP teachers."""
        f = self.features(x, stream)
        if out is None:
            out = SoftLabels(torch.empty(self.B, k, device=self.device),
                             torch.empty(self.B, k, dtype=torch.int32, device=self.device), float(temperature))
        s = (stream or torch.cuda.current_stream()).cuda_stream
        _lib.call("edl_teacher_head_softmax_topk", f.data_ptr(), f.stride(0), self.fc_w.data_ptr(), self.feat_p,
                  self.fc_b.data_ptr(), self.B, self.classes, self.feat_p, float(temperature), int(k),
                  out.probs.data_ptr(), out.classes.data_ptr(), s)
        return out

    def flops_per_sample(self) -> float:
        """Algorithmic GEMM FLOPs per image (padded channels included)."""
        H = W = self.cfg.image
        total = 0.0
        h, w = self.stem.out_hw(H, W)
        total += 2.0 * h * w * self.stem.cout_p * self.stem.kdim
        h, w = self.pool_hw[2], self.pool_hw[3]
        for (convs, sc), (_, _, bh, bw) in zip(self.blocks, self.buffers):
            if sc is not None:
                oh, ow = sc.out_hw(bh, bw)
                total += 2.0 * oh * ow * sc.cout_p * sc.kdim
            h, w = bh, bw
            for c in convs:
                oh, ow = c.out_hw(h, w)
                total += 2.0 * oh * ow * c.cout_p * c.kdim
                h, w = oh, ow
        total += 2.0 * self.classes * self.feat_p
        return total


def to_nhwc(images: np.ndarray, device) -> torch.Tensor:
    """NCHW float images -> NHWC bf16 with channels padded to 16."""
    n, c, h, w = images.shape
    x = torch.zeros(n, h, w, pad(c), dtype=torch.bfloat16, device=device)
    x[..., :c] = torch.from_numpy(np.ascontiguousarray(images.transpose(0, 2, 3, 1), dtype=np.float32)).to(device).to(torch.bfloat16)
    return x
