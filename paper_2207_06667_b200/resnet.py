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
from .nnkit import SoftLabels, img_pad, pad


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
    """Folded conv + BN: w fp32 [cout][cin][k][k], b fp32 [cout]. A student
    conv followed by training-mode BatchNorm carries gamma (b is then BN's
    beta and the conv itself has no bias)."""
    w: np.ndarray
    b: np.ndarray
    stride: int
    pad: int
    relu: bool = True
    gamma: np.ndarray | None = None


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
    bn: bool = False                   # every conv followed by training-mode BatchNorm (student)


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
        self.cin, self.cin_p, self.cout_p = cin, img_pad(cin), pad(cout)
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
    def implicit(self) -> bool:
        """Implicit GEMM (edl_conv_fwd_nhwc: TMA im2col loads, no column
        matrix) for every windowed conv on >= 64-channel inputs; the packed
        RGB stem keeps its explicit im2col, 1x1 / stride-1 convs are plain GEMMs."""
        return not self.packed and self.cin_p % 64 == 0 and not (self.k == 1 and self.stride == 1)

    def fwd_implicit(self, x, n, h, w, out, residual, s):
        act = _lib.EDL_ACT_RELU if (self.relu or residual is not None) else _lib.EDL_ACT_IDENT
        _lib.call("edl_conv_fwd_nhwc", x.data_ptr(), n, h, w, self.cin_p, self.w.data_ptr(), self.kdim,
                  self.b.data_ptr(), self.cout_p, self.k, self.k, self.stride, self.pad,
                  None if residual is None else residual.data_ptr(), self.cout_p, out.data_ptr(), self.cout_p, act, s)

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
        self.in_c = img_pad(self.cfg.in_channels)
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
                col = max(col, B * oh * ow * c.kdim if ((c.k > 1 or c.stride > 1) and not c.implicit) else 0)
                outs.append(torch.empty(B, oh, ow, c.cout_p, dtype=torch.bfloat16, device=dev))
                bh, bw = oh, ow
            sc_out = None
            if sc is not None:
                oh, ow = sc.out_hw(h, w)
                col = max(col, B * oh * ow * sc.kdim if (sc.stride > 1 and not sc.implicit) else 0)
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
        if c.implicit:
            c.fwd_implicit(x, self.B, h, w, out, residual, s)
            return oh, ow
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
        """x: NHWC bf16 [B][image][image][img_pad(in_channels)] -> pooled features bf16 [B][feat_p]."""
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
    """NCHW float images -> NHWC bf16 with channels padded to img_pad(c)
    (8 for RGB, the packed stems' input pitch)."""
    n, c, h, w = images.shape
    x = torch.zeros(n, h, w, img_pad(c), dtype=torch.bfloat16, device=device)
    x[..., :c] = torch.from_numpy(np.ascontiguousarray(images.transpose(0, 2, 3, 1), dtype=np.float32)).to(device).to(torch.bfloat16)
    return x


# ---------------------------------------------------------------------------
# cfg4 student: ResNet-18-style training step (basic blocks). Default: every
# conv followed by training-mode BatchNorm (batch statistics, bn.cu; conv
# without bias, BN's beta in the bias slot, gamma in its own slot). bn=False:
# the BN-free variant (each residual branch's second conv starts small,
# Fixup-style). Parameters live in one flat fp32 master + bf16 copy (Model's
# layout idea), gradients in one flat fp32 vector, so SGD is one edl_sgd_step.

@dataclass(frozen=True)
class StudentResNetConfig:
    layers: tuple = (2, 2, 2, 2)
    width: int = 64
    classes: int = 1000
    image: int = 224
    in_channels: int = 3
    bn: bool = True


def _bn_conv(rng, cin, cout, k, stride, relu=True, gain=1.0):
    """A plain He-normal conv (no bias) followed by BatchNorm: gamma 1, beta 0."""
    w = rng.normal(0.0, np.sqrt(2.0 / (cin * k * k)), size=(cout, cin, k, k)).astype(np.float32)
    return HostConv(w, np.zeros(cout, dtype=np.float32), stride, k // 2, relu, np.ones(cout, dtype=np.float32))


def init_student_resnet(cfg: StudentResNetConfig, seed: int) -> HostResNet:
    rng = np.random.default_rng(seed)
    rcfg = ResNetConfig(block="basic", layers=cfg.layers, width=cfg.width, classes=cfg.classes, image=cfg.image,
                        in_channels=cfg.in_channels)
    mk = _bn_conv if cfg.bn else _conv
    net = HostResNet(rcfg, mk(rng, cfg.in_channels, cfg.width, 7, 2), bn=cfg.bn)
    net.stem.pad = 3
    net.stem.b[:] = 0.0
    cin = cfg.width
    for stage, n in enumerate(cfg.layers):
        cout = cfg.width * (2 ** stage)
        for i in range(n):
            stride = 2 if (i == 0 and stage > 0) else 1
            c1 = mk(rng, cin, cout, 3, stride)
            c2 = mk(rng, cout, cout, 3, 1, relu=True, gain=0.25)
            shortcut = None
            if stride != 1 or cin != cout:
                shortcut = mk(rng, cin, cout, 1, stride, relu=False)
                shortcut.pad = 0
            net.blocks.append(HostBlock([c1, c2], shortcut))
            cin = cout
    net.fc_w = (rng.normal(0.0, np.sqrt(1.0 / cin), size=(cfg.classes, cin))).astype(np.float32)
    net.fc_b = np.zeros(cfg.classes, dtype=np.float32)
    return net


class _Param:
    """A [rows][cols] weight + [rows] bias (BN's beta) view pair inside the flat
    buffers, and BN's gamma [rows] when the conv is followed by BatchNorm."""

    def __init__(self, off_w, rows, cols, off_b, off_g=None):
        self.off_w, self.rows, self.cols, self.off_b, self.off_g = off_w, rows, cols, off_b, off_g


class ResNetStudent:
    """Device ResNet-18-style student: forward (convs + training-mode
    BatchNorm, or BN-free), the fused logit-layer KD head (the MLP students'
    kernel), full backward and SGD, for a fixed batch."""

    BN_EPS = 1e-5

    def __init__(self, host: HostResNet, device=None, batch_size: int = 64):
        self.device = dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.B = B = batch_size
        self.cfg = host.cfg
        self.bn = bool(getattr(host, "bn", False))
        hosts = [host.stem]
        for blk in host.blocks:
            hosts += [blk.convs[0], blk.convs[1]] + ([blk.shortcut] if blk.shortcut is not None else [])
        self.convs = [_DevConv(host.stem, "cpu")]
        self.block_idx = []                                 # (conv1, conv2, shortcut or None) indices
        for blk in host.blocks:
            i1 = len(self.convs); self.convs.append(_DevConv(blk.convs[0], "cpu"))
            i2 = len(self.convs); self.convs.append(_DevConv(blk.convs[1], "cpu"))
            isc = None
            if blk.shortcut is not None:
                isc = len(self.convs); self.convs.append(_DevConv(blk.shortcut, "cpu"))
            self.block_idx.append((i1, i2, isc))
        feat = host.fc_w.shape[1]
        self.feat_p = pad(feat)
        self.classes = host.fc_w.shape[0]
        self.classes_p = pad(self.classes)
        # flat layout: every conv [cout_p][kdim] + bias [cout_p] (+ gamma [cout_p]
        # with BN), then fc [classes_p][feat_p] + [classes_p]
        self.params, off = [], 0
        for c in self.convs:
            p = _Param(off, c.cout_p, c.kdim, off + c.cout_p * c.kdim)
            off = p.off_b + c.cout_p
            if self.bn:
                p.off_g = off
                off += c.cout_p
            self.params.append(p)
        self.fc = _Param(off, self.classes_p, self.feat_p, off + self.classes_p * self.feat_p)
        self.size = self.fc.off_b + self.classes_p
        flat = torch.zeros(self.size, dtype=torch.float32)
        for c, p, hc in zip(self.convs, self.params, hosts):
            flat[p.off_w:p.off_w + p.rows * p.cols] = c.w.float().reshape(-1)
            flat[p.off_b:p.off_b + p.rows] = c.b
            if self.bn:
                flat[p.off_g:p.off_g + hc.gamma.shape[0]] = torch.from_numpy(hc.gamma)
        fcw = torch.zeros(self.classes_p, self.feat_p)
        fcw[:self.classes, :feat] = torch.from_numpy(host.fc_w)
        flat[self.fc.off_w:self.fc.off_w + self.classes_p * self.feat_p] = fcw.reshape(-1)
        flat[self.fc.off_b:self.fc.off_b + self.classes] = torch.from_numpy(host.fc_b)
        self.flat = flat.to(dev)
        self.flat_bf16 = self.flat.to(torch.bfloat16)
        self.grads = torch.zeros(self.size, dtype=torch.float32, device=dev)
        for c in self.convs:                                # device copies are views into the flat buffers
            c.w = c.b = None
        # activations (post-ReLU outputs are kept for the backward masks)
        H = self.cfg.image
        stem = self.convs[0]
        h, w = stem.out_hw(H, H)
        self.stem_hw = (h, w)
        self.y0 = torch.empty(B, h, w, stem.cout_p, dtype=torch.bfloat16, device=dev)
        ph, pw = (h + 2 - 3) // 2 + 1, (w + 2 - 3) // 2 + 1
        self.pool_hw = (ph, pw)
        self.x1 = torch.empty(B, ph, pw, stem.cout_p, dtype=torch.bfloat16, device=dev)
        self.pool_arg = torch.empty(B * ph * pw * stem.cout_p // 8, dtype=torch.int32, device=dev)
        col = B * h * w * stem.kdim
        self.acts, hw = [], (ph, pw)                        # per block: (in_hw, h1, sc, y)
        for i1, i2, isc in self.block_idx:
            c1, c2 = self.convs[i1], self.convs[i2]
            oh, ow = c1.out_hw(*hw)
            h1 = torch.empty(B, oh, ow, c1.cout_p, dtype=torch.bfloat16, device=dev)
            y = torch.empty(B, oh, ow, c2.cout_p, dtype=torch.bfloat16, device=dev)
            sc = torch.empty(B, oh, ow, c2.cout_p, dtype=torch.bfloat16, device=dev) if isc is not None else None
            col = max(col, B * oh * ow * max(c1.kdim, c2.kdim))
            self.acts.append((hw, h1, sc, y))
            hw = (oh, ow)
        self.final_hw = hw
        # implicit-GEMM convs (>= 64 input channels) read their input through
        # TMA im2col maps in the forward and the weight gradient: no column
        # matrix. The packed RGB stem keeps its forward column matrix for its
        # weight gradient; self.col is the data-gradient scratch
        self.in_hw = [(H, H)] + [None] * (len(self.convs) - 1)
        for (i1, i2, isc), (hw_in, _, _, _) in zip(self.block_idx, self.acts):
            self.in_hw[i1] = hw_in
            self.in_hw[i2] = self.convs[i1].out_hw(*hw_in)
            if isc is not None:
                self.in_hw[isc] = hw_in
        self.cols, ws = [], 0
        for i, c in enumerate(self.convs):
            oh, ow = c.out_hw(*self.in_hw[i])
            M = B * oh * ow
            self.cols.append(None if (c.k == 1 and c.stride == 1) or c.implicit else
                             torch.empty(M, c.kdim, dtype=torch.bfloat16, device=dev))
            ws = max(ws, int(_lib.load().edl_bwd_weight_workspace_floats(M, c.cout_p, c.kdim)))
        self.wgrad_ws = torch.empty(max(ws, 1), dtype=torch.float32, device=dev)
        # stride-1 data gradients run as implicit-GEMM convolutions of dZ with
        # the flipped filter (refreshed from the forward's bf16 weights each step)
        self.wflip = [torch.empty(c.cin_p, c.k * c.k * c.cout_p, dtype=torch.bfloat16, device=dev)
                      if i > 0 and self._dgrad_implicit(c) else None for i, c in enumerate(self.convs)]
        import ctypes
        fl = [(c, p, wf) for c, p, wf in zip(self.convs, self.params, self.wflip) if wf is not None]
        n = len(fl)
        self._flip_keep = (
            (ctypes.c_void_p * n)(*[self._w16(p).data_ptr() for _, p, _ in fl]),
            (ctypes.c_longlong * n)(*[c.kdim for c, _, _ in fl]),
            (ctypes.c_int * n)(*[c.cout_p for c, _, _ in fl]),
            (ctypes.c_int * n)(*[c.cin_p for c, _, _ in fl]),
            (ctypes.c_int * n)(*[c.k for c, _, _ in fl]),
            (ctypes.c_int * n)(*[c.k for c, _, _ in fl]),
            (ctypes.c_void_p * n)(*[wf.data_ptr() for _, _, wf in fl]),
            (ctypes.c_longlong * n)(*[wf.stride(0) for _, _, wf in fl]))
        self._flip_args = (n, *[ctypes.cast(a, ctypes.c_void_p) for a in self._flip_keep])
        self.col = torch.empty(col, dtype=torch.bfloat16, device=dev)
        # backward buffers: gradient ping-pong at the largest activation size + a shortcut buffer
        big = max(B * h * w * stem.cout_p, max(a[1].numel() for a in self.acts))
        self.g = [torch.empty(big, dtype=torch.bfloat16, device=dev) for _ in range(4 if self.bn else 3)]
        cmax = max(c.cout_p for c in self.convs)
        self.zero_b = torch.zeros(cmax, dtype=torch.float32, device=dev)
        if self.bn:
            # pre-BN conv outputs z (the backward recomputes xhat from them),
            # per-conv batch mean / rstd, the reductions' workspace
            self.z0 = torch.empty_like(self.y0)
            self.zs = [(torch.empty_like(h1), torch.empty_like(y), torch.empty_like(sc) if sc is not None else None)
                       for (_, h1, sc, y) in self.acts]
            self.bn_stats = torch.empty(len(self.convs), 2, cmax, dtype=torch.float32, device=dev)
            wsn = 0
            for i, c in enumerate(self.convs):
                oh, ow = c.out_hw(*self.in_hw[i])
                wsn = max(wsn, int(_lib.load().edl_bn_workspace_floats(B * oh * ow, c.cout_p)))
            self.bn_ws = torch.empty(max(wsn, 1), dtype=torch.float32, device=dev)
        self.features = torch.empty(B, self.feat_p, dtype=torch.bfloat16, device=dev)
        self.logits = torch.empty(B, self.classes_p, dtype=torch.float32, device=dev)
        self.dlogits = torch.empty(B, self.classes_p, dtype=torch.bfloat16, device=dev)
        self.dfeat = torch.empty(B, self.feat_p, dtype=torch.bfloat16, device=dev)
        self.row_loss = torch.empty(B, dtype=torch.float32, device=dev)
        self.loss = torch.zeros(1, dtype=torch.float32, device=dev)
        self.ticket = torch.zeros(1, dtype=torch.int32, device=dev)
        self.status = torch.zeros(1, dtype=torch.int32, device=dev)
        self.colsum_ws = torch.empty(max(int(_lib.load().edl_colsum_workspace_floats(B, self.classes_p)), 1),
                                     dtype=torch.float32, device=dev)   # the head's db

    # views
    def _w16(self, p):
        return self.flat_bf16[p.off_w:p.off_w + p.rows * p.cols]

    def _b(self, p):
        return self.flat[p.off_b:p.off_b + p.rows]

    def _g(self, p):
        return self.flat[p.off_g:p.off_g + p.rows]

    def _gg(self, p):
        return self.grads[p.off_g:p.off_g + p.rows]

    def _gw(self, p):
        return self.grads[p.off_w:p.off_w + p.rows * p.cols]

    def _gb(self, p):
        return self.grads[p.off_b:p.off_b + p.rows]

    def _im2col(self, i, x, hw, s):
        c = self.convs[i]
        if c.k == 1 and c.stride == 1:
            return x, c.cin_p
        _lib.call("edl_im2col_nhwc", x.data_ptr(), self.B, hw[0], hw[1], c.cin_p, c.cin if c.packed else c.cin_p,
                  c.k, c.k, c.stride, c.pad, self.cols[i].data_ptr(), c.kdim, s)
        return self.cols[i], c.kdim

    def _fwd(self, i, x, hw, out, residual, s, raw=False):
        """Conv i: out = act(conv(x) + b [+ residual]); raw=True (BN): out = conv(x)."""
        c, p = self.convs[i], self.params[i]
        oh, ow = c.out_hw(*hw)
        bias = self.zero_b if raw else self._b(p)
        if c.implicit:
            act = _lib.EDL_ACT_IDENT if raw else (
                _lib.EDL_ACT_RELU if (c.relu or residual is not None) else _lib.EDL_ACT_IDENT)
            _lib.call("edl_conv_fwd_nhwc", x.data_ptr(), self.B, hw[0], hw[1], c.cin_p, self._w16(p).data_ptr(),
                      c.kdim, bias.data_ptr(), c.cout_p, c.k, c.k, c.stride, c.pad,
                      None if residual is None else residual.data_ptr(), c.cout_p, out.data_ptr(), c.cout_p, act, s)
            return
        a, lda = self._im2col(i, x, hw, s)
        M = self.B * oh * ow
        if raw:
            _lib.call("edl_linear_fwd", a.data_ptr(), lda, self._w16(p).data_ptr(), c.kdim, bias.data_ptr(),
                      out.data_ptr(), c.cout_p, M, c.cout_p, c.kdim, _lib.EDL_ACT_IDENT, s)
            return
        if residual is not None:
            _lib.call("edl_linear_fwd_residual", a.data_ptr(), lda, self._w16(p).data_ptr(), c.kdim,
                      self._b(p).data_ptr(), residual.data_ptr(), c.cout_p, out.data_ptr(), c.cout_p, M, c.cout_p,
                      c.kdim, s)
        else:
            _lib.call("edl_linear_fwd", a.data_ptr(), lda, self._w16(p).data_ptr(), c.kdim, self._b(p).data_ptr(),
                      out.data_ptr(), c.cout_p, M, c.cout_p, c.kdim,
                      _lib.EDL_ACT_RELU if c.relu else _lib.EDL_ACT_IDENT, s)

    def _bn_stats(self, i, z, s):
        """Batch mean / rstd of conv i's output z into bn_stats[i]."""
        c = self.convs[i]
        M = z.numel() // c.cout_p
        _lib.call("edl_bn_stats_nhwc", z.data_ptr(), M, c.cout_p, self.bn_ws.data_ptr(), self.bn_ws.numel(),
                  self.bn_stats[i, 0].data_ptr(), self.bn_stats[i, 1].data_ptr(), self.BN_EPS, s)

    def _bn_fwd(self, i, z, y, residual, relu, s):
        """Batch statistics of conv i's output z, then y = [relu](gamma xhat + beta [+ residual])."""
        c, p = self.convs[i], self.params[i]
        M = z.numel() // c.cout_p
        mean, rstd = self.bn_stats[i, 0], self.bn_stats[i, 1]
        self._bn_stats(i, z, s)
        _lib.call("edl_bn_apply_nhwc", z.data_ptr(), M, c.cout_p, mean.data_ptr(), rstd.data_ptr(),
                  self._g(p).data_ptr(), self._b(p).data_ptr(), None if residual is None else residual.data_ptr(),
                  1 if relu else 0, y.data_ptr(), s)

    def _bn_bwd(self, i, g, z, dz, s):
        """dgamma, dbeta into the flat gradient; dz = BN's input gradient."""
        c, p = self.convs[i], self.params[i]
        M = z.numel() // c.cout_p
        _lib.call("edl_bn_bwd_nhwc", g.data_ptr(), z.data_ptr(), M, c.cout_p, self.bn_stats[i, 0].data_ptr(),
                  self.bn_stats[i, 1].data_ptr(), self._g(p).data_ptr(), self.bn_ws.data_ptr(), self.bn_ws.numel(),
                  self._gg(p).data_ptr(), self._gb(p).data_ptr(), dz.data_ptr(), s)

    def _features_into(self, x, s):
        """Stem, max pool, residual blocks, global average pool -> self.features."""
        H = self.cfg.image
        h, w = self.stem_hw
        if self.bn:
            # the stem's BN + ReLU run inside its max pool (the 411 MB y0 is
            # never written); argmax words carry the ReLU mask
            self._fwd(0, x, (H, H), self.z0, None, s, raw=True)
            c, p = self.convs[0], self.params[0]
            self._bn_stats(0, self.z0, s)
            _lib.call("edl_bn_relu_maxpool_argmax_nhwc", self.z0.data_ptr(), self.B, h, w, c.cout_p,
                      self.bn_stats[0, 0].data_ptr(), self.bn_stats[0, 1].data_ptr(), self._g(p).data_ptr(),
                      self._b(p).data_ptr(), 3, 2, 1, self.x1.data_ptr(), self.pool_arg.data_ptr(), s)
        else:
            self._fwd(0, x, (H, H), self.y0, None, s)
            # the pool input is the stem's ReLU output: argmax words carry its mask
            _lib.call("edl_maxpool_argmax_relu_nhwc", self.y0.data_ptr(), self.B, h, w, self.y0.shape[-1], 3, 2, 1,
                      self.x1.data_ptr(), self.pool_arg.data_ptr(), s)
        cur = self.x1
        for bi, ((i1, i2, isc), (hw, h1, sc, y)) in enumerate(zip(self.block_idx, self.acts)):
            shortcut = cur
            c1hw = self.convs[i1].out_hw(*hw)
            if self.bn:
                z1, z2, zsc = self.zs[bi]
                if isc is not None:
                    self._fwd(isc, cur, hw, zsc, None, s, raw=True)
                    self._bn_fwd(isc, zsc, sc, None, False, s)
                    shortcut = sc
                self._fwd(i1, cur, hw, z1, None, s, raw=True)
                self._bn_fwd(i1, z1, h1, None, True, s)
                self._fwd(i2, h1, c1hw, z2, None, s, raw=True)
                self._bn_fwd(i2, z2, y, shortcut, True, s)
            else:
                if isc is not None:
                    self._fwd(isc, cur, hw, sc, None, s)
                    shortcut = sc
                self._fwd(i1, cur, hw, h1, None, s)
                self._fwd(i2, h1, c1hw, y, shortcut, s)
            cur = y
        fh, fw = self.final_hw
        _lib.call("edl_avgpool_nhwc", cur.data_ptr(), self.B, fh * fw, cur.shape[-1], self.features.data_ptr(),
                  self.feat_p, s)

    def forward(self, x, s):
        """features + the linear head: fp32 logits in self.logits (dense API)."""
        self._features_into(x, s)
        _lib.call("edl_linear_fwd", self.features.data_ptr(), self.feat_p, self._w16(self.fc).data_ptr(), self.feat_p,
                  self._b(self.fc).data_ptr(), self.logits.data_ptr(), self.classes_p, self.B, self.classes_p,
                  self.feat_p, _lib.EDL_ACT_NONE, s)

    def _wgrad(self, i, dz, x, hw, s):
        """dW_i = dz^T im2col(x), db_i = colsum(dz) (fp32, into the flat gradient);
        im2col(x) is the forward's kept column matrix. Split-K tcgen05 GEMM
        (edl_linear_bwd_weight_ws): the reduction runs over all B*H*W pixels."""
        c, p = self.convs[i], self.params[i]
        oh, ow = c.out_hw(*hw)
        M = self.B * oh * ow
        db = None if self.bn else self._gb(p).data_ptr()   # with BN the conv has no bias (beta's grad: _bn_bwd)
        if c.implicit:
            _lib.call("edl_conv_bwd_weight_nhwc", x.data_ptr(), self.B, hw[0], hw[1], c.cin_p, c.k, c.k, c.stride,
                      c.pad, dz.data_ptr(), c.cout_p, c.cout_p, self._gw(p).data_ptr(), c.kdim,
                      db, self.wgrad_ws.data_ptr(), self.wgrad_ws.numel(), 1.0, s)
            return
        a, lda = (x, c.cin_p) if self.cols[i] is None else (self.cols[i], c.kdim)
        _lib.call("edl_linear_bwd_weight_ws", dz.data_ptr(), c.cout_p, a.data_ptr(), lda, self._gw(p).data_ptr(),
                  c.kdim, db, self.wgrad_ws.data_ptr(), self.wgrad_ws.numel(), M, c.cout_p,
                  c.kdim, 1.0, s)

    @staticmethod
    def _dgrad_implicit(c) -> bool:
        return c.stride == 1 and not c.packed and c.cout_p % 64 == 0 and c.pad == c.k // 2

    def _dgrad(self, i, dz, hw, out, add, mask, s):
        """out = col2im(dz W_i) (+ add) (* mask > 0): the gradient w.r.t. conv i's input.
        Stride 1: one implicit-GEMM convolution of dz with the flipped filter
        (edl_conv_dgrad_nhwc, add and mask in its epilogue); stride 2: the
        column gradient dz W_i, then the col2im gather."""
        c, p = self.convs[i], self.params[i]
        oh, ow = c.out_hw(*hw)
        if self.wflip[i] is not None:
            _lib.call("edl_conv_dgrad_nhwc", dz.data_ptr(), self.B, oh, ow, c.cout_p, self.wflip[i].data_ptr(),
                      self.wflip[i].stride(0), c.cin_p, c.k, c.k, c.pad, None if add is None else add.data_ptr(),
                      None if mask is None else mask.data_ptr(), out.data_ptr(), s)
            return
        M = self.B * oh * ow
        dcol = self.col[:M * c.kdim]
        _lib.call("edl_linear_bwd_data", dz.data_ptr(), c.cout_p, self._w16(p).data_ptr(), c.kdim, None, 0,
                  dcol.data_ptr(), c.kdim, M, c.cout_p, c.kdim, s)
        _lib.call("edl_col2im_nhwc", dcol.data_ptr(), c.kdim, self.B, hw[0], hw[1], c.cin_p, c.k, c.k, c.stride,
                  c.pad, None if add is None else add.data_ptr(), None if mask is None else mask.data_ptr(),
                  out.data_ptr(), s)

    def train_step(self, x, hard_labels, soft: SoftLabels | None, alpha: float, beta: float, temperature: float,
                   eta: float, stream=None, process_group=None, world_size: int = 1):
        """Forward, fused KD loss (edl/nnkit.py:283-309 semantics), backward, SGD.
        world_size > 1: the flat gradient is all-reduced over `process_group`
        (NCCL, edl/allreduce.py:77-120) and the mean folded into SGD's step."""
        s = (stream or torch.cuda.current_stream()).cuda_stream
        B = self.B
        self._features_into(x, s)
        # every stride-1 layer's flipped filter, in one launch
        _lib.call("edl_conv_flip_weights_many", *self._flip_args, s)
        q_vals = soft.probs if (soft is not None and beta > 0) else None
        q_idx = soft.classes if (soft is not None and beta > 0) else None
        k = soft.probs.shape[1] if q_vals is not None else 0
        # the logit layer with the KD loss and dlogits in its epilogue (the MLP
        # students' kd_head_kernel, edl/nnkit.py:283-299): no fp32 logits stored
        _lib.call("edl_linear_kd_loss_fwd_bwd", self.features.data_ptr(), self.feat_p, self._w16(self.fc).data_ptr(),
                  self.feat_p, self._b(self.fc).data_ptr(), hard_labels.data_ptr(),
                  None if q_vals is None else q_vals.data_ptr(), None if q_idx is None else q_idx.data_ptr(), B,
                  self.classes, self.feat_p, k, float(alpha), float(beta), float(temperature),
                  self.row_loss.data_ptr(), self.loss.data_ptr(), self.dlogits.data_ptr(), self.classes_p,
                  self.status.data_ptr(), s)
        # head: dW_fc / db_fc, dfeat = dz W_fc
        _lib.call("edl_linear_bwd_weight", self.dlogits.data_ptr(), self.classes_p, self.features.data_ptr(),
                  self.feat_p, self._gw(self.fc).data_ptr(), self.feat_p, self._gb(self.fc).data_ptr(),
                  self.colsum_ws.data_ptr(), B, self.classes_p, self.feat_p, 1.0, s)
        _lib.call("edl_linear_bwd_data", self.dlogits.data_ptr(), self.classes_p, self._w16(self.fc).data_ptr(),
                  self.feat_p, None, 0, self.dfeat.data_ptr(), self.feat_p, B, self.classes_p, self.feat_p, s)
        # the last block output's ReLU: dZ = avgpool_bwd(dfeat) * (y > 0)
        fh, fw = self.final_hw
        y_last = self.acts[-1][3]
        dz = self.g[0][:y_last.numel()].view_as(y_last)
        _lib.call("edl_avgpool_bwd_nhwc", self.dfeat.data_ptr(), self.feat_p, B, fh * fw, y_last.shape[-1],
                  y_last.data_ptr(), dz.data_ptr(), s)
        cur = 0                                             # dz lives in self.g[cur]
        nb = len(self.g)
        for bi in range(len(self.block_idx) - 1, -1, -1):
            i1, i2, isc = self.block_idx[bi]
            hw, h1, sc, y = self.acts[bi]
            xin = self.x1 if bi == 0 else self.acts[bi - 1][3]
            h1_hw = self.convs[i1].out_hw(*hw)
            if self.bn:
                # dz is g2: the gradient at bn2's output (+ the shortcut), ReLU-masked
                z1, z2, zsc = self.zs[bi]
                b1, b2, b3 = [j for j in range(nb) if j != cur]
                dz2 = self.g[b1][:y.numel()].view_as(y)
                self._bn_bwd(i2, dz, z2, dz2, s)
                self._wgrad(i2, dz2, h1, h1_hw, s)
                g1 = self.g[b2][:h1.numel()].view_as(h1)
                self._dgrad(i2, dz2, h1_hw, g1, None, h1, s)
                dz1 = self.g[b1][:h1.numel()].view_as(h1)     # dz2's readers ran above (stream order)
                self._bn_bwd(i1, g1, z1, dz1, s)
                if isc is not None:
                    dzsc = self.g[b2][:sc.numel()].view_as(sc)  # g1's reader ran above
                    self._bn_bwd(isc, dz, zsc, dzsc, s)
                    self._wgrad(isc, dzsc, xin, hw, s)
                    add = self.g[b3][:xin.numel()].view_as(xin)
                    self._dgrad(isc, dzsc, hw, add, None, None, s)
                    out_buf = cur                               # g2's last readers ran above
                else:
                    add = dz
                    out_buf = b2
                self._wgrad(i1, dz1, xin, hw, s)
                dx = self.g[out_buf][:xin.numel()].view_as(xin)
                self._dgrad(i1, dz1, hw, dx, add, xin if bi > 0 else None, s)
                dz, cur = dx, out_buf
                continue
            b1, b2 = [j for j in range(3) if j != cur]
            # conv2: dW2, db2; dZ1 = col2im(dZ2 W2) * (h1 > 0)
            self._wgrad(i2, dz, h1, h1_hw, s)
            dz1 = self.g[b1][:h1.numel()].view_as(h1)
            self._dgrad(i2, dz, h1_hw, dz1, None, h1, s)
            # the shortcut's gradient (projection: its own dW / dgrad; identity: dZ2)
            if isc is not None:
                self._wgrad(isc, dz, xin, hw, s)
                add = self.g[b2][:xin.numel()].view_as(xin)
                self._dgrad(isc, dz, hw, add, None, None, s)
                out_buf = cur                               # dZ2's last reader ran above (stream order)
            else:
                add = dz
                out_buf = b2
            # conv1: dW1, db1; dX = col2im(dZ1 W1) + shortcut gradient, masked by the input's ReLU
            self._wgrad(i1, dz1, xin, hw, s)
            dx = self.g[out_buf][:xin.numel()].view_as(xin)
            self._dgrad(i1, dz1, hw, dx, add, xin if bi > 0 else None, s)
            dz, cur = dx, out_buf
        # maxpool + stem ReLU, then the stem's weight gradient (the images need no gradient)
        h, w = self.stem_hw
        dy0 = self.g[(cur + 1) % nb][:self.y0.numel()].view_as(self.y0)
        _lib.call("edl_maxpool_bwd_argmax_nhwc", self.pool_arg.data_ptr(), B, h, w, self.y0.shape[-1], 3, 2, 1,
                  dz.data_ptr(), None, dy0.data_ptr(), s)   # ReLU mask folded into the argmax words
        if self.bn:
            dz0 = self.g[(cur + 2) % nb][:self.y0.numel()].view_as(self.y0)
            self._bn_bwd(0, dy0, self.z0, dz0, s)
            dy0 = dz0
        self._wgrad(0, dy0, x, (self.cfg.image, self.cfg.image), s)
        if world_size > 1:
            with torch.cuda.stream(stream or torch.cuda.current_stream()):
                torch.distributed.all_reduce(self.grads, group=process_group)
        _lib.call("edl_sgd_step", self.flat.data_ptr(), self.flat_bf16.data_ptr(), self.grads.data_ptr(), self.size,
                  float(eta) / world_size, s)
        return self.loss

    def flops_per_sample(self) -> float:
        """Algorithmic GEMM FLOPs per image for one training step: forward,
        dgrad (all but the stem) and wgrad."""
        total = 0.0
        H = self.cfg.image
        for idx, c in enumerate(self.convs):
            if idx == 0:
                oh, ow = c.out_hw(H, H)
                total += 2 * 2.0 * oh * ow * c.cout_p * c.kdim
                continue
        for (i1, i2, isc), (hw, _, _, _) in zip(self.block_idx, self.acts):
            for i, inhw in ((i1, hw), (i2, self.convs[i1].out_hw(*hw))) + (((isc, hw),) if isc is not None else ()):
                c = self.convs[i]
                oh, ow = c.out_hw(*inhw)
                total += 3 * 2.0 * oh * ow * c.cout_p * c.kdim
        total += 3 * 2.0 * self.classes_p * self.feat_p
        return total
