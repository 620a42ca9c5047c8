"""Device mirror of edl.nnkit (reference: pkg/src/edl/nnkit.py) on sm_100a.

Same names, argument meaning and exception classes as the reference; the
arithmetic runs in libedl_b200.so (tcgen05 GEMMs + fused loss / softmax /
top-k / SGD kernels). Differences that follow from the device design, all
deliberate:

* Parameters live on the GPU as one flat fp32 master buffer (the reference's
  flatten order W0,b0,W1,b1,... of edl/nnkit.py:342-347, each matrix padded to
  multiples of 16 with zeros) plus a bf16 copy that feeds the tensor cores.
* `sgd_step` updates the master in place and returns the same Model (the
  reference returns a new frozen Model, edl/nnkit.py:312-322).
* `kd_loss` returns a `DeviceLoss` (device scalar) instead of a Python float so
  the step never blocks; `float(loss)` synchronises and raises NumericError for
  a non-finite loss exactly where the reference would (edl/nnkit.py:296-297).
* Soft labels are the teacher's top-k (probability, class) pairs
  (`SoftLabels`); k = K carries the dense distribution of the reference.
"""

from __future__ import annotations

import os
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .formats import HostModel, ModelFileError  # noqa: F401  (re-export, edl/nnkit.py:39)


class ShapeError(ValueError):
    """Model/batch dimensions do not line up (edl/nnkit.py:31-32)."""


class NumericError(ArithmeticError):
    """A loss or parameter became non-finite (edl/nnkit.py:35-36)."""


PAD = 16


def pad(n: int) -> int:
    return (int(n) + PAD - 1) // PAD * PAD


def img_pad(c: int) -> int:
    """Channel pitch of NHWC image inputs: 8 for the RGB stems' packed im2col
    (< 8 channels: one 16-byte load per pixel, half the bytes of a 16-pitch),
    else pad(c)."""
    return 8 if int(c) < 8 else pad(c)


def _stream(stream=None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def _ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


# ---------------------------------------------------------------------------
# Value types


@dataclass(frozen=True)
class TrainConfig:
    """edl/nnkit.py:138-155 (same defaults and validation)."""

    eta: float = 0.05
    alpha: float = 1.0
    beta: float = 0.0
    temperature: float = 2.0
    batch_size: int = 32
    seed: int = 0

    def __post_init__(self):
        if self.eta <= 0:
            raise ValueError("eta must be > 0")
        if self.alpha < 0 or self.beta < 0 or self.alpha + self.beta <= 0:
            raise ValueError("need alpha, beta >= 0 and alpha + beta > 0")
        if self.temperature <= 0:
            raise ValueError("temperature must be > 0")
        if self.batch_size < 1:
            raise ValueError("batch_size must be >= 1")


class _FlatLayout:
    """Offsets of W_l / b_l inside the flat padded parameter vector."""

    def __init__(self, dims: tuple[int, ...]):
        self.dims = dims
        self.dims_p = tuple(pad(d) for d in dims)
        self.w_off, self.b_off = [], []
        off = 0
        for l in range(len(dims) - 1):
            self.w_off.append(off)
            off += self.dims_p[l + 1] * self.dims_p[l]
            self.b_off.append(off)
            off += self.dims_p[l + 1]
        self.size = off

    @property
    def layers(self) -> int:
        return len(self.dims) - 1


class Model:
    """Device-resident tanh MLP (edl/nnkit.py:51-86): fp32 master + bf16 copy."""

    def __init__(self, layer_dims, device=None):
        dims = tuple(int(d) for d in layer_dims)
        if len(dims) < 2 or any(d < 1 for d in dims):
            raise ShapeError(f"need >=2 positive layer dims, got {dims}")
        self.layer_dims = dims
        self.layout = _FlatLayout(dims)
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.flat = torch.zeros(self.layout.size, dtype=torch.float32, device=self.device)
        self.flat_bf16 = torch.zeros(self.layout.size, dtype=torch.bfloat16, device=self.device)

    # reference accessors
    @property
    def input_dim(self) -> int:
        return self.layer_dims[0]

    @property
    def num_classes(self) -> int:
        return self.layer_dims[-1]

    def num_params(self) -> int:
        d = self.layer_dims
        return sum(d[l + 1] * d[l] + d[l + 1] for l in range(len(d) - 1))

    # padded views
    def w(self, l: int) -> torch.Tensor:
        L = self.layout
        n = L.dims_p[l + 1] * L.dims_p[l]
        return self.flat[L.w_off[l]:L.w_off[l] + n].view(L.dims_p[l + 1], L.dims_p[l])

    def w_bf16(self, l: int) -> torch.Tensor:
        L = self.layout
        n = L.dims_p[l + 1] * L.dims_p[l]
        return self.flat_bf16[L.w_off[l]:L.w_off[l] + n].view(L.dims_p[l + 1], L.dims_p[l])

    def b(self, l: int) -> torch.Tensor:
        L = self.layout
        return self.flat[L.b_off[l]:L.b_off[l] + L.dims_p[l + 1]]

    # host <-> device
    @classmethod
    def from_host(cls, host: HostModel, device=None) -> "Model":
        m = cls(host.layer_dims, device)
        m.load_host(host)
        return m

    def load_host(self, host: HostModel) -> None:
        if tuple(host.layer_dims) != self.layer_dims:
            raise ShapeError(f"dims {host.layer_dims} != {self.layer_dims}")
        L = self.layout
        buf = np.zeros(L.size, dtype=np.float32)
        for l, (w, b) in enumerate(zip(host.weights, host.biases)):
            if w.shape != (self.layer_dims[l + 1], self.layer_dims[l]) or b.shape != (self.layer_dims[l + 1],):
                raise ShapeError(f"layer {l}: weight {w.shape} / bias {b.shape} do not match dims")
            if not (np.isfinite(w).all() and np.isfinite(b).all()):
                raise NumericError(f"layer {l} has non-finite parameters")
            view = buf[L.w_off[l]:L.w_off[l] + L.dims_p[l + 1] * L.dims_p[l]].reshape(L.dims_p[l + 1], L.dims_p[l])
            view[:w.shape[0], :w.shape[1]] = w
            buf[L.b_off[l]:L.b_off[l] + b.shape[0]] = b
        self.flat.copy_(torch.from_numpy(buf))
        self.refresh_bf16()

    def refresh_bf16(self) -> None:
        _lib.call("edl_cast_bf16", self.flat.data_ptr(), self.layout.size, self.flat_bf16.data_ptr(),
                  self.layout.size, 1, self.layout.size, _stream())

    def to_host(self) -> HostModel:
        flat = self.flat.detach().to("cpu", torch.float64).numpy()
        L = self.layout
        ws, bs = [], []
        for l in range(L.layers):
            w = flat[L.w_off[l]:L.w_off[l] + L.dims_p[l + 1] * L.dims_p[l]].reshape(L.dims_p[l + 1], L.dims_p[l])
            ws.append(w[:self.layer_dims[l + 1], :self.layer_dims[l]].copy())
            bs.append(flat[L.b_off[l]:L.b_off[l] + self.layer_dims[l + 1]].copy())
        return HostModel(self.layer_dims, tuple(ws), tuple(bs))


@dataclass
class Gradients:
    """Flat fp32 gradient vector in the Model's padded layout."""

    flat: torch.Tensor
    layout: _FlatLayout


@dataclass
class Batch:
    """Device batch: inputs bf16 [B][pad(D)] (zero padded), labels int64 [B]."""

    inputs: torch.Tensor
    hard_labels: torch.Tensor
    dim: int

    @property
    def size(self) -> int:
        return self.inputs.shape[0]


@dataclass
class SoftLabels:
    """Teacher top-k soft labels: probs fp32 [B][k], classes int32 [B][k]
    (probability desc, ties -> lower class), tempered at `temperature`."""

    probs: torch.Tensor
    classes: torch.Tensor
    temperature: float
    # the iteration's input batch when the teacher worker gathered it into the
    # reader's slot on the student's device (DistilReader share_batch): the
    # student trains on it instead of gathering the same rows again
    batch: "Batch | None" = None
    # the producing teacher's class count (its head width); kd_loss raises
    # ShapeError when it differs from the student's (edl/nnkit.py:272-274)
    num_classes: int | None = None

    @property
    def size(self) -> int:
        return self.probs.shape[0]

    @property
    def k(self) -> int:
        return self.probs.shape[1]


class DeviceLoss:
    """Batch-mean loss still on the device; float() syncs and validates."""

    def __init__(self, value: torch.Tensor, status: torch.Tensor):
        self.value = value
        self.status = status

    def __float__(self) -> float:
        v = float(self.value.item())
        check_status(self.status)
        if not np.isfinite(v):
            raise NumericError(f"loss is not finite: {v}")
        return v


def check_status(status: torch.Tensor) -> None:
    """Read a loss workspace's device status word (synchronises) and raise the
    reference's exception for a device-detected error (bad label / class id
    -> ShapeError, non-finite loss -> NumericError, edl/nnkit.py:272-297).
    The word is sticky across launches until read here; raising clears it, so
    one bad batch does not poison later checks on the same workspace."""
    st = int(status.item())
    if st == 0:
        return
    status.zero_()
    if st == _lib.EDL_ERR_SHAPE:
        raise ShapeError("label or soft-label class out of range")
    raise NumericError("loss is not finite")


def make_batch(inputs, labels, device=None) -> Batch:
    """Upload a host (B x D float, B int) batch into the padded bf16 layout."""
    x = np.asarray(inputs)
    if x.ndim != 2 or x.shape[0] < 1:
        raise ShapeError(f"inputs must be a non-empty B x D matrix, got {x.shape}")
    y = np.asarray(labels, dtype=np.int64)
    if y.shape != (x.shape[0],):
        raise ShapeError("one hard label per input row required")
    dev = device or torch.device("cuda", torch.cuda.current_device())
    xb = torch.zeros(x.shape[0], pad(x.shape[1]), dtype=torch.bfloat16)
    xb[:, :x.shape[1]] = torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).to(torch.bfloat16)
    return Batch(xb.to(dev, non_blocking=True), torch.from_numpy(y).to(dev, non_blocking=True), x.shape[1])


# ---------------------------------------------------------------------------
# Workspace (allocated once per (model shape, batch size); the step path never
# allocates)


class Workspace:
    def __init__(self, model: Model, batch_size: int):
        L = model.layout
        dev = model.device
        B = int(batch_size)
        self.batch_size = B
        self.acts = [None] + [torch.empty(B, L.dims_p[l], dtype=torch.bfloat16, device=dev)
                              for l in range(1, L.layers)]
        self.logits = torch.empty(B, L.dims_p[-1], dtype=torch.float32, device=dev)
        self.deltas = [None] + [torch.empty(B, L.dims_p[l], dtype=torch.bfloat16, device=dev)
                                for l in range(1, L.layers + 1)]
        self.row_loss = torch.empty(B, dtype=torch.float32, device=dev)
        self.loss = torch.zeros(1, dtype=torch.float32, device=dev)
        self.ticket = torch.zeros(1, dtype=torch.int32, device=dev)
        self.status = torch.zeros(1, dtype=torch.int32, device=dev)
        ws = max(_lib.colsum_group_workspace_floats([B] * len(part), [L.dims_p[l + 1] for l in part])
                 for part in (list(range(L.layers))[c:c + 4] for c in range(0, L.layers, 4)))
        self.colsum = torch.empty(max(ws, 1), dtype=torch.float32, device=dev)
        self.grads = Gradients(torch.zeros(L.size, dtype=torch.float32, device=dev), L)
        self.probs = None
        self._head_ws: dict = {}

    def head_workspace(self, N: int, k: int) -> torch.Tensor:
        """Zeroed scratch of the pair head (class-chunk states + tickets)."""
        key = (N, k)
        t = self._head_ws.get(key)
        if t is None:
            nbytes = int(_lib.load().edl_teacher_head_workspace_bytes(self.batch_size, N, k))
            t = self._head_ws[key] = torch.zeros(max(nbytes, 1), dtype=torch.uint8, device=self.grads.flat.device)
        return t


_WS: dict = {}


def workspace_for(model: Model, batch_size: int) -> Workspace:
    key = (model.layer_dims, int(batch_size), str(model.device), id(model))
    ws = _WS.get(key)
    if ws is None:
        if len(_WS) > 64:
            _WS.clear()
        ws = _WS[key] = Workspace(model, batch_size)
    return ws


# ---------------------------------------------------------------------------
# Core math (edl/nnkit.py:193-335)


def _forward_into(model: Model, x: torch.Tensor, ws: Workspace, stream=None, layer_ready=None,
                  layers: int | None = None) -> torch.Tensor:
    """acts[1..L-1] = tanh layers, ws.logits = last layer (fp32); `layers`
    stops early (kd_loss runs the logit layer fused with the loss).
    layer_ready[l] (optional CUDA event) gates layer l's GEMM: its parameters
    are still being updated on another stream (StudentStep's overlapped
    gradient exchange)."""
    L = model.layout
    B = x.shape[0]
    s = _stream(stream)
    h = x
    for l in range(L.layers if layers is None else layers):
        if layer_ready is not None and layer_ready[l] is not None:
            (stream or torch.cuda.current_stream()).wait_event(layer_ready[l])
        last = l == L.layers - 1
        out = ws.logits if last else ws.acts[l + 1]
        _lib.call("edl_linear_fwd", h.data_ptr(), h.stride(0), model.w_bf16(l).data_ptr(), L.dims_p[l],
                  model.b(l).data_ptr(), out.data_ptr(), out.stride(0), B, L.dims_p[l + 1], L.dims_p[l],
                  _lib.EDL_ACT_NONE if last else _lib.EDL_ACT_TANH, s)
        h = out
    return ws.logits


def _check_inputs(model: Model, x: torch.Tensor) -> None:
    if x.dim() != 2 or x.dtype != torch.bfloat16 or x.shape[1] != pad(model.input_dim):
        raise ShapeError(f"inputs must be B x {model.input_dim} (bf16, padded to {pad(model.input_dim)}),"
                         f" got {tuple(x.shape)} {x.dtype}")
    if x.shape[0] < 1:
        raise ShapeError("empty batch")


def forward(model: Model, inputs, stream=None) -> torch.Tensor:
    """Logits fp32 [B][K] (edl/nnkit.py:223-234)."""
    x = inputs.inputs if isinstance(inputs, Batch) else inputs
    if not isinstance(x, torch.Tensor):
        x = make_batch(x, np.zeros(len(x), dtype=np.int64), model.device).inputs
    _check_inputs(model, x)
    ws = workspace_for(model, x.shape[0])
    return _forward_into(model, x, ws, stream)[:, :model.num_classes]


def tempered_softmax(logits: torch.Tensor, temperature: float, stream=None) -> torch.Tensor:
    """Row-wise softmax(z / T) (edl/nnkit.py:193-208), fp32 on device."""
    if not np.isfinite(temperature) or temperature <= 0:
        raise ValueError(f"temperature must be a positive finite real, got {temperature}")
    z = logits if logits.dim() == 2 else logits.view(1, -1)
    if z.dtype != torch.float32:
        raise ShapeError("logits must be fp32")
    out = torch.empty(z.shape[0], z.shape[1], dtype=torch.float32, device=z.device)
    _lib.call("edl_tempered_softmax", z.data_ptr(), z.stride(0), out.data_ptr(), out.stride(0),
              z.shape[0], z.shape[1], float(temperature), _stream(stream))
    return out if logits.dim() == 2 else out.view(-1)


def teacher_soft_labels(model: Model, inputs, temperature: float, k: int, out: SoftLabels | None = None,
                        stream=None, probe: tuple | None = None, ws: Workspace | None = None) -> SoftLabels:
    """Fused teacher inference: hidden tanh layers, then the head GEMM with the
    tempered-softmax + top-k epilogue (edl/teacher_node.py:54 + top-k)."""
    x = inputs.inputs if isinstance(inputs, Batch) else inputs
    _check_inputs(model, x)
    if not np.isfinite(temperature) or temperature <= 0:
        raise ValueError(f"temperature must be a positive finite real, got {temperature}")
    K = model.num_classes
    if not 1 <= k <= min(K, 32):
        raise ValueError(f"k must be in [1, {min(K, 32)}], got {k}")
    L = model.layout
    B = x.shape[0]
    ws = ws or workspace_for(model, B)
    s = _stream(stream)
    h = x
    for l in range(L.layers - 1):
        # probe = (layer, list): CUDA events bracketing that layer's GEMM (bench timing)
        timed = probe is not None and probe[0] == l
        if timed:
            ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
            ev[0].record(stream or torch.cuda.current_stream())
        _lib.call("edl_linear_fwd", h.data_ptr(), h.stride(0), model.w_bf16(l).data_ptr(), L.dims_p[l],
                  model.b(l).data_ptr(), ws.acts[l + 1].data_ptr(), ws.acts[l + 1].stride(0), B,
                  L.dims_p[l + 1], L.dims_p[l], _lib.EDL_ACT_TANH, s)
        if timed:
            ev[1].record(stream or torch.cuda.current_stream())
            probe[1].append(ev)
        h = ws.acts[l + 1]
    if out is None:
        out = SoftLabels(torch.empty(B, k, dtype=torch.float32, device=x.device),
                         torch.empty(B, k, dtype=torch.int32, device=x.device), float(temperature))
    out.num_classes = K
    l = L.layers - 1
    hws = ws.head_workspace(K, int(k))
    _lib.call("edl_teacher_head_softmax_topk_ws", h.data_ptr(), h.stride(0), model.w_bf16(l).data_ptr(),
              L.dims_p[l], model.b(l).data_ptr(), B, K, L.dims_p[l], float(temperature), int(k),
              out.probs.data_ptr(), out.classes.data_ptr(), hws.data_ptr(), hws.numel(), s)
    return out


_KD_UNFUSED = os.environ.get("EDL_KD_UNFUSED") == "1"   # A/B switch: logits GEMM + separate loss kernel


def kd_loss(model: Model, batch: Batch, soft: SoftLabels | None, cfg: TrainConfig,
            stream=None, ws: Workspace | None = None,
            loss_slot: torch.Tensor | None = None,
            fused_sgd_eta: float | None = None, layer_ready=None,
            fused: bool | None = None) -> tuple[DeviceLoss, Gradients | None]:
    """Combined distillation loss and analytic gradients (edl/nnkit.py:254-309):
    hidden forward GEMMs -> the logit GEMM with the loss and dlogits in its
    epilogue (edl_linear_kd_loss_fwd_bwd; fp32 logits never reach HBM) ->
    backward GEMMs. fused=False (or K > 2048) runs the logit GEMM and the
    separate loss kernel instead (ws.logits then holds the logits)."""
    if cfg.beta > 0:
        if soft is None:
            raise ShapeError("beta > 0 requires soft labels")
        if soft.size != batch.size:
            raise ShapeError(f"soft batch {soft.size} != input batch {batch.size}")
        if soft.temperature != cfg.temperature:
            raise ValueError(f"soft labels tempered at {soft.temperature}, config says {cfg.temperature}")
        if soft.k > model.num_classes or (soft.num_classes is not None
                                          and soft.num_classes != model.num_classes):
            raise ShapeError(f"soft labels over {soft.num_classes} classes (k={soft.k}), "
                             f"student has {model.num_classes}")
    x = batch.inputs
    _check_inputs(model, x)
    B = x.shape[0]
    L = model.layout
    ws = ws or workspace_for(model, B)
    s = _stream(stream)
    q_vals = soft.probs if (soft is not None and cfg.beta > 0) else None
    q_idx = soft.classes if (soft is not None and cfg.beta > 0) else None
    k = soft.k if q_vals is not None else 0
    use_fused = (not _KD_UNFUSED if fused is None else fused) and pad(model.num_classes) <= 2048 and k <= 32
    _forward_into(model, x, ws, stream, layer_ready, layers=L.layers - 1 if use_fused else None)
    dz = ws.deltas[L.layers]
    loss = ws.loss if loss_slot is None else loss_slot
    if use_fused:
        l = L.layers - 1
        if layer_ready is not None and layer_ready[l] is not None:
            (stream or torch.cuda.current_stream()).wait_event(layer_ready[l])
        h = x if l == 0 else ws.acts[l]
        _lib.call("edl_linear_kd_loss_fwd_bwd", h.data_ptr(), h.stride(0), model.w_bf16(l).data_ptr(), L.dims_p[l],
                  model.b(l).data_ptr(), batch.hard_labels.data_ptr(), _ptr(q_vals), _ptr(q_idx), B,
                  model.num_classes, L.dims_p[l], k, float(cfg.alpha), float(cfg.beta), float(cfg.temperature),
                  ws.row_loss.data_ptr(), loss.data_ptr(), dz.data_ptr(), dz.stride(0), ws.status.data_ptr(), s)
    else:
        _lib.call("edl_kd_loss_fwd_bwd", ws.logits.data_ptr(), ws.logits.stride(0), batch.hard_labels.data_ptr(),
                  _ptr(q_vals), _ptr(q_idx), B, model.num_classes, k, float(cfg.alpha), float(cfg.beta),
                  float(cfg.temperature), ws.row_loss.data_ptr(), loss.data_ptr(), ws.ticket.data_ptr(),
                  dz.data_ptr(), dz.stride(0), ws.status.data_ptr(), s)
    backward_into(model, x, ws, stream, sgd_eta=fused_sgd_eta)
    # fused_sgd_eta: the model was already updated (kd_loss + sgd_step in one
    # pass, single student); there is no gradient to return
    return DeviceLoss(loss, ws.status), (None if fused_sgd_eta is not None else ws.grads)


def backward_into(model: Model, x: torch.Tensor, ws: Workspace, stream=None,
                  sgd_eta: float | None = None) -> None:
    """dW_l = delta^T a_l, db_l = colsum(delta), delta <- (delta W_l)(1 - a_l^2)
    (edl/nnkit.py:303-308), from ws.deltas[L] = dlogits. With `sgd_eta` the
    update p -= eta * g (edl/nnkit.py:312-322) is fused into the dW / db
    kernels and no gradient is materialised (single-student step)."""
    L = model.layout
    B = x.shape[0]
    s = _stream(stream)
    g = ws.grads.flat
    # the delta chain first (each step needs the previous one) ...
    for l in range(L.layers - 1, 0, -1):
        d = ws.deltas[l + 1]
        a = ws.acts[l]
        _lib.call("edl_linear_bwd_data", d.data_ptr(), d.stride(0), model.w_bf16(l).data_ptr(),
                  L.dims_p[l], a.data_ptr(), a.stride(0), ws.deltas[l].data_ptr(),
                  ws.deltas[l].stride(0), B, L.dims_p[l + 1], L.dims_p[l], s)
    # ... then every layer's dW / db: independent, so one grouped launch
    # (chunks of 4 layers for deeper nets)
    layers = list(range(L.layers - 1, -1, -1))
    for c in range(0, len(layers), 4):
        part = layers[c:c + 4]
        if sgd_eta is not None:
            _lib.bwd_weight_grouped_sgd(
                [ws.deltas[l + 1] for l in part], [x if l == 0 else ws.acts[l] for l in part],
                [model.w(l) for l in part], [model.w_bf16(l) for l in part], [model.b(l) for l in part],
                [model.flat_bf16[L.b_off[l]:L.b_off[l] + L.dims_p[l + 1]] for l in part], ws.colsum,
                [B] * len(part), [L.dims_p[l + 1] for l in part], [L.dims_p[l] for l in part],
                float(sgd_eta), s)
            continue
        _lib.bwd_weight_grouped(
            [ws.deltas[l + 1] for l in part], [x if l == 0 else ws.acts[l] for l in part],
            [g[L.w_off[l]:L.w_off[l] + L.dims_p[l + 1] * L.dims_p[l]] for l in part],
            [g[L.b_off[l]:L.b_off[l] + L.dims_p[l + 1]] for l in part], ws.colsum,
            [B] * len(part), [L.dims_p[l + 1] for l in part], [L.dims_p[l] for l in part], 1.0, s)


def sgd_step(model: Model, grads: Gradients, eta: float, world_size: int = 1, stream=None) -> Model:
    """p <- p - eta * g (edl/nnkit.py:312-322) in place on the fp32 master; the
    all-reduce mean (edl/allreduce.py:119) is folded in as eta / world_size."""
    if grads.layout.size != model.layout.size or grads.layout.dims != model.layer_dims:
        raise ShapeError("gradient layout does not match model")
    _lib.call("edl_sgd_step", model.flat.data_ptr(), model.flat_bf16.data_ptr(), grads.flat.data_ptr(),
              model.layout.size, float(eta) / world_size, _stream(stream))
    return model


def evaluate(model: Model, samples, labels, k: int = 1, batch: int = 4096) -> float:
    """Top-k accuracy, ties toward the lower class (edl/nnkit.py:325-335)."""
    n = len(labels)
    if n < 1:
        raise ValueError("cannot evaluate on an empty dataset")
    if k < 1 or k > model.num_classes:
        raise ValueError(f"k must be in [1, {model.num_classes}], got {k}")
    hits = torch.zeros(1, dtype=torch.int32, device=model.device)
    for i in range(0, n, batch):
        b = make_batch(samples[i:i + batch], labels[i:i + batch], model.device)
        z = forward(model, b.inputs)
        _lib.call("edl_topk_hits", z.data_ptr(), z.stride(0), b.hard_labels.data_ptr(), b.size,
                  model.num_classes, int(k), hits.data_ptr(), _stream())
    return int(hits.item()) / n


# ---------------------------------------------------------------------------
# Model files (edl/nnkit.py:480-487): EDLD v1 in, device model out (fp64 ->
# fp32 master + bf16 copy, dims padded); device model in, EDLD out (fp32
# master widened to f64) — the reference's pretrained teachers and
# checkpoints load unchanged.


def load_model(path: str, device=None) -> tuple[Model, int]:
    from .formats import deserialize_model
    with open(path, "rb") as fh:
        host, iteration = deserialize_model(fh.read())
    return Model.from_host(host, device), iteration


def save_model(path: str, model: Model, iteration: int = 0) -> None:
    import os

    from .formats import serialize_model
    blob = serialize_model(model.to_host(), iteration)
    tmp = f"{path}.tmp.{os.getpid()}"
    with open(tmp, "wb") as fh:
        fh.write(blob)
    os.replace(tmp, path)


# ---------------------------------------------------------------------------
# Parameter flattening (edl/nnkit.py:342-364) — host views in reference order


def flatten_grads(grads: Gradients) -> np.ndarray:
    flat = grads.flat.detach().to("cpu", torch.float64).numpy()
    L = grads.layout
    parts = []
    for l in range(L.layers):
        w = flat[L.w_off[l]:L.w_off[l] + L.dims_p[l + 1] * L.dims_p[l]].reshape(L.dims_p[l + 1], L.dims_p[l])
        parts.append(w[:L.dims[l + 1], :L.dims[l]].ravel())
        parts.append(flat[L.b_off[l]:L.b_off[l] + L.dims[l + 1]])
    return np.concatenate(parts)


def flatten_params(model: Model) -> np.ndarray:
    return flatten_grads(Gradients(model.flat, model.layout))


def unflatten_grads(flat: np.ndarray, model: Model) -> Gradients:
    L = model.layout
    need = model.num_params()
    if flat.size != need:
        raise ShapeError(f"flat vector has {flat.size} elements, model needs {need}")
    buf = np.zeros(L.size, dtype=np.float32)
    off = 0
    for l in range(L.layers):
        r, c = L.dims[l + 1], L.dims[l]
        view = buf[L.w_off[l]:L.w_off[l] + L.dims_p[l + 1] * L.dims_p[l]].reshape(L.dims_p[l + 1], L.dims_p[l])
        view[:r, :c] = flat[off:off + r * c].reshape(r, c)
        off += r * c
        buf[L.b_off[l]:L.b_off[l] + r] = flat[off:off + r]
        off += r
    return Gradients(torch.from_numpy(buf).to(model.device), L)
