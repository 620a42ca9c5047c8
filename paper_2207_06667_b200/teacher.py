"""Device teacher worker — mirror of edl/teacher_node.py.

`soft_label_reply` keeps the reference's request/reply contract
(edl/teacher_node.py:47-58): INFER_REQUEST -> INFER_REPLY or an ERROR that
carries the batch_id, never an exception. The payload differs by design: the
request names dataset rows (or carries a device tensor) instead of shipping
B x D floats as JSON, and the reply carries the fused head's top-k
(probability, class) pairs instead of the dense B x K matrix.

`TeacherWorker` replaces TeacherServer (edl/teacher_node.py:65-203): instead
of a socket reader feeding a depth-4 queue drained by one compute thread, a
job is enqueued on the worker's own CUDA stream (gather rows -> hidden tanh
GEMMs -> head GEMM with softmax/top-k epilogue -> optional peer copy into the
student's slot) and completion is a CUDA event. Stream order is the serial
compute loop; COMPUTE_QUEUE_DEPTH bounds the jobs a student may have in
flight per teacher exactly as the socket queue did.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib, nnkit
from .data import DeviceDataset, gather_batch
from .nnkit import Batch, Model, SoftLabels

COMPUTE_QUEUE_DEPTH = 4   # edl/teacher_node.py:27


@dataclass(frozen=True)
class TeacherConfig:
    node_id: str
    temperature: float = 2.0
    k: int = 16
    simulated_delay: float = 0.0   # seconds per batch, spent on the worker's stream (edl_stream_delay_ns)

    def __post_init__(self):
        if self.temperature <= 0:
            raise ValueError("temperature must be > 0")
        if self.simulated_delay < 0:
            raise ValueError("simulated delay must be >= 0")
        if not 1 <= self.k <= 32:
            raise ValueError("k must be in [1, 32]")


def soft_label_reply(model: Model, temperature: float, request: dict, k: int | None = None,
                     data: DeviceDataset | None = None) -> dict:
    """INFER_REQUEST -> INFER_REPLY (or an ERROR carrying the batch_id).

    request["inputs"]: device bf16 batch (B x pad(D)) or a host B x D array;
    or request["rows"]: dataset row indices (needs `data`)."""
    batch_id = request.get("batch_id")
    try:
        if "rows" in request:
            if data is None:
                raise nnkit.ShapeError("row-indexed request needs the HBM-resident dataset")
            rows = torch.as_tensor(np.asarray(request["rows"], dtype=np.int64)).to(data.device)
            x = gather_batch(data, rows).inputs
        else:
            x = request["inputs"]
            if not isinstance(x, torch.Tensor):
                arr = np.asarray(x, dtype=np.float64)
                if arr.ndim != 2:
                    raise nnkit.ShapeError(f"inputs must be a matrix, got shape {arr.shape}")
                if arr.shape[1] != model.input_dim:
                    raise nnkit.ShapeError(f"inputs must be B x {model.input_dim}, got {arr.shape}")
                x = nnkit.make_batch(arr, np.zeros(arr.shape[0], dtype=np.int64), model.device).inputs
        kk = model.num_classes if k is None else k
        soft = nnkit.teacher_soft_labels(model, x, temperature, min(kk, 32, model.num_classes))
    except (nnkit.ShapeError, ValueError, TypeError) as exc:
        return {"type": "ERROR", "reason": f"bad inference request: {exc}", "batch_id": batch_id}
    return {"type": "INFER_REPLY", "batch_id": batch_id, "probs": soft, "temperature": temperature}


class TeacherWorker:
    """One teacher (model replica) bound to a device and a CUDA stream."""

    def __init__(self, cfg: TeacherConfig, model: Model, data: DeviceDataset, sm_reserve: int = 0):
        """sm_reserve > 0 caps this worker's persistent GEMMs at (SMs - reserve)
        CTAs, leaving SMs for the co-located student's NCCL collectives."""
        if model.device != data.device:
            raise ValueError("teacher model and its dataset replica must share a device")
        self.cfg = cfg
        self.node_id = cfg.node_id
        self.model = model
        self.data = data
        self.device = model.device
        self.stream = torch.cuda.Stream(device=self.device)
        if sm_reserve > 0:
            with torch.cuda.device(self.device):
                sms = _lib.load().edl_device_sms()
            _lib.call("edl_set_stream_max_ctas", self.stream.cuda_stream, max(1, sms - sm_reserve))
        self.alive = True
        self.batches_served = 0
        self._batch: Batch | None = None
        self._ws: nnkit.Workspace | None = None   # private: workers may share a model replica
        self._staging: SoftLabels | None = None
        self.probe: tuple | None = None   # (layer, list) -> events around that layer (bench)

    def submit(self, rows: torch.Tensor, slot) -> None:
        """Enqueue one batch: rows (int64, any device) -> top-k soft labels in
        `slot` (on the slot's device); slot.done is recorded when they land."""
        if not self.alive:
            raise RuntimeError(f"teacher {self.node_id} is stopped")
        B = rows.shape[0]
        with torch.cuda.device(self.device), torch.cuda.stream(self.stream):
            if slot.release is not None:
                self.stream.wait_event(slot.release)          # consumer done with the slot
            if rows.device != self.device:
                rows = rows.to(self.device, non_blocking=True)
            if self._batch is None or self._batch.size != B:
                self._batch = Batch(torch.empty(B, self.data.samples.shape[1], dtype=torch.bfloat16,
                                                device=self.device),
                                    torch.empty(B, dtype=torch.int64, device=self.device), self.data.dim)
            if self._ws is None or self._ws.batch_size != B:
                self._ws = nnkit.Workspace(self.model, B)
            local = slot.probs.device == self.device
            # gather straight into the student's slot when it offers input
            # buffers on this device (reader share_batch): one gather per batch
            target = self._batch
            if local and getattr(slot, "batch", None) is not None and slot.batch.size == B:
                target = slot.batch
            batch = gather_batch(self.data, rows, target, self.stream)
            if target is not self._batch:
                slot.batch_filled = True
                target.inputs.record_stream(self.stream)
                target.hard_labels.record_stream(self.stream)
            if local:
                out = SoftLabels(slot.probs, slot.classes, self.cfg.temperature)
            else:
                if self._staging is None or self._staging.probs.shape != slot.probs.shape:
                    self._staging = SoftLabels(torch.empty_like(slot.probs, device=self.device),
                                               torch.empty_like(slot.classes, device=self.device),
                                               self.cfg.temperature)
                out = self._staging
            nnkit.teacher_soft_labels(self.model, batch.inputs, self.cfg.temperature, slot.probs.shape[1],
                                      out=out, stream=self.stream, probe=self.probe, ws=self._ws)
            if self.cfg.simulated_delay > 0:
                _lib.call("edl_stream_delay_ns", int(self.cfg.simulated_delay * 1e9), self.stream.cuda_stream)
            if not local:
                # NVLink peer copy into the student-owned slot, ordered on this
                # stream only (the student's stream never waits on it here;
                # it waits on slot.done when it consumes the slot)
                for dst, src in ((slot.probs, out.probs), (slot.classes, out.classes)):
                    _lib.call("edl_memcpy_peer_async", dst.data_ptr(), dst.device.index, src.data_ptr(),
                              src.device.index, src.numel() * src.element_size(), self.stream.cuda_stream)
            if local:
                # the slot's memory belongs to the student's allocator: keep it
                # from being recycled while this stream may still write it
                # (a remote slot is held by the reader until slot.done, or
                # retired behind this stream if the teacher fails)
                slot.probs.record_stream(self.stream)
                slot.classes.record_stream(self.stream)
            slot.num_classes = self.model.num_classes
            slot.done = torch.cuda.Event()
            slot.done.record(self.stream)
        self.batches_served += 1

    def stop(self) -> None:
        """Abrupt stop, like a process kill: queued work is abandoned from the
        student's point of view (its replies are never accepted)."""
        self.alive = False
