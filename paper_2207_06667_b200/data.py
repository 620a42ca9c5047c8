"""HBM-resident dataset and the device ShardSampler.

The reference ships every batch's B x D inputs through JSON (INFER_REQUEST,
edl/student_node.py:369-372), which caps B. Here the dataset is
uploaded once as bf16 rows padded to a multiple of 16 and both the student and
its teachers read batches by row index (the paper's own future-work item).

DeviceShardSampler mirrors ShardSampler (edl/student_node.py:125-151): the
same contiguous shard (edl/nnkit.py:391-399), the same per-epoch permutation
(edl/nnkit.py:402-405) and the same equal batches-per-epoch across ranks, so
batch_for(it) selects exactly the rows the reference would.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib
from .formats import Dataset, epoch_order
from .nnkit import Batch, img_pad, pad


class DeviceDataset:
    def __init__(self, data: Dataset, device=None, chunk_rows: int = 65536):
        self.id = data.id
        self.size = data.size
        self.dim = data.dim
        self.classes = int(data.labels.max()) + 1
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.samples = torch.zeros(self.size, pad(self.dim), dtype=torch.bfloat16, device=self.device)
        for lo in range(0, self.size, chunk_rows):
            hi = min(lo + chunk_rows, self.size)
            blk = torch.from_numpy(np.ascontiguousarray(data.samples[lo:hi], dtype=np.float32))
            self.samples[lo:hi, :self.dim] = blk.to(self.device).to(torch.bfloat16)
        self.labels = torch.from_numpy(np.ascontiguousarray(data.labels, dtype=np.int64)).to(self.device)


class DeviceImageDataset:
    """cfg4's synthetic image set, HBM-resident: n NHWC bf16 images
    [image][image][img_pad(channels)] stored as rows of one [n][image*image*img_pad(c)]
    matrix (so DeviceShardSampler / gather_rows select batches by row index,
    as for the MLP datasets) + int64 labels. Deterministic in (seed, n,
    image, classes): every teacher and student process builds the same set."""

    def __init__(self, seed: int, n: int, image: int = 224, classes: int = 1000, channels: int = 3,
                 device=None, chunk: int = 64):
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.image, self.channels, self.classes = image, channels, classes
        self.cp = img_pad(channels)
        self.size = n
        self.dim = image * image * self.cp
        self.id = f"images-{seed}-{n}-{image}-{classes}"
        self.samples = torch.zeros(n, self.dim, dtype=torch.bfloat16, device=self.device)
        rng = np.random.default_rng(seed)
        view = self.samples.view(n, image, image, self.cp)
        for lo in range(0, n, chunk):
            hi = min(lo + chunk, n)
            imgs = rng.standard_normal(size=(hi - lo, image, image, channels), dtype=np.float32)
            view[lo:hi, :, :, :channels] = torch.from_numpy(imgs).to(self.device).to(torch.bfloat16)
        self.labels = torch.from_numpy(rng.integers(0, classes, size=n).astype(np.int64)).to(self.device)

    def nhwc(self, rows_view: torch.Tensor) -> torch.Tensor:
        """A gathered [B][dim] batch as NHWC [B][image][image][img_pad(c)]."""
        return rows_view.view(rows_view.shape[0], self.image, self.image, self.cp)


class DeviceShardSampler:
    """batch_for(iteration) -> Batch gathered on the device from the shard."""

    def __init__(self, data: DeviceDataset, world_size: int, rank: int, batch_size: int, seed: int):
        if world_size < 1 or not 0 <= rank < world_size:
            raise ValueError(f"bad world_size={world_size} rank={rank}")
        n = data.size
        self.data = data
        self.lo, self.hi = (n * rank) // world_size, (n * (rank + 1)) // world_size
        self.batch_size = batch_size
        self.seed = seed
        self.rank = rank
        self.batches_per_epoch = (n // world_size) // batch_size
        if self.batches_per_epoch < 1:
            raise ValueError("shard smaller than one batch")
        self._orders: dict[int, tuple] = {}
        self._copy_stream = torch.cuda.Stream(data.device)

    # Epoch permutations are uploaded on a private copy stream one epoch
    # ahead. Their readers are gathers on several streams (the student's, each
    # teacher worker's), so the upload must be complete before any of them is
    # enqueued: rows_for waits on the upload's event on the host, which costs
    # nothing because it was issued an epoch earlier. (An upload on the
    # caller's stream left teacher-stream gathers racing it.)
    _KEEP = 4   # epochs kept: the current one, two behind (in-flight readers), one ahead

    def _upload(self, epoch: int) -> None:
        host = torch.from_numpy((epoch_order(self.seed, epoch, self.rank, self.hi - self.lo)
                                 + self.lo).astype(np.int64)).pin_memory()
        with torch.cuda.stream(self._copy_stream):
            order = host.to(self.data.device, non_blocking=True)
            done = torch.cuda.Event()
            done.record(self._copy_stream)
        self._orders[epoch] = (order, host, done)

    def rows_for(self, iteration: int) -> torch.Tensor:
        """Global dataset row indices (device int64 [B]) of batch `iteration`."""
        epoch, i = divmod(iteration, self.batches_per_epoch)
        if epoch not in self._orders:
            self._upload(epoch)
        order, _, done = self._orders[epoch]
        done.synchronize()
        if epoch + 1 not in self._orders:
            self._upload(epoch + 1)
        while len(self._orders) > self._KEEP:   # drop the epoch farthest from the current one
            self._orders.pop(max(self._orders, key=lambda e: (abs(e - epoch), e)))
        return order[i * self.batch_size:(i + 1) * self.batch_size]

    def batch_for(self, iteration: int, out: Batch | None = None, stream=None) -> Batch:
        rows = self.rows_for(iteration)
        return gather_batch(self.data, rows, out, stream)


def gather_batch(data: DeviceDataset, rows: torch.Tensor, out: Batch | None = None, stream=None) -> Batch:
    B = rows.shape[0]
    if out is None:
        out = Batch(torch.empty(B, data.samples.shape[1], dtype=torch.bfloat16, device=data.device),
                    torch.empty(B, dtype=torch.int64, device=data.device), data.dim)
    st = stream or torch.cuda.current_stream(data.device)
    s = st.cuda_stream
    # the epoch-order tensor `rows` views was allocated on the sampler's copy
    # stream: keep its block from being recycled while this gather may run
    rows.record_stream(st)
    _lib.call("edl_gather_rows", data.samples.data_ptr(), data.samples.stride(0), rows.data_ptr(),
              out.inputs.data_ptr(), out.inputs.stride(0), B, data.samples.shape[1],
              data.labels.data_ptr(), out.hard_labels.data_ptr(), s)
    return out
