"""Host-side data formats on either side of the hot path.

These reproduce, on the host, the reference's synthetic data, parameter
initialisation, sampling order and EDLD model file so that the device path
consumes exactly the inputs the reference would (same seeds -> same bits):

  init_model      edl/nnkit.py:211-220   seeded Glorot-uniform weights, zero biases
  make_blobs      edl/nnkit.py:371-388   Gaussian blobs, labels cycle 0..K-1
  partition       edl/nnkit.py:391-399   contiguous shard per rank
  epoch_order     edl/nnkit.py:402-405   per-(seed, epoch, rank) permutation
  serialize/deserialize_model  edl/nnkit.py:433-477  EDLD v1 (BE header, LE f64)

All arithmetic here is numpy float64 because it defines inputs, not compute;
the compute path is the sm_100a library.
"""

from __future__ import annotations

import hashlib
import struct
from dataclasses import dataclass, field

import numpy as np

MODEL_MAGIC = b"EDLD"
MODEL_FORMAT_VERSION = 1


class ModelFileError(ValueError):
    """Model file is corrupt, truncated, or not ours (edl/nnkit.py:39-40)."""


@dataclass(frozen=True)
class HostModel:
    """Parameter container in the reference layout: weights[l] is
    (dims[l+1], dims[l]) row-major float64, biases[l] has dims[l+1] entries."""

    layer_dims: tuple
    weights: tuple
    biases: tuple

    def num_params(self) -> int:
        return sum(w.size + b.size for w, b in zip(self.weights, self.biases))


@dataclass(frozen=True)
class Dataset:
    samples: np.ndarray   # N x D float64
    labels: np.ndarray    # N int64
    id: str = field(default="")

    def __post_init__(self):
        if self.samples.ndim != 2 or self.samples.shape[0] < 1:
            raise ValueError(f"samples must be a non-empty N x D matrix, got {self.samples.shape}")
        if self.labels.shape != (self.samples.shape[0],):
            raise ValueError("one label per sample required")
        if not self.id:
            object.__setattr__(self, "id", content_hash(self.samples, self.labels))

    @property
    def size(self) -> int:
        return self.samples.shape[0]

    @property
    def dim(self) -> int:
        return self.samples.shape[1]


def content_hash(samples: np.ndarray, labels: np.ndarray) -> str:
    """Dataset id used by checkpoints (edl/nnkit.py:181-186)."""
    h = hashlib.sha256()
    h.update(str(samples.shape).encode())
    h.update(np.ascontiguousarray(samples, dtype=np.float64).tobytes())
    h.update(np.ascontiguousarray(labels, dtype=np.int64).tobytes())
    return h.hexdigest()[:16]


def init_model(layer_dims, seed: int) -> HostModel:
    rng = np.random.Generator(np.random.PCG64(np.random.SeedSequence(seed)))
    dims = tuple(int(d) for d in layer_dims)
    ws, bs = [], []
    for l in range(len(dims) - 1):
        a = np.sqrt(6.0 / (dims[l] + dims[l + 1]))
        ws.append(rng.uniform(-a, a, size=(dims[l + 1], dims[l])))
        bs.append(np.zeros(dims[l + 1]))
    return HostModel(dims, tuple(ws), tuple(bs))


def make_blobs(seed: int, n_samples: int, dim: int, classes: int, spread: float) -> Dataset:
    if n_samples < 1 or dim < 1 or classes < 2:
        raise ValueError("need n_samples >= 1, dim >= 1, classes >= 2")
    if spread < 0:
        raise ValueError("spread must be >= 0")
    rng = np.random.Generator(np.random.PCG64(np.random.SeedSequence([seed, 0xB10B5])))
    centers = rng.normal(size=(classes, dim))
    centers *= 3.0 / np.linalg.norm(centers, axis=1, keepdims=True)
    labels = np.arange(n_samples, dtype=np.int64) % classes
    samples = centers[labels] + rng.normal(scale=spread, size=(n_samples, dim))
    return Dataset(samples, labels)


def partition(data: Dataset, world_size: int, rank: int) -> Dataset:
    if world_size < 1 or not 0 <= rank < world_size:
        raise ValueError(f"bad world_size={world_size} rank={rank}")
    n = data.size
    start, stop = (n * rank) // world_size, (n * (rank + 1)) // world_size
    return Dataset(data.samples[start:stop].copy(), data.labels[start:stop].copy())


def epoch_order(seed: int, epoch: int, rank: int, n: int) -> np.ndarray:
    ss = np.random.SeedSequence([seed, epoch, rank, 0x0A7A])
    return np.random.Generator(np.random.PCG64(ss)).permutation(n)


def serialize_model(model: HostModel, iteration: int = 0) -> bytes:
    if iteration < 0:
        raise ValueError("iteration must be >= 0")
    out = [MODEL_MAGIC, struct.pack(">I", MODEL_FORMAT_VERSION), struct.pack(">Q", iteration),
           struct.pack(">I", len(model.layer_dims))]
    out.extend(struct.pack(">I", d) for d in model.layer_dims)
    for w, b in zip(model.weights, model.biases):
        out.append(np.ascontiguousarray(w, dtype="<f8").tobytes())
        out.append(np.ascontiguousarray(b, dtype="<f8").tobytes())
    return b"".join(out)


def deserialize_model(blob: bytes) -> tuple[HostModel, int]:
    if len(blob) < 20 or blob[:4] != MODEL_MAGIC:
        raise ModelFileError("not a model file (bad magic or truncated header)")
    version = struct.unpack(">I", blob[4:8])[0]
    if version != MODEL_FORMAT_VERSION:
        raise ModelFileError(f"unsupported format version {version}")
    iteration = struct.unpack(">Q", blob[8:16])[0]
    ndims = struct.unpack(">I", blob[16:20])[0]
    off = 20
    if ndims < 2 or len(blob) < off + 4 * ndims:
        raise ModelFileError("truncated layer dim table")
    dims = struct.unpack(f">{ndims}I", blob[off:off + 4 * ndims])
    off += 4 * ndims
    ws, bs = [], []
    for l in range(ndims - 1):
        wn, bn = dims[l + 1] * dims[l], dims[l + 1]
        if len(blob) < off + 8 * (wn + bn):
            raise ModelFileError(f"truncated parameters at layer {l}")
        ws.append(np.frombuffer(blob, dtype="<f8", count=wn, offset=off).reshape(dims[l + 1], dims[l]).copy())
        off += 8 * wn
        bs.append(np.frombuffer(blob, dtype="<f8", count=bn, offset=off).copy())
        off += 8 * bn
    if off != len(blob):
        raise ModelFileError(f"{len(blob) - off} trailing bytes after parameters")
    if any(d < 1 for d in dims):
        raise ModelFileError("invalid parameters: non-positive layer dim")
    if not all(np.isfinite(w).all() and np.isfinite(b).all() for w, b in zip(ws, bs)):
        raise ModelFileError("invalid parameters: non-finite values")
    return HostModel(tuple(int(d) for d in dims), tuple(ws), tuple(bs)), iteration
