"""Student gradient exchange over NVSwitch multicast (NVLS), fused with SGD.

Reference (edl/student_node.py:738-745): with world > 1 every rank ring-
all-reduces its flat gradient to the mean (edl/allreduce.py:77-120) and then
runs sgd_step (edl/nnkit.py:312-322). Here `edl_nvls_allreduce_sgd` (csrc/
exchange.cu) does both in one kernel per rank: rank r sums shard r of every
rank's gradient inside the switch (multimem.ld_reduce), applies the update,
and multicasts the new fp32 master and bf16 weights into every replica.

torch.distributed's symmetric memory is the plumbing: one symmetric
allocation per rank holds [gradient | fp32 master | bf16 copy], and
rendezvous provides its multicast address and the per-rank signal pads the
kernel's barriers use. The model's and the workspace's flat buffers are
re-pointed into that allocation, so the GEMM kernels read and write it
directly and nothing is copied per step.
"""

from __future__ import annotations

import torch

from . import _lib
from .nnkit import Gradients, Model


class ExchangeUnavailable(RuntimeError):
    """No symmetric memory / NVLS multicast for this group (e.g. CPU gloo, or
    GPUs without an NVSwitch multicast object): the caller uses NCCL."""


class NvlsGradientExchange:
    def __init__(self, model: Model, grads: Gradients, group=None):
        import torch.distributed as dist
        try:
            import torch.distributed._symmetric_memory as symm
        except ImportError as ex:  # pragma: no cover - torch without symmetric memory
            raise ExchangeUnavailable(str(ex)) from ex
        group = group or dist.group.WORLD
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        if self.world < 2:
            raise ExchangeUnavailable("single rank: nothing to exchange")
        if model.device.type != "cuda":
            raise ExchangeUnavailable("NVLS exchange needs CUDA tensors")
        n = model.layout.size
        q = 8 * self.world
        self.n = (n + q - 1) // q * q        # padded: whole 8-element items per shard
        dev = model.device
        try:
            buf = symm.empty(2 * self.n + self.n // 2, dtype=torch.float32, device=dev)
            h = symm.rendezvous(buf, group.group_name)
        except Exception as ex:  # noqa: BLE001 - any failure here means "not on this box"
            raise ExchangeUnavailable(f"symmetric memory rendezvous failed: {ex}") from ex
        mc = int(getattr(h, "multicast_ptr", 0) or 0)
        if not mc:
            raise ExchangeUnavailable("no NVLS multicast address for this group")
        grad = buf[:self.n]
        param = buf[self.n:2 * self.n]
        bf16 = buf[2 * self.n:].view(torch.bfloat16)
        buf.zero_()
        param[:n].copy_(model.flat)
        bf16[:n].copy_(model.flat_bf16)
        model.flat = param[:n]
        model.flat_bf16 = bf16[:n]
        grads.flat = grad[:n]
        self.param = param
        self.mc_grad, self.mc_param, self.mc_bf16 = mc, mc + 4 * self.n, mc + 8 * self.n
        self.pad_bytes = int(h.signal_pad_size)
        self.pads = torch.tensor([int(p) for p in h.signal_pad_ptrs], dtype=torch.int64, device=dev)
        h.get_signal_pad(self.rank, (self.pad_bytes // 4,), torch.int32).zero_()
        self.counter = torch.zeros(1, dtype=torch.int32, device=dev)
        self.epoch = 0
        self._keep = (buf, h)
        torch.cuda.synchronize(dev)
        dist.barrier(group)

    def step(self, eta: float, stream=None) -> None:
        """Enqueue the fused exchange + SGD (p -= eta * mean_r(g_r)) on `stream`."""
        self.epoch += 1
        s = (stream or torch.cuda.current_stream()).cuda_stream
        _lib.call("edl_nvls_allreduce_sgd", self.mc_grad, self.mc_param, self.mc_bf16, self.param.data_ptr(),
                  self.pads.data_ptr(), self.pad_bytes, self.counter.data_ptr(), self.rank, self.world, self.n,
                  float(eta) / self.world, self.epoch & 0xFFFFFFFF, s)
