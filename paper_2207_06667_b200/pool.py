"""Teacher pool on dedicated GPUs feeding student GPUs over NVLink.

BASELINE.json configs[2] / SURVEY §8(e): a pool of teacher ranks produces
soft labels for the student ranks' batches; each batch's packed (prob, class)
pairs cross NVLink straight into a slot of the student's device ring, either
by peer copy with stream-ordered READY / CREDIT flags (PeerSoftLabelRing, the
default: no NCCL, no host waits, no SM held while waiting) or as one NCCL
send/recv per batch (teacher_serve / RemoteSoftLabels without a ring). The
student ranks run data-parallel SGD with the gradient all-reduced over an
NCCL group that contains students only, so teacher churn never re-forms the
student communicator.

Requests need no wire message: every teacher rank holds a replica of the
HBM-resident dataset and of each student's ShardSampler (same seed, rank and
epoch permutation as edl/student_node.py:125-151), so "serve iteration i of
student s" fully determines the rows. The static assignment below is the
steady state of the reference's JSQ dispatch with equal-speed teachers
(edl/student_node.py:111-118): iteration i of student s goes to
teachers_of(s)[i % len(teachers_of(s))], where teachers_of(s) = the teacher
ranks t with t % n_students == s (static_schedule gives each student
ceil(n_teachers / n_students) or floor(...) of them).
"""

from __future__ import annotations

from dataclasses import dataclass

import torch
import torch.distributed as dist

from . import _lib, nnkit
from .data import DeviceDataset, DeviceShardSampler, gather_batch
from .nnkit import Batch, Model, SoftLabels


@dataclass(frozen=True)
class Placement:
    world: int
    n_teachers: int

    def __post_init__(self):
        if not 1 <= self.n_teachers < self.world:
            raise ValueError("need at least one teacher and one student rank")
        if self.n_teachers < self.world - self.n_teachers:
            raise ValueError("the teacher pool must be at least as large as the student set "
                             "(every student needs a teacher of its own)")

    @property
    def n_students(self) -> int:
        return self.world - self.n_teachers

    def is_student(self, rank: int) -> bool:
        return rank < self.n_students

    def student_index(self, rank: int) -> int:
        return rank

    def teacher_ranks_of(self, s: int) -> list[int]:
        return [self.n_students + t for t in range(self.n_teachers) if t % self.n_students == s]

    def student_of(self, teacher_rank: int) -> int:
        return (teacher_rank - self.n_students) % self.n_students

    def server(self, s: int, iteration: int) -> int:
        ts = self.teacher_ranks_of(s)
        return ts[iteration % len(ts)]

    def iterations_of(self, teacher_rank: int, s: int, start: int, end: int) -> list[int]:
        ts = self.teacher_ranks_of(s)
        k = ts.index(teacher_rank)
        return [i for i in range(start, end) if i % len(ts) == k]


def pair_groups(pl: Placement) -> dict:
    """One 2-rank process group per (student, teacher) pair. Every rank must
    call this, in the same order (new_group is collective). With eager NCCL
    initialisation, unbatched send/recv on the default group are serialised
    with every other op of that group: the student's receives from its
    teachers queued behind each other. Measured at 3T+1S, 12.3 M samples/s
    on the default group."""
    groups = {}
    for s in range(pl.n_students):
        for t in pl.teacher_ranks_of(s):
            groups[(s, t)] = dist.new_group([s, t])
    return groups


def wire_slot(batch_size: int, k: int, temperature: float, device) -> tuple[torch.Tensor, SoftLabels]:
    """One transfer per batch: (prob fp32, class int32)[B][k] packed as an
    int32 [2][B][k] buffer; the SoftLabels views alias it."""
    buf = torch.empty(2, batch_size, k, dtype=torch.int32, device=device)
    return buf, SoftLabels(buf[0].view(torch.float32), buf[1], temperature)


class PeerSoftLabelRing:
    """Teacher-pool -> student handoff over NVLink peer memory, no NCCL.

    Every rank allocates the same symmetric buffer (torch symmetric memory is
    the plumbing): `depth` slots of one packed batch (wire_slot layout). On a
    student it is the receive ring, on a teacher the staging area. Per-rank
    uint32 signal pad: READY[j] (student side) = 1 + the iteration whose batch
    sits in slot j; CREDIT[s] (teacher side) = iterations student s has
    consumed. For iteration `it` of student s, slot j = it % depth:

      teacher stream: wait CREDIT[s] >= it - depth + 1   (slot j free again)
                      infer into staging slot j
                      copy staging j -> student s's slot j (copy engine, NVLink)
                      write student s's READY[j] = it + 1
      student stream: wait READY[j] >= it + 1, run the step, then write
                      CREDIT[s] = it + 1 into each of its teachers' pads

    Waits and writes are stream-ordered (edl_stream_wait_geq /
    edl_stream_write_u32): no host blocking, and no SM is held while a batch
    is in flight. Iterations must increase across runs that share a ring.
    """

    CREDIT = 64          # pad word offset of the credit words (READY uses 0..depth-1)

    def __init__(self, pl: Placement, rank: int, batch_size: int, k: int, temperature: float, device,
                 depth: int = 4, group=None):
        import torch.distributed._symmetric_memory as symm
        if not 1 <= depth <= self.CREDIT:
            raise ValueError(f"depth must be in [1, {self.CREDIT}]")
        self.pl, self.rank, self.depth = pl, rank, depth
        self.B, self.k, self.T = batch_size, k, temperature
        self.words = 2 * batch_size * k
        group = group or dist.group.WORLD
        self.buf = symm.empty(depth * self.words, dtype=torch.int32, device=device)
        self.h = symm.rendezvous(self.buf, group.group_name)
        pad_words = int(self.h.signal_pad_size) // 4
        if self.CREDIT + pl.n_students > pad_words:
            raise ValueError("signal pad too small for the credit words")
        self.h.get_signal_pad(rank, (pad_words,), torch.int32).zero_()
        self.pads = [int(p) for p in self.h.signal_pad_ptrs]
        torch.cuda.synchronize(device)
        dist.barrier(group)

    @classmethod
    def local(cls, pl: Placement, batch_size: int, k: int, temperature: float, device, depth: int = 4,
              view_rank: int = 0) -> "PeerSoftLabelRing":
        """Every rank's ring slots and signal pad as separate buffers on ONE
        device, with the same flag protocol: the teacher and student loops run
        as two streams of one process (tests on a single GPU)."""
        self = cls.__new__(cls)
        self.pl, self.rank, self.depth = pl, view_rank, depth
        self.B, self.k, self.T = batch_size, k, temperature
        self.words = 2 * batch_size * k
        self._bufs = [torch.zeros(depth * self.words, dtype=torch.int32, device=device) for _ in range(pl.world)]
        self._pads = [torch.zeros(cls.CREDIT + pl.n_students, dtype=torch.int32, device=device)
                      for _ in range(pl.world)]
        self.buf = self._bufs[view_rank]
        self.h = None
        self.pads = [int(p.data_ptr()) for p in self._pads]
        return self

    def as_rank(self, rank: int) -> "PeerSoftLabelRing":
        """The same local ring seen from another rank (local rings only)."""
        other = object.__new__(type(self))
        other.__dict__.update(self.__dict__)
        other.rank, other.buf = rank, self._bufs[rank]
        return other

    def slot(self, j: int) -> tuple[torch.Tensor, SoftLabels]:
        buf = self.buf[j * self.words:(j + 1) * self.words].view(2, self.B, self.k)
        return buf, SoftLabels(buf[0].view(torch.float32), buf[1], self.T)

    def peer_slot(self, rank: int, j: int) -> torch.Tensor:
        if self.h is None:
            return self._bufs[rank][j * self.words:(j + 1) * self.words].view(2, self.B, self.k)
        return self.h.get_buffer(rank, (2, self.B, self.k), torch.int32, j * self.words)

    def pad(self, rank: int, word: int) -> int:
        return self.pads[rank] + 4 * word

    @staticmethod
    def _s(stream) -> int:
        return (stream or torch.cuda.current_stream()).cuda_stream

    # teacher side
    def teacher_put(self, s: int, it: int, staged, stream=None) -> None:
        """Copy the staged batch of iteration `it` (staging slot it % depth,
        already written on `stream`) into student s's ring and signal it."""
        j = it % self.depth
        self.peer_slot(s, j).copy_(staged, non_blocking=True)
        _lib.call("edl_stream_write_u32", self.pad(s, j), (it + 1) & 0xFFFFFFFF, self._s(stream))

    def teacher_wait_credit(self, s: int, it: int, stream=None) -> None:
        need = it - self.depth + 1
        if need > 0:
            _lib.call("edl_stream_wait_geq", self.pad(self.rank, self.CREDIT + s), need & 0xFFFFFFFF,
                      self._s(stream))

    # student side
    def student_take(self, it: int, stream=None) -> SoftLabels:
        j = it % self.depth
        _lib.call("edl_stream_wait_geq", self.pad(self.rank, j), (it + 1) & 0xFFFFFFFF, self._s(stream))
        return self.slot(j)[1]

    def student_release(self, it: int, stream=None) -> None:
        s = self.pl.student_index(self.rank)
        for t in self.pl.teacher_ranks_of(s):
            _lib.call("edl_stream_write_u32", self.pad(t, self.CREDIT + s), (it + 1) & 0xFFFFFFFF, self._s(stream))


def ring_server(pl: Placement, rank: int, model: Model, data: DeviceDataset, batch_size: int, seed: int,
                temperature: float, k: int, ring: PeerSoftLabelRing):
    """A teacher rank's per-iteration step for the peer ring: serve(it) waits
    (on the stream) for the slot's credit, gathers the batch, runs the fused
    head into the staging slot and puts it into the student's ring. All
    buffers are allocated here, up front: with stream-memory waits queued, a
    later allocation that synchronises the device could deadlock a process
    that also drives the consumer's stream."""
    s = pl.student_of(rank)
    sampler = DeviceShardSampler(data, pl.n_students, s, batch_size, seed)
    batch = Batch(torch.empty(batch_size, data.samples.shape[1], dtype=torch.bfloat16, device=data.device),
                  torch.empty(batch_size, dtype=torch.int64, device=data.device), data.dim)
    ws = nnkit.Workspace(model, batch_size)

    def serve(it: int) -> None:
        ring.teacher_wait_credit(s, it)            # staging + student slot it % depth are free
        gather_batch(data, sampler.rows_for(it), batch)
        staged, out = ring.slot(it % ring.depth)
        nnkit.teacher_soft_labels(model, batch.inputs, temperature, k, out=out, ws=ws)
        ring.teacher_put(s, it, staged)
    return serve


def teacher_serve(pl: Placement, rank: int, model: Model, data: DeviceDataset, batch_size: int, seed: int,
                  temperature: float, k: int, start: int, end: int, depth: int = 4,
                  groups: dict | None = None, ring: PeerSoftLabelRing | None = None) -> int:
    """Teacher rank loop: infer its share of one student's iterations and
    hand each soft-label batch to that student: over peer memory when a
    PeerSoftLabelRing is given, else as an NCCL isend (at most `depth`
    outstanding; the student's ring bounds how far teachers run ahead)."""
    s = pl.student_of(rank)
    if ring is not None:
        serve = ring_server(pl, rank, model, data, batch_size, seed, temperature, k, ring)
        served = 0
        for it in pl.iterations_of(rank, s, start, end):
            serve(it)
            served += 1
        return served
    group = groups.get((s, rank)) if groups else None
    sampler = DeviceShardSampler(data, pl.n_students, s, batch_size, seed)
    B = batch_size
    ring = [wire_slot(B, k, temperature, data.device) for _ in range(depth)]
    works: list = [None] * depth
    batch = Batch(torch.empty(B, data.samples.shape[1], dtype=torch.bfloat16, device=data.device),
                  torch.empty(B, dtype=torch.int64, device=data.device), data.dim)
    ws = nnkit.Workspace(model, B)
    served = 0
    for n, it in enumerate(pl.iterations_of(rank, s, start, end)):
        slot = n % depth
        if works[slot] is not None:
            works[slot].wait()          # the slot's previous transfer must have left
        gather_batch(data, sampler.rows_for(it), batch)
        buf, out = ring[slot]
        nnkit.teacher_soft_labels(model, batch.inputs, temperature, k, out=out, ws=ws)
        works[slot] = dist.isend(buf, s, group=group)
        served += 1
    for w in works:
        if w is not None:
            w.wait()
    return served


class RemoteSoftLabels:
    """Student-side receive ring: irecv's posted `depth` iterations ahead from
    the serving teacher rank; consume(i) orders the current stream after the
    transfer (no host sync)."""

    def __init__(self, pl: Placement, rank: int, batch_size: int, k: int, temperature: float, device,
                 start: int, end: int, depth: int = 4, groups: dict | None = None):
        self.pl, self.rank, self.depth = pl, rank, depth
        self.T = temperature
        self.end = end
        self.groups = groups
        wires = [wire_slot(batch_size, k, temperature, device) for _ in range(depth)]
        self.bufs = [w[0] for w in wires]
        self.slots = [w[1] for w in wires]
        self.works: dict[int, list] = {}
        self.release: list = [None] * depth
        self.next_post = start
        self.consumed = 0
        self._post_until(start + depth)

    def _post_until(self, limit: int) -> None:
        while self.next_post < min(limit, self.end):
            it = self.next_post
            slot = it % self.depth
            if self.release[slot] is not None:
                # the step that read this slot must be done before NCCL overwrites it
                torch.cuda.current_stream().wait_event(self.release[slot])
            s = self.pl.student_index(self.rank)
            src = self.pl.server(s, it)
            group = self.groups.get((s, src)) if self.groups else None
            self.works[it] = dist.irecv(self.bufs[slot], src, group=group)
            self.next_post += 1

    def consume(self, iteration: int) -> SoftLabels:
        self.works.pop(iteration).wait()   # stream-ordered wait (NCCL): no host block
        self.consumed += 1
        return self.slots[iteration % self.depth]

    def released(self, iteration: int) -> None:
        """Call after enqueuing the step that consumed `iteration`."""
        ev = torch.cuda.Event()
        ev.record()
        self.release[iteration % self.depth] = ev
        self._post_until(iteration + 1 + self.depth)


class PeerSoftLabels:
    """Student-side view of a PeerSoftLabelRing with RemoteSoftLabels'
    consume / released interface."""

    def __init__(self, ring: PeerSoftLabelRing):
        self.ring = ring

    def consume(self, iteration: int) -> SoftLabels:
        return self.ring.student_take(iteration)

    def released(self, iteration: int) -> None:
        self.ring.student_release(iteration)
