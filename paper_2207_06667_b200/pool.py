"""Teacher pool on dedicated GPUs feeding student GPUs over NVLink.

BASELINE.json configs[2] / SURVEY §8(e): a pool of teacher ranks produces
soft labels for the student ranks' batches; each batch's (prob, class) pairs
cross NVLink as one NCCL point-to-point transfer (teacher rank -> owning
student rank) on NCCL's side stream, straight into a slot of the student's
device ring. The student ranks run data-parallel SGD with the gradient
all-reduced over an NCCL group that contains students only, so teacher
churn never re-forms the student communicator.

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

from . import nnkit
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


def teacher_serve(pl: Placement, rank: int, model: Model, data: DeviceDataset, batch_size: int, seed: int,
                  temperature: float, k: int, start: int, end: int, depth: int = 4) -> int:
    """Teacher rank loop: infer its share of one student's iterations and
    isend each soft-label batch to that student. At most `depth` sends are
    outstanding (the student's ring bounds how far teachers run ahead)."""
    s = pl.student_of(rank)
    sampler = DeviceShardSampler(data, pl.n_students, s, batch_size, seed)
    B = batch_size
    ring = [SoftLabels(torch.empty(B, k, device=data.device), torch.empty(B, k, dtype=torch.int32,
                                                                          device=data.device), temperature)
            for _ in range(depth)]
    works: list = [None] * depth
    batch = Batch(torch.empty(B, data.samples.shape[1], dtype=torch.bfloat16, device=data.device),
                  torch.empty(B, dtype=torch.int64, device=data.device), data.dim)
    ws = nnkit.Workspace(model, B)
    served = 0
    for n, it in enumerate(pl.iterations_of(rank, s, start, end)):
        slot = n % depth
        if works[slot] is not None:
            for w in works[slot]:
                w.wait()        # the slot's previous transfer must have left
        gather_batch(data, sampler.rows_for(it), batch)
        out = nnkit.teacher_soft_labels(model, batch.inputs, temperature, k, out=ring[slot], ws=ws)
        works[slot] = [dist.isend(out.probs, s), dist.isend(out.classes, s)]
        served += 1
    for ws_ in works:
        for w in ws_ or []:
            w.wait()
    return served


class RemoteSoftLabels:
    """Student-side receive ring: irecv's posted `depth` iterations ahead from
    the serving teacher rank; consume(i) orders the current stream after the
    transfer (no host sync)."""

    def __init__(self, pl: Placement, rank: int, batch_size: int, k: int, temperature: float, device,
                 start: int, end: int, depth: int = 4):
        self.pl, self.rank, self.depth = pl, rank, depth
        self.T = temperature
        self.end = end
        B = batch_size
        self.slots = [SoftLabels(torch.empty(B, k, device=device), torch.empty(B, k, dtype=torch.int32,
                                                                               device=device), temperature)
                      for _ in range(depth)]
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
            src = self.pl.server(self.pl.student_index(self.rank), it)
            self.works[it] = [dist.irecv(self.slots[slot].probs, src), dist.irecv(self.slots[slot].classes, src)]
            self.next_post += 1

    def consume(self, iteration: int) -> SoftLabels:
        for w in self.works.pop(iteration):
            w.wait()            # stream-ordered wait (NCCL): no host block
        self.consumed += 1
        return self.slots[iteration % self.depth]

    def released(self, iteration: int) -> None:
        """Call after enqueuing the step that consumed `iteration`."""
        ev = torch.cuda.Event()
        ev.record()
        self.release[iteration % self.depth] = ev
        self._post_until(iteration + 1 + self.depth)
