"""DistilReader on the device — mirror of edl/student_node.py:58-560.

Pure scheduling logic (`scheduler_tick`, `pick_teacher`, `static_schedule`,
`SchedulerConfig`) keeps the reference's semantics line for line. The buffer
changes representation: `_ready: dict[int, SoftLabelBatch]` of JSON-decoded
fp64 matrices becomes a student-owned ring of device slots, each holding one
batch's top-k (prob fp32, class int32) pairs plus two CUDA events:

  slot.done     recorded by the teacher after its head kernel (or after the
                NVLink peer copy when the teacher sits on another GPU);
  slot.release  recorded on the student stream after the step that consumed
                the slot; a teacher reusing the slot waits on it on-device.

A reply "arrives" when slot.done has completed (event query, never a host
sync on the hot path). The reader is driven by `pump()` from the training
thread (dispatch + arrival polling + the Alg. 1 probe), so no helper threads
contend for the GIL while kernels are being launched.

Fail-over keeps the reference's three cases (edl/student_node.py:492-523):
an unassigned teacher dying is invisible; an assigned teacher dying is
reported to the pool, replaced via acquire(1), and exactly its unanswered
iterations go back to the front of the pending queue; late replies from a
dead teacher are never accepted; duplicates are counted and dropped.
"""

from __future__ import annotations

import json
import math
import threading
import time
from collections import deque
from dataclasses import dataclass

import torch

from .nnkit import SoftLabels

STOP_SENDING = "STOP_SENDING"
RESUME_SENDING = "RESUME_SENDING"
REQUEST_ADDITIONAL_TEACHER = "REQUEST_ADDITIONAL_TEACHER"
NONE = "NONE"


# ---------------------------------------------------------------------------
# Pure scheduling logic (edl/student_node.py:62-118)


@dataclass(frozen=True)
class SchedulerConfig:
    lt: int = 4
    ut: int = 32
    n_static: int = 1
    acquire_cooldown: float = 2.0
    probe_interval: float = 0.1
    pipeline_depth: int = 2

    def __post_init__(self):
        if not 0 <= self.lt < self.ut:
            raise ValueError("need 0 <= lt < ut")
        if self.n_static < 1:
            raise ValueError("n_static must be >= 1")
        if self.pipeline_depth < 1:
            raise ValueError("pipeline_depth must be >= 1")


@dataclass(frozen=True)
class ThroughputProfile:
    t_s: float
    t_t: float

    def __post_init__(self):
        if self.t_s <= 0 or self.t_t <= 0:
            raise ValueError("throughputs must be positive")


def static_schedule(profile: ThroughputProfile) -> int:
    """Teachers per student: ceil(t_s / t_t), at least 1 (edl/student_node.py:90-96)."""
    return max(1, math.ceil(profile.t_s / profile.t_t))


def scheduler_tick(volume: int, sending_enabled: bool, cooldown_elapsed: bool,
                   cfg: SchedulerConfig) -> str:
    """Alg. 1 hysteresis, precedence stop > acquire > resume (edl/student_node.py:99-108)."""
    if volume > cfg.ut:
        return STOP_SENDING
    if volume == 0 and sending_enabled and cooldown_elapsed:
        return REQUEST_ADDITIONAL_TEACHER
    if volume < cfg.lt and not sending_enabled:
        return RESUME_SENDING
    return NONE


def pick_teacher(outstanding: dict, depth: int):
    """Join-shortest-queue, node-id tie break; None if all full (edl/student_node.py:111-118)."""
    best = None
    for node_id in sorted(outstanding):
        n = outstanding[node_id]
        if n < depth and (best is None or n < outstanding[best]):
            best = node_id
    return best


# ---------------------------------------------------------------------------
# Event log (edl/student_node.py:201-218)


class EventLog:
    def __init__(self, path: str | None = None):
        self._lock = threading.Lock()
        self._fh = open(path, "a", buffering=1) if path else None
        self.entries: list[dict] = []

    def append(self, kind: str, **fields) -> None:
        entry = {"event": kind, "ts": round(time.time(), 6), **fields}
        with self._lock:
            self.entries.append(entry)
            if self._fh:
                self._fh.write(json.dumps(entry, separators=(",", ":")) + "\n")

    def close(self) -> None:
        with self._lock:
            if self._fh:
                self._fh.close()
                self._fh = None


# ---------------------------------------------------------------------------
# In-process teacher pool with the Registry's acquire / release / failure
# semantics (edl/coordinator.py:99-197): exclusive assignment,
# longest-available-first, report_failure expires immediately.

AVAILABLE, ASSIGNED, EXPIRED = "AVAILABLE", "ASSIGNED", "EXPIRED"


class TeacherPool:
    def __init__(self):
        self._lock = threading.Lock()
        self._workers: dict = {}
        self._status: dict[str, str] = {}
        self._owner: dict = {}
        self._since: dict[str, int] = {}
        self._clock = 0
        self.events: list[dict] = []

    def _tick(self) -> int:
        self._clock += 1
        return self._clock

    def _transition(self, node_id: str, to: str, **detail) -> None:
        self.events.append({"seq": len(self.events) + 1, "node_id": node_id,
                            "from": self._status.get(node_id, "(none)"), "to": to, **detail})
        self._status[node_id] = to

    def register(self, worker) -> None:
        with self._lock:
            nid = worker.node_id
            if self._status.get(nid) in (AVAILABLE, ASSIGNED) and self._workers[nid] is not worker:
                raise ValueError(f"{nid} is live; refusing a second registration")
            self._workers[nid] = worker
            self._owner[nid] = None
            self._since[nid] = self._tick()
            self._transition(nid, AVAILABLE)

    def acquire_teachers(self, student_id: str, count: int) -> list:
        if count < 1:
            raise ValueError("count must be >= 1")
        with self._lock:
            free = sorted((nid for nid, st in self._status.items()
                           if st == AVAILABLE and self._workers[nid].alive),
                          key=lambda n: (self._since[n], n))
            granted = []
            for nid in free[:count]:
                self._owner[nid] = student_id
                self._transition(nid, ASSIGNED, student_id=student_id)
                granted.append(self._workers[nid])
            return granted

    def release_teacher(self, student_id: str, node_id: str) -> None:
        with self._lock:
            if self._status.get(node_id) != ASSIGNED or self._owner.get(node_id) != student_id:
                raise ValueError(f"{node_id} is not assigned to {student_id}")
            self._owner[node_id] = None
            self._since[node_id] = self._tick()
            self._transition(node_id, AVAILABLE, released_by=student_id)

    def report_failure(self, student_id: str, node_id: str) -> None:
        with self._lock:
            if node_id not in self._status:
                raise ValueError(f"{node_id} unknown")
            if self._status[node_id] != EXPIRED:
                self._owner[node_id] = None
                self._transition(node_id, EXPIRED, cause="reported", reported_by=student_id)

    def kill(self, node_id: str) -> None:
        """Fault injection: the worker dies abruptly (SIGKILL analogue)."""
        with self._lock:
            w = self._workers.get(node_id)
        if w is not None:
            w.stop()

    def status(self, node_id: str) -> str | None:
        with self._lock:
            return self._status.get(node_id)


# ---------------------------------------------------------------------------
# The reader


class _Slot:
    __slots__ = ("probs", "classes", "done", "release", "iteration", "teacher", "batch", "batch_filled",
                 "num_classes", "index")

    def __init__(self, B: int, k: int, device, batch=None):
        self.probs = torch.empty(B, k, dtype=torch.float32, device=device)
        self.classes = torch.empty(B, k, dtype=torch.int32, device=device)
        self.done: torch.cuda.Event | None = None
        self.release: torch.cuda.Event | None = None
        self.iteration = -1
        self.teacher = None
        self.batch = batch              # input buffers a same-device teacher gathers into
        self.batch_filled = False
        self.num_classes = None         # the producing teacher's head width
        self.index = -1                 # position in a fixed (IPC-exported) ring, elastic.SlotRing


class _TeacherHandle:
    def __init__(self, worker):
        self.worker = worker
        self.node_id = worker.node_id
        self.outstanding: dict[int, _Slot] = {}
        self.dead = False


class DistilReader:
    """Soft-label acquisition pipeline for one student (device buffer)."""

    def __init__(self, student_id: str, pool: TeacherPool, cfg: SchedulerConfig, sampler,
                 start_iteration: int, end_iteration: int, session: int, events: EventLog,
                 expected_temperature: float, k: int, clock=None, share_batch: bool = True):
        self.student_id = student_id
        self.pool = pool
        self.cfg = cfg
        self.sampler = sampler
        self.session = session
        self.events = events
        self.expected_temperature = expected_temperature
        self.k = k
        self.clock = clock or time.monotonic
        self.device = sampler.data.device
        # slots carry input buffers a same-device teacher gathers into, so the
        # student trains on them instead of gathering the rows a second time
        self.share_batch = share_batch and hasattr(getattr(sampler, "data", None), "samples")
        self._teachers: dict[str, _TeacherHandle] = {}
        self._ready: dict[int, _Slot] = {}
        self._free: list[_Slot] = []
        # a pool of teacher PROCESSES (elastic.ElasticPool) hands out slots of
        # the student's IPC-exported ring; in-process teachers get lazily
        # allocated slots
        source = getattr(pool, "slot_source", None)
        self._ring = source() if source is not None else None
        if self._ring is not None:
            self._free = list(self._ring.slots)
        # slots a failed teacher may still write (its queued kernels / copies):
        # (slot, event recorded on that teacher's stream at failure time);
        # recycled only once the event has completed
        self._retired: list[tuple[_Slot, torch.cuda.Event | None]] = []
        self._pending: deque[int] = deque()
        self._waiting_for: int | None = None    # the iteration consume() is blocked on
        self._next_new = start_iteration
        self._end = end_iteration
        self._consumed: set[int] = set()
        self._last_consumed: _Slot | None = None
        self.sending_enabled = True
        self._last_acquire = -float("inf")
        self._last_probe = -float("inf")
        self._stopped = False
        self.max_volume_seen = 0
        self.max_teachers_seen = 0
        self.dispatch_count: dict[int, int] = {}
        self.consume_count: dict[int, int] = {}
        self.duplicate_replies = 0
        self.reply_times: list[float] = []
        self.started_at = self.clock()

    # -- metrics -----------------------------------------------------------
    @property
    def volume(self) -> int:
        return len(self._ready)

    @property
    def teacher_count(self) -> int:
        return sum(1 for h in self._teachers.values() if not h.dead)

    def in_flight_capacity(self) -> int:
        return self.cfg.pipeline_depth * max(self.max_teachers_seen, 1)

    # -- pool calls ----------------------------------------------------------
    def acquire(self, count: int) -> int:
        self._last_acquire = self.clock()
        added = 0
        for w in self.pool.acquire_teachers(self.student_id, count):
            self._teachers[w.node_id] = _TeacherHandle(w)
            self.max_teachers_seen = max(self.max_teachers_seen, self.teacher_count)
            self.events.append("teacher_added", node=w.node_id)
            added += 1
        return added

    # -- dispatch ------------------------------------------------------------
    def _have_work(self) -> bool:
        return bool(self._pending) or self._next_new < self._end

    def _take_next_iteration(self) -> int:
        if self._pending:
            return self._pending.popleft()
        it = self._next_new
        self._next_new += 1
        return it

    def _slot(self) -> _Slot | None:
        if self._retired:
            keep = []
            for slot, ev in self._retired:
                if ev is None or ev.query():
                    slot.done = None
                    self._free.append(slot)
                else:
                    keep.append((slot, ev))
            self._retired = keep
        if self._ring is not None:
            # fixed ring: a slot goes back to a teacher only once the step
            # that read it has completed (its release event), because a remote
            # teacher cannot order its stream after ours
            for i, slot in enumerate(self._free):
                if slot.release is None or slot.release.query():
                    slot.release = None
                    slot.batch_filled = False
                    return self._free.pop(i)
            return None
        if self._free:
            slot = self._free.pop()
        else:
            batch = None
            if self.share_batch:
                from .nnkit import Batch
                data = self.sampler.data
                B = self.sampler.batch_size
                batch = Batch(torch.empty(B, data.samples.shape[1], dtype=torch.bfloat16, device=self.device),
                              torch.empty(B, dtype=torch.int64, device=self.device), data.dim)
            slot = _Slot(self.sampler.batch_size, self.k, self.device, batch)
        slot.batch_filled = False
        return slot

    def _demanded(self) -> bool:
        """The consumer is blocked on an iteration that nobody is computing: a
        failed teacher's unanswered batch, re-queued at the head of _pending.
        Alg. 1's hysteresis may have stopped sending (the buffer holds the
        LATER iterations that did arrive), and the buffer cannot drain past the
        missing one, so that one batch is dispatched regardless (the reference,
        edl/student_node.py:351-376, waits for the volume to drain and hangs in
        this case; the iteration ledger is unchanged)."""
        return self._waiting_for is not None and bool(self._pending) and self._pending[0] == self._waiting_for

    def _dispatch(self) -> None:
        while not self._stopped and self._have_work() and (self.sending_enabled or self._demanded()):
            out = {nid: len(h.outstanding) for nid, h in self._teachers.items() if not h.dead}
            target = pick_teacher(out, self.cfg.pipeline_depth)
            if target is None:
                return
            slot = self._slot()
            if slot is None:
                return          # every ring slot is in flight or still being read
            it = self._take_next_iteration()
            handle = self._teachers[target]
            slot.iteration, slot.teacher = it, target
            self.dispatch_count[it] = self.dispatch_count.get(it, 0) + 1
            rows = self.sampler.rows_for(it) if getattr(handle.worker, "needs_rows", True) else None
            try:
                handle.worker.submit(rows, slot)
            except RuntimeError:
                self._pending.appendleft(it)
                self._free.append(slot)
                self.handle_teacher_failure(target, "send")
                continue
            handle.outstanding[it] = slot

    # -- arrivals ------------------------------------------------------------
    def _poll(self) -> None:
        for nid, h in list(self._teachers.items()):
            if not h.worker.alive and not h.dead:
                self.handle_teacher_failure(nid, "recv")
                continue
            for it, slot in list(h.outstanding.items()):
                if slot.done is not None and slot.done.query():
                    del h.outstanding[it]
                    self._accept(it, slot)

    def _accept(self, it: int, slot: _Slot) -> None:
        if it in self._consumed or it in self._ready:
            self.duplicate_replies += 1   # re-dispatch answered twice
            self._free.append(slot)
            return
        self._ready[it] = slot
        self.reply_times.append(self.clock())
        self.max_volume_seen = max(self.max_volume_seen, self.volume)
        self._apply_tick()

    # -- scheduler -----------------------------------------------------------
    def _cooldown_elapsed(self) -> bool:
        return self.clock() - self._last_acquire >= self.cfg.acquire_cooldown

    def _apply_tick(self) -> str:
        action = scheduler_tick(self.volume, self.sending_enabled, self._cooldown_elapsed(), self.cfg)
        if action == STOP_SENDING and self.sending_enabled:
            self.sending_enabled = False
            self.events.append("stop_sending", volume=self.volume)
        elif action == RESUME_SENDING:
            self.sending_enabled = True
            self.events.append("resume_sending", volume=self.volume)
        return action

    def _probe(self) -> None:
        now = self.clock()
        if now - self._last_probe < self.cfg.probe_interval:
            return
        self._last_probe = now
        action = self._apply_tick()
        if action == REQUEST_ADDITIONAL_TEACHER and self._have_work():
            self.events.append("request_additional_teacher")
            self.acquire(1)

    def pump(self) -> None:
        """One non-blocking pass: arrivals, probe (Alg. 1), dispatch."""
        if self._stopped:
            return
        self._poll()
        self._probe()
        self._dispatch()

    # -- consume -------------------------------------------------------------
    def consume(self, iteration: int, timeout: float | None = None,
                stream: torch.cuda.Stream | None = None) -> SoftLabels:
        """Block until `iteration`'s soft labels are buffered, take them, and
        order `stream` after their arrival. The previously consumed slot is
        released once the work enqueued so far on `stream` completes."""
        stream = stream or torch.cuda.current_stream(self.device)
        deadline = None if timeout is None else time.monotonic() + timeout
        if self._last_consumed is not None:
            ev = torch.cuda.Event()
            ev.record(stream)
            self._last_consumed.release = ev
            self._free.append(self._last_consumed)
            self._last_consumed = None
        self.pump()
        self._waiting_for = iteration
        try:
            while iteration not in self._ready:
                if self._stopped:
                    raise RuntimeError("reader stopped while waiting for soft labels")
                if deadline is not None and time.monotonic() > deadline:
                    raise TimeoutError(f"no soft labels for iteration {iteration}")
                slot = self._inflight_slot(iteration)
                if slot is not None and slot.done is not None:
                    slot.done.synchronize()     # blocking wait only when the buffer is empty
                else:
                    time.sleep(0.0002)
                self.pump()
        finally:
            self._waiting_for = None
        slot = self._ready.pop(iteration)
        self._consumed.add(iteration)
        self.consume_count[iteration] = self.consume_count.get(iteration, 0) + 1
        self._apply_tick()
        if isinstance(slot.done, torch.cuda.Event):
            stream.wait_event(slot.done)
        # (a remote reply, elastic.HostFlag, is complete in memory once seen)
        self._last_consumed = slot
        self.pump()
        return SoftLabels(slot.probs, slot.classes, self.expected_temperature,
                          slot.batch if slot.batch_filled else None, slot.num_classes)

    def _inflight_slot(self, iteration: int):
        for h in self._teachers.values():
            if not h.dead and iteration in h.outstanding:
                return h.outstanding[iteration]
        return None

    # -- failures --------------------------------------------------------------
    def handle_teacher_failure(self, node_id: str, context: str) -> None:
        h = self._teachers.get(node_id)
        if h is None or h.dead:
            return
        h.dead = True
        del self._teachers[node_id]
        unanswered = sorted(h.outstanding)
        for it in reversed(unanswered):
            self._pending.appendleft(it)
        # slots of a dead teacher may still be written by its queued kernels
        # or peer copies: retire them behind an event on its stream (recycled
        # once everything it had queued has drained; never, if it is hung)
        drained = None
        stream = getattr(h.worker, "stream", None)
        if hasattr(h.worker, "drain_marker"):
            drained = h.worker.drain_marker()       # a teacher process: until it has exited
        elif isinstance(stream, torch.cuda.Stream):
            drained = torch.cuda.Event()
            drained.record(stream)
        for slot in h.outstanding.values():
            self._retired.append((slot, drained))
        h.outstanding.clear()
        self.events.append("teacher_failure", node=node_id, context=context, unanswered=unanswered,
                           why=getattr(h.worker, "failure", None))
        if self._stopped:
            return
        try:
            self.pool.report_failure(self.student_id, node_id)
        except ValueError:
            pass
        replaced = self.acquire(1)
        self.events.append("teacher_replaced" if replaced else "no_replacement", node=node_id)

    # -- lifecycle -------------------------------------------------------------
    def start(self) -> None:
        self.pump()

    def ledger(self) -> dict:
        consumed_once = all(v == 1 for v in self.consume_count.values())
        dispatched = all(it in self.dispatch_count for it in self.consume_count)
        return {
            "consumed": len(self.consume_count),
            "dispatched": len(self.dispatch_count),
            "redispatches": sum(v - 1 for v in self.dispatch_count.values() if v > 1),
            "duplicate_replies": self.duplicate_replies,
            "ok": consumed_once and dispatched,
        }

    def close(self, release: bool = True) -> None:
        self._stopped = True
        for h in list(self._teachers.values()):
            if release and not h.dead:
                try:
                    self.pool.release_teacher(self.student_id, h.node_id)
                except ValueError:
                    pass
        self._teachers.clear()
