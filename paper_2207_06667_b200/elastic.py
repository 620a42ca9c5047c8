"""Elastic teacher pool across processes on one box (BASELINE configs[2] and
configs[4]).

The reference runs teachers as separate processes that register with a
coordinator (edl/coordinator.py:99-197), are acquired exclusively by a
student (longest-available-first), receive INFER_REQUESTs over TCP and answer
with INFER_REPLYs (edl/student_node.py:351-457, edl/teacher_node.py:157-170);
a student that loses a teacher reports it, acquires a replacement and
re-dispatches exactly the unanswered iterations (edl/student_node.py:492-523).

Here the same roles and semantics run over two planes:

* control plane — one shared-memory block (/dev/shm, `ControlBlock`): the
  registry (teacher entries with state, pid, epoch, heartbeat, owner), one
  request mailbox per teacher and one section per student (its slot ring's
  CUDA IPC handle, sampler parameters and a READY word per slot). Registry
  transitions take an flock, like the coordinator's lock.
* data plane — device memory only: the student owns a ring of soft-label
  slots and exports it over CUDA IPC; a teacher gathers the iteration's rows
  from its HBM replica of the dataset (replicated ShardSampler), runs the
  fused head with the student's slot as the output (a peer write over NVLink
  when the student sits on another GPU) and then, on the same stream,
  writes the dispatch's tag into the slot's READY word in the host-mapped
  block (edl_stream_write_u32, system-scope fence first).

The student's DistilReader (reader.py) drives remote teachers through
`RemoteTeacher` proxies with the TeacherWorker interface, so JSQ, Alg. 1 and
the fail-over code are the in-process ones. Nothing on the student's stream
ever waits for a teacher: a reply is accepted when the host sees its tag, so
a teacher that dies can delay soft labels but never hang a student stream.
Failure detection (the watchdog): the teacher's pid is gone (SIGKILL), its
heartbeat is older than `ttl`, or a dispatch is older than `reply_timeout`.
Tags are unique per dispatch, a failed teacher's entry is revoked (epoch
bump) and its slots are quarantined until its process has exited, so a late
write can neither be accepted nor land in a re-dispatched slot.
"""

from __future__ import annotations

import argparse
import contextlib
import ctypes
import fcntl
import mmap
import os
import signal
import sys
import time

import numpy as np
import torch

from . import _lib

MAGIC = 0x45444C50            # "EDLP"
VERSION = 1
FREE, AVAILABLE, ASSIGNED, EXPIRED = 0, 1, 2, 3
STATE_NAMES = {FREE: "FREE", AVAILABLE: "AVAILABLE", ASSIGNED: "ASSIGNED", EXPIRED: "EXPIRED"}
NO_OWNER = 0xFFFFFFFF
CLOSED, OPEN = 0, 1

HEADER = np.dtype([("magic", "<u4"), ("version", "<u4"), ("max_students", "<u4"), ("max_teachers", "<u4"),
                   ("max_slots", "<u4"), ("ring_len", "<u4"), ("shutdown", "<u4"), ("clock", "<u4"),
                   ("created_ns", "<u8")])
STUDENT = lambda max_slots: np.dtype([  # noqa: E731
    ("state", "<u4"), ("pid", "<u4"), ("rank", "<u4"), ("world", "<u4"), ("batch", "<u4"), ("k", "<u4"),
    ("n_slots", "<u4"), ("seed", "<u4"), ("temperature", "<f4"), ("num_classes", "<u4"),
    ("ring_offset", "<u8"), ("slot_bytes", "<u8"), ("generation", "<u8"),
    ("ipc", "u1", (64,)), ("ready", "<u4", (max_slots,))])
REQUEST = np.dtype([("seq", "<u8"), ("iteration", "<u8"), ("student", "<u4"), ("slot", "<u4"), ("tag", "<u4"),
                    ("pad", "<u4")])
TEACHER = lambda ring_len: np.dtype([  # noqa: E731
    ("state", "<u4"), ("pid", "<u4"), ("epoch", "<u4"), ("owner", "<u4"), ("heartbeat_ns", "<u8"),
    ("since", "<u8"), ("head", "<u8"), ("tail", "<u8"), ("served", "<u8"), ("node_id", "S32"),
    ("mailbox", REQUEST, (ring_len,))])


def _align(n: int, a: int = 4096) -> int:
    return (n + a - 1) // a * a


def pid_alive(pid: int) -> bool:
    """True while the process exists and is not a zombie (a SIGKILLed child
    that its parent has not reaped yet still answers kill(pid, 0))."""
    if pid <= 0:
        return False
    try:
        os.kill(pid, 0)
    except ProcessLookupError:
        return False
    except PermissionError:
        return True
    try:
        with open(f"/proc/{pid}/stat", "rb") as fh:
            stat = fh.read()
        return stat[stat.rindex(b")") + 2:stat.rindex(b")") + 3] not in (b"Z", b"X")
    except (OSError, ValueError):
        return False


class ControlBlock:
    """The pool's shared-memory block: header | students[S] | teachers[T]."""

    def __init__(self, path: str, create: bool = False, max_students: int = 8, max_teachers: int = 32,
                 max_slots: int = 128, ring_len: int = 64):
        self.path = path
        if create:
            fd = os.open(path, os.O_RDWR | os.O_CREAT | os.O_EXCL, 0o600)
            sd, td = STUDENT(max_slots), TEACHER(ring_len)
            size = _align(HEADER.itemsize) + _align(sd.itemsize * max_students) + _align(td.itemsize * max_teachers)
            os.ftruncate(fd, size)
            mm = mmap.mmap(fd, size)
            hdr = np.frombuffer(mm, HEADER, 1, 0)[0:1]
            hdr["max_students"], hdr["max_teachers"] = max_students, max_teachers
            hdr["max_slots"], hdr["ring_len"] = max_slots, ring_len
            hdr["created_ns"] = time.monotonic_ns()
            hdr["version"] = VERSION
            hdr["magic"] = MAGIC          # last: attachers wait for it
        else:
            fd = os.open(path, os.O_RDWR)
            size = os.fstat(fd).st_size
            mm = mmap.mmap(fd, size)
            hdr = np.frombuffer(mm, HEADER, 1, 0)[0:1]
            deadline = time.monotonic() + 30
            while int(hdr["magic"][0]) != MAGIC:
                if time.monotonic() > deadline:
                    raise RuntimeError(f"{path}: not an EDL pool control block")
                time.sleep(0.01)
            if int(hdr["version"][0]) != VERSION:
                raise RuntimeError(f"{path}: control block version {int(hdr['version'][0])} != {VERSION}")
        self.fd, self.mm, self.size = fd, mm, size
        self.hdr = hdr
        S, T = int(hdr["max_students"][0]), int(hdr["max_teachers"][0])
        self.max_slots, self.ring_len = int(hdr["max_slots"][0]), int(hdr["ring_len"][0])
        off = _align(HEADER.itemsize)
        self.students = np.frombuffer(mm, STUDENT(self.max_slots), S, off)
        off += _align(self.students.nbytes)
        self.teachers = np.frombuffer(mm, TEACHER(self.ring_len), T, off)
        self._dev_base = None      # device address of the block (host-registered) in this process
        self._anchor = ctypes.c_char.from_buffer(mm)
        self.host_base = ctypes.addressof(self._anchor)

    # -- addresses ------------------------------------------------------------
    def device_base(self) -> int:
        """Map the block for device writes (READY tags) once per process."""
        if self._dev_base is None:
            dev = ctypes.c_void_p()
            _lib.call("edl_host_register", self.host_base, self.size, ctypes.byref(dev))
            self._dev_base = int(dev.value)
        return self._dev_base

    def ready_offset(self, s: int, slot: int) -> int:
        field = self.students.dtype.fields["ready"][1]
        return (self.students.ctypes.data - self.host_base) + s * self.students.itemsize + field + 4 * slot

    # -- locking / clock --------------------------------------------------------
    @contextlib.contextmanager
    def locked(self):
        fcntl.flock(self.fd, fcntl.LOCK_EX)
        try:
            yield
        finally:
            fcntl.flock(self.fd, fcntl.LOCK_UN)

    def tick(self) -> int:
        """Registry clock (under the lock): orders available-since stamps."""
        self.hdr["clock"] += 1
        return int(self.hdr["clock"][0])

    @property
    def shutdown(self) -> bool:
        return bool(self.hdr["shutdown"][0])

    def request_shutdown(self) -> None:
        self.hdr["shutdown"] = 1

    def close(self) -> None:
        if self._dev_base is not None:
            with contextlib.suppress(Exception):
                _lib.call("edl_host_unregister", self.host_base)
            self._dev_base = None
        # numpy / ctypes views pin the buffer; drop them before the map goes away
        self.hdr = self.students = self.teachers = self._anchor = None
        with contextlib.suppress(BufferError):
            self.mm.close()
        os.close(self.fd)

    # -- registry (edl/coordinator.py:99-197) -----------------------------------
    def register_teacher(self, node_id: str, pid: int) -> tuple[int, int]:
        """A teacher joins: reuse its own expired entry (same node id) or a
        free / expired one; epoch + 1 revokes whatever ran there before."""
        with self.locked():
            t = self.teachers
            names = [bytes(n).rstrip(b"\0").decode() for n in t["node_id"]]
            live = [j for j in range(len(t)) if names[j] == node_id and t["state"][j] in (AVAILABLE, ASSIGNED)]
            if live and pid_alive(int(t["pid"][live[0]])):
                raise ValueError(f"{node_id} is live; refusing a second registration")
            cands = [j for j in range(len(t)) if names[j] == node_id] + \
                    [j for j in range(len(t)) if t["state"][j] == FREE] + \
                    [j for j in range(len(t)) if t["state"][j] == EXPIRED]
            if not cands:
                raise RuntimeError("teacher table full")
            j = cands[0]
            e = t[j:j + 1]
            e["epoch"] += 1
            e["pid"], e["owner"] = pid, NO_OWNER
            e["head"], e["tail"], e["served"] = 0, 0, 0
            e["node_id"] = node_id.encode()[:32]
            e["heartbeat_ns"] = time.monotonic_ns()
            e["since"] = self.tick()
            e["state"] = AVAILABLE
            return j, int(e["epoch"][0])

    def teacher_status(self, node_id: str) -> str | None:
        for j in range(len(self.teachers)):
            if bytes(self.teachers["node_id"][j]).rstrip(b"\0").decode() == node_id and \
                    self.teachers["state"][j] != FREE:
                return STATE_NAMES[int(self.teachers["state"][j])]
        return None


# ---------------------------------------------------------------------------
# Student side


class HostFlag:
    """slot.done for a remote reply: complete when the slot's READY word
    holds this dispatch's tag (the teacher's stream wrote it after its head
    kernel; the write is fenced, so the slot's data is in place)."""

    __slots__ = ("ready", "slot", "tag", "pending")

    def __init__(self, ready: np.ndarray, slot: int, tag: int, pending: dict):
        self.ready, self.slot, self.tag, self.pending = ready, slot, tag, pending

    def query(self) -> bool:
        if int(self.ready[self.slot]) == self.tag:
            self.pending.pop(self.tag, None)     # the watchdog stops timing it
            return True
        return False

    def synchronize(self, max_wait: float = 0.002) -> None:
        """Bounded spin: returns after max_wait even if the reply is not in,
        so the reader's watchdog gets to run between waits."""
        end = time.monotonic() + max_wait
        while not self.query() and time.monotonic() < end:
            time.sleep(2e-5)


class _QuarantineEnd:
    """Retirement marker for a failed remote teacher's slots: its writes can
    only stop once its process is gone."""

    def __init__(self, pid: int):
        self.pid = pid

    def query(self) -> bool:
        return not pid_alive(self.pid)


class SlotRing:
    """The student's device ring of soft-label slots, exported over CUDA IPC:
    slot j = (prob fp32 [B][k], class int32 [B][k]) at j * slot_bytes."""

    def __init__(self, cb: ControlBlock, s: int, batch_size: int, k: int, n_slots: int, device):
        from .reader import _Slot
        if not 1 <= n_slots <= cb.max_slots:
            raise ValueError(f"n_slots must be in [1, {cb.max_slots}]")
        self.B, self.k, self.n = batch_size, k, n_slots
        self.words = 2 * batch_size * k
        self.slot_bytes = 4 * self.words
        self.buf = torch.zeros(n_slots * self.words, dtype=torch.int32, device=device)
        self.handle = (ctypes.c_ubyte * 64)()
        off = ctypes.c_longlong()
        _lib.call("edl_ipc_export", self.buf.data_ptr(), self.handle, ctypes.byref(off))
        self.offset = int(off.value)
        self.slots = []
        for j in range(n_slots):
            v = self.buf[j * self.words:(j + 1) * self.words].view(2, batch_size, k)
            slot = _Slot.__new__(_Slot)
            slot.probs, slot.classes = v[0].view(torch.float32), v[1]
            slot.done = slot.release = None
            slot.iteration, slot.teacher, slot.batch, slot.batch_filled = -1, None, None, False
            slot.num_classes = None
            slot.index = j
            self.slots.append(slot)


class RemoteTeacher:
    """TeacherWorker interface for a teacher process (reader.py drives it)."""

    needs_rows = False   # the teacher replicates the student's sampler

    def __init__(self, pool: "ElasticPool", j: int, epoch: int, node_id: str):
        self.pool, self.cb = pool, pool.cb
        self.j, self.epoch, self.node_id = j, epoch, node_id
        self.pid = int(self.cb.teachers["pid"][j])
        self._sent: dict[int, float] = {}        # tag -> dispatch time (watchdog)
        self.failure: str | None = None
        self.batches_served = 0
        self._next_check = 0.0                    # the process / heartbeat checks run every check_period

    def _entry(self):
        return self.cb.teachers[self.j:self.j + 1]

    @property
    def alive(self) -> bool:
        """The watchdog. The reader asks on every pump (several times a step),
        so the syscall-backed checks (pid, heartbeat, reply deadlines) run at
        most every pool.check_period seconds; revocation is a shared-memory
        read and is checked every time."""
        if self.failure is not None:
            return False
        e = self._entry()
        now = time.monotonic()
        if int(e["epoch"][0]) != self.epoch or int(e["state"][0]) not in (AVAILABLE, ASSIGNED):
            self.failure = "revoked"
        elif now < self._next_check:
            return True
        elif not pid_alive(self.pid):
            self.failure = "process exited"
        elif time.monotonic_ns() - int(e["heartbeat_ns"][0]) > self.pool.ttl * 1e9:
            self.failure = "heartbeat expired"
        else:
            self._next_check = now + self.pool.check_period
            ready = self.pool.ready
            for tag, (t0, slot) in list(self._sent.items()):
                if int(ready[slot]) == tag:
                    self._sent.pop(tag, None)
                elif now - t0 > self.pool.reply_timeout:
                    self.failure = f"no reply within {self.pool.reply_timeout} s"
                    break
        return self.failure is None

    def submit(self, rows, slot) -> None:
        if not self.alive:
            raise RuntimeError(f"teacher {self.node_id} is not alive ({self.failure})")
        e = self._entry()
        head, tail = int(e["head"][0]), int(e["tail"][0])
        if head - tail >= self.cb.ring_len:
            raise RuntimeError(f"teacher {self.node_id} mailbox full")
        tag = self.pool.next_tag()
        self.pool.ready[slot.index] = 0
        rec = e["mailbox"][0, head % self.cb.ring_len:head % self.cb.ring_len + 1]
        rec["iteration"], rec["student"], rec["slot"], rec["tag"] = slot.iteration, self.pool.s, slot.index, tag
        rec["seq"] = head + 1
        e["head"] = head + 1               # x86-TSO: the record is visible before the head
        slot.done = HostFlag(self.pool.ready, slot.index, tag, self._sent)
        slot.num_classes = int(self.pool.cb.students["num_classes"][self.pool.s]) or None
        self._sent[tag] = (time.monotonic(), slot.index)
        self.batches_served += 1

    def drain_marker(self):
        return _QuarantineEnd(self.pid)

    def stop(self) -> None:
        """Fault injection: SIGKILL the teacher process."""
        with contextlib.suppress(ProcessLookupError):
            os.kill(self.pid, signal.SIGKILL)


class ElasticPool:
    """The student's view of the shared pool, with TeacherPool's interface
    (acquire_teachers / release_teacher / report_failure / status / kill)
    plus `slot_source` for the DistilReader."""

    def __init__(self, cb: ControlBlock, student_index: int, ttl: float = 5.0, reply_timeout: float = 30.0,
                 check_period: float = 0.005):
        self.cb, self.s = cb, student_index
        self.ttl, self.reply_timeout, self.check_period = ttl, reply_timeout, check_period
        self.ring: SlotRing | None = None
        self.ready = cb.students["ready"][student_index]
        self._tag = (os.getpid() & 0xFFFF) << 16
        self._proxies: dict[str, RemoteTeacher] = {}
        self.events: list[dict] = []

    def next_tag(self) -> int:
        self._tag = (self._tag + 1) & 0xFFFFFFFF or 1
        return self._tag

    def open(self, world: int, rank: int, batch_size: int, k: int, seed: int, temperature: float,
             num_classes: int, n_slots: int, device) -> SlotRing:
        """Publish this student's section: ring handle + sampler parameters."""
        self.ring = SlotRing(self.cb, self.s, batch_size, k, n_slots, device)
        with self.cb.locked():
            st = self.cb.students[self.s:self.s + 1]
            st["state"] = CLOSED
            st["pid"], st["rank"], st["world"], st["batch"], st["k"] = os.getpid(), rank, world, batch_size, k
            st["n_slots"], st["seed"], st["temperature"], st["num_classes"] = n_slots, seed, temperature, num_classes
            st["ring_offset"], st["slot_bytes"] = self.ring.offset, self.ring.slot_bytes
            st["ipc"][0, :] = np.frombuffer(bytes(self.ring.handle), dtype=np.uint8)
            st["ready"] = 0
            st["generation"] += 1
            st["state"] = OPEN
        return self.ring

    def slot_source(self):
        return self.ring

    def close(self) -> None:
        with self.cb.locked():
            self.cb.students["state"][self.s] = CLOSED

    # -- registry ----------------------------------------------------------------
    def _expire_dead(self) -> None:
        """The coordinator's TTL sweep (edl/coordinator.py:174-187), run by
        students under the lock before they pick teachers."""
        t = self.cb.teachers
        now = time.monotonic_ns()
        for j in range(len(t)):
            if t["state"][j] in (AVAILABLE, ASSIGNED) and (
                    not pid_alive(int(t["pid"][j])) or now - int(t["heartbeat_ns"][j]) > self.ttl * 1e9):
                t["state"][j] = EXPIRED
                t["owner"][j] = NO_OWNER
                self.events.append({"node_id": self._name(j), "to": "EXPIRED", "cause": "ttl"})

    def _name(self, j: int) -> str:
        return bytes(self.cb.teachers["node_id"][j]).rstrip(b"\0").decode()

    def acquire_teachers(self, student_id: str, count: int) -> list:
        if count < 1:
            raise ValueError("count must be >= 1")
        with self.cb.locked():
            self._expire_dead()
            t = self.cb.teachers
            free = sorted((j for j in range(len(t)) if t["state"][j] == AVAILABLE),
                          key=lambda j: (int(t["since"][j]), self._name(j)))
            granted = []
            for j in free[:count]:
                t["state"][j], t["owner"][j] = ASSIGNED, self.s
                name = self._name(j)
                proxy = RemoteTeacher(self, j, int(t["epoch"][j]), name)
                self._proxies[name] = proxy
                self.events.append({"node_id": name, "to": "ASSIGNED", "student_id": student_id})
                granted.append(proxy)
            return granted

    def release_teacher(self, student_id: str, node_id: str) -> None:
        with self.cb.locked():
            p = self._proxies.get(node_id)
            t = self.cb.teachers
            if p is None or t["state"][p.j] != ASSIGNED or t["owner"][p.j] != self.s or t["epoch"][p.j] != p.epoch:
                raise ValueError(f"{node_id} is not assigned to {student_id}")
            t["owner"][p.j] = NO_OWNER
            t["since"][p.j] = self.cb.tick()
            t["state"][p.j] = AVAILABLE
            self.events.append({"node_id": node_id, "to": "AVAILABLE", "released_by": student_id})

    def report_failure(self, student_id: str, node_id: str) -> None:
        """Expire the entry and revoke its epoch: a teacher process that is
        merely slow sees the bump and exits instead of serving stale work."""
        with self.cb.locked():
            p = self._proxies.get(node_id)
            if p is None:
                raise ValueError(f"{node_id} unknown")
            t = self.cb.teachers
            if t["epoch"][p.j] == p.epoch and t["state"][p.j] != EXPIRED:
                t["state"][p.j], t["owner"][p.j] = EXPIRED, NO_OWNER
                t["epoch"][p.j] += 1
                self.events.append({"node_id": node_id, "to": "EXPIRED", "cause": "reported",
                                    "reported_by": student_id, "why": p.failure})

    def status(self, node_id: str) -> str | None:
        return self.cb.teacher_status(node_id)

    def kill(self, node_id: str) -> None:
        p = self._proxies.get(node_id)
        if p is not None:
            p.stop()
        else:
            for j in range(len(self.cb.teachers)):
                if self._name(j) == node_id and self.cb.teachers["state"][j] in (AVAILABLE, ASSIGNED):
                    with contextlib.suppress(ProcessLookupError):
                        os.kill(int(self.cb.teachers["pid"][j]), signal.SIGKILL)

    def available_count(self) -> int:
        t = self.cb.teachers
        return int(sum(1 for j in range(len(t)) if t["state"][j] == AVAILABLE and pid_alive(int(t["pid"][j]))))


# ---------------------------------------------------------------------------
# Teacher side (edl/teacher_node.py:65-203)


class _RawView:
    """A device pointer with a shape (an IPC-mapped slot of the student's
    ring): all the fused head needs of its output buffers."""

    def __init__(self, ptr: int, shape: tuple):
        self._ptr, self.shape = ptr, shape

    def data_ptr(self) -> int:
        return self._ptr


class TeacherServer:
    """One teacher process: registers, serves its mailbox until revoked or
    shut down. Each request = (student, iteration, slot, tag): gather the
    iteration's rows from the HBM dataset replica (the student's sampler,
    replicated), run hidden GEMMs + the fused softmax/top-k head with the
    student's slot as the output, then write the tag into the slot's READY
    word — all on this process's stream."""

    def __init__(self, cb: ControlBlock, node_id: str, model, data, temperature: float | None = None,
                 simulated_delay: float = 0.0, sm_reserve: int = 0, idle_sleep: float = 2e-5):
        from . import nnkit
        self.cb, self.node_id = cb, node_id
        self.model, self.data = model, data
        self.device = model.device
        self.T = temperature
        self.delay_ns = int(simulated_delay * 1e9)
        self.idle_sleep = idle_sleep
        self.stream = torch.cuda.Stream(self.device)
        if sm_reserve > 0:
            sms = _lib.load().edl_device_sms()
            _lib.call("edl_set_stream_max_ctas", self.stream.cuda_stream, max(1, sms - sm_reserve))
        self._nk = nnkit
        self._rings: dict = {}        # student -> (generation, base ptr, sampler, ...)
        self._ws = None
        self._batch = None
        # an MLP teacher (nnkit.Model) or a cfg4 ResNet teacher (resnet.ResNetTeacher
        # over a data.DeviceImageDataset: rows are NHWC images)
        self._resnet = hasattr(model, "soft_labels")
        self.dev_base = cb.device_base()
        self.j, self.epoch = cb.register_teacher(node_id, os.getpid())
        self.served = 0

    def _student(self, s: int):
        from .data import DeviceShardSampler
        from .nnkit import Batch
        st = self.cb.students[s]
        gen = int(st["generation"])
        cached = self._rings.get(s)
        if cached is not None and cached[0] == gen:
            return cached
        if cached is not None:
            with contextlib.suppress(Exception):
                _lib.call("edl_ipc_close", cached[1])
        if int(st["state"]) != OPEN:
            raise RuntimeError(f"student section {s} is not open")
        base = ctypes.c_void_p()
        _lib.call("edl_ipc_open", bytes(st["ipc"]), ctypes.byref(base))
        B, k = int(st["batch"]), int(st["k"])
        sampler = DeviceShardSampler(self.data, int(st["world"]), int(st["rank"]), B, int(st["seed"]))
        if self._batch is None or self._batch.size != B:
            self._batch = Batch(torch.empty(B, self.data.samples.shape[1], dtype=torch.bfloat16, device=self.device),
                                torch.empty(B, dtype=torch.int64, device=self.device), self.data.dim)
            if self._resnet:
                if self.model.B != B:
                    raise RuntimeError(f"ResNet teacher built for batch {self.model.B}, student asks {B}")
            else:
                self._ws = self._nk.Workspace(self.model, B)
        entry = (gen, int(base.value), sampler, B, k, float(st["temperature"]),
                 int(base.value) + int(st["ring_offset"]), int(st["slot_bytes"]))
        self._rings[s] = entry
        return entry

    def _serve(self, rec) -> None:
        from .data import gather_batch
        from .nnkit import SoftLabels
        s, it, slot, tag = int(rec["student"]), int(rec["iteration"]), int(rec["slot"]), int(rec["tag"])
        _, _, sampler, B, k, T, ring, slot_bytes = self._student(s)
        ptr = ring + slot * slot_bytes
        probs, classes = _RawView(ptr, (B, k)), _RawView(ptr + 4 * B * k, (B, k))
        with torch.cuda.device(self.device), torch.cuda.stream(self.stream):
            rows = sampler.rows_for(it)
            batch = gather_batch(self.data, rows, self._batch, self.stream)
            out = SoftLabels(probs, classes, self.T or T)
            if self._resnet:
                self.model.soft_labels(self.data.nhwc(batch.inputs), self.T or T, k, out=out, stream=self.stream)
            else:
                self._nk.teacher_soft_labels(self.model, batch.inputs, self.T or T, k, out=out, stream=self.stream,
                                             ws=self._ws)
            if self.delay_ns:
                _lib.call("edl_stream_delay_ns", self.delay_ns, self.stream.cuda_stream)
            _lib.call("edl_stream_write_u32", self.dev_base + self.cb.ready_offset(s, slot), tag,
                      self.stream.cuda_stream)
        self.served += 1

    def serve_forever(self, max_requests: int | None = None) -> int:
        e = self.cb.teachers[self.j:self.j + 1]
        tail = int(e["tail"][0])
        while True:
            e["heartbeat_ns"] = time.monotonic_ns()
            if self.cb.shutdown or int(e["epoch"][0]) != self.epoch or int(e["state"][0]) == EXPIRED:
                break
            head = int(e["head"][0])
            if tail < head:
                rec = e["mailbox"][0, tail % self.cb.ring_len]
                if int(rec["seq"]) != tail + 1:     # the record lands before head moves; re-read
                    continue
                self._serve(rec)
                tail += 1
                e["tail"] = tail
                e["served"] = self.served
                if max_requests is not None and self.served >= max_requests:
                    break
            else:
                time.sleep(self.idle_sleep)
        self.stream.synchronize()
        return self.served


# ---------------------------------------------------------------------------
# Teacher process entry point: python -m paper_2207_06667_b200.elastic ...


def _parse_ints(s: str) -> tuple:
    return tuple(int(v) for v in s.split(","))


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(description="EDL teacher process serving an elastic pool")
    ap.add_argument("--control", required=True, help="pool control block (/dev/shm/...)")
    ap.add_argument("--node-id", required=True)
    ap.add_argument("--device", type=int, default=0)
    ap.add_argument("--teacher-file", help="EDLD model file (edl/nnkit.py:480-487)")
    ap.add_argument("--teacher-dims", help="init_model dims, e.g. 3072,8192,8192,1000")
    ap.add_argument("--teacher-seed", type=int, default=1)
    ap.add_argument("--data", help="make_blobs seed,n,dim,classes[,spread]")
    ap.add_argument("--images", help="cfg4: DeviceImageDataset seed,n,image,classes (with --resnet)")
    ap.add_argument("--resnet", help="cfg4: ResNet-50-style teacher seed,batch[,width]")
    ap.add_argument("--temperature", type=float, default=None)
    ap.add_argument("--simulated-delay", type=float, default=0.0)
    ap.add_argument("--sm-reserve", type=int, default=0)
    a = ap.parse_args(argv)
    from . import formats, nnkit
    from .data import DeviceDataset
    torch.cuda.set_device(a.device)
    if a.resnet:
        from .data import DeviceImageDataset
        from .resnet import ResNetConfig, ResNetTeacher, init_resnet
        iseed, n, image, classes = _parse_ints(a.images)
        rs = _parse_ints(a.resnet)
        width = rs[2] if len(rs) > 2 else 64
        data = DeviceImageDataset(iseed, n, image, classes)
        model = ResNetTeacher(init_resnet(ResNetConfig(image=image, classes=classes, width=width), rs[0]),
                              batch_size=rs[1])
    else:
        if a.teacher_file:
            model, _ = nnkit.load_model(a.teacher_file)
        else:
            model = nnkit.Model.from_host(formats.init_model(_parse_ints(a.teacher_dims), a.teacher_seed))
        parts = a.data.split(",")
        seed, n, dim, classes = (int(v) for v in parts[:4])
        spread = float(parts[4]) if len(parts) > 4 else 1.0
        data = DeviceDataset(formats.make_blobs(seed, n, dim, classes, spread))
    cb = ControlBlock(a.control)
    server = TeacherServer(cb, a.node_id, model, data, a.temperature, a.simulated_delay, a.sm_reserve)
    sys.stdout.write(f"teacher {a.node_id} registered as entry {server.j} epoch {server.epoch}\n")
    sys.stdout.flush()
    served = server.serve_forever()
    sys.stdout.write(f"teacher {a.node_id} served {served}\n")
    return 0


if __name__ == "__main__":
    sys.exit(main())
