"""Host logic of the elastic teacher pool (elastic.py) — CPU only.

The registry semantics follow edl/coordinator.py:99-197 (exclusive
acquisition, longest-available-first, report_failure expires at once, TTL
sweep) and the reference's tests/test_coordinator.py; the request mailbox,
dispatch tags and the watchdog are the device design's replacement for the
INFER_REQUEST / INFER_REPLY socket path (edl/student_node.py:351-457)."""

import os
import subprocess
import sys
import time

import numpy as np
import pytest

from paper_2207_06667_b200 import elastic
from paper_2207_06667_b200.elastic import ControlBlock, ElasticPool, HostFlag


@pytest.fixture
def cb(tmp_path):
    c = ControlBlock(str(tmp_path / "pool"), create=True, max_students=2, max_teachers=6, max_slots=16, ring_len=8)
    yield c
    c.close()


def dead_pid():
    p = subprocess.Popen([sys.executable, "-c", "pass"])
    p.wait()
    return p.pid


class FakeSlot:
    def __init__(self, index, iteration):
        self.index, self.iteration = index, iteration
        self.done = None
        self.num_classes = None


def test_attach_sees_the_same_block(cb):
    other = ControlBlock(cb.path)
    try:
        j, epoch = other.register_teacher("t1", os.getpid())
        assert cb.teacher_status("t1") == "AVAILABLE" and epoch == 1
        assert other.max_slots == 16 and other.ring_len == 8
    finally:
        other.close()


def test_acquire_is_exclusive_and_longest_available_first(cb):
    me = os.getpid()
    for name in ("t3", "t1", "t2"):
        cb.register_teacher(name, me)
    a, b = ElasticPool(cb, 0), ElasticPool(cb, 1)
    got = [w.node_id for w in a.acquire_teachers("student-0", 2)]
    assert got == ["t3", "t1"]                       # registration order = available-since order
    assert [w.node_id for w in b.acquire_teachers("student-1", 5)] == ["t2"]
    assert b.acquire_teachers("student-1", 1) == []
    a.release_teacher("student-0", "t3")
    assert cb.teacher_status("t3") == "AVAILABLE"
    with pytest.raises(ValueError):
        b.release_teacher("student-1", "t1")         # not b's teacher
    assert [w.node_id for w in b.acquire_teachers("student-1", 1)] == ["t3"]
    with pytest.raises(ValueError):
        a.acquire_teachers("student-0", 0)


def test_report_failure_expires_and_revokes_epoch(cb):
    j, epoch = cb.register_teacher("t1", os.getpid())
    pool = ElasticPool(cb, 0)
    (w,) = pool.acquire_teachers("student-0", 1)
    assert w.alive
    pool.report_failure("student-0", "t1")
    assert cb.teacher_status("t1") == "EXPIRED"
    assert int(cb.teachers["epoch"][j]) == epoch + 1  # a slow teacher process sees this and exits
    assert not w.alive and w.failure == "revoked"
    pool.report_failure("student-0", "t1")            # idempotent
    with pytest.raises(ValueError):
        pool.report_failure("student-0", "nobody")


def test_dead_process_is_detected_and_swept(cb):
    pid = dead_pid()
    cb.register_teacher("t1", pid)
    cb.register_teacher("t2", os.getpid())
    pool = ElasticPool(cb, 0)
    got = pool.acquire_teachers("student-0", 2)      # the sweep expires t1 first
    assert [w.node_id for w in got] == ["t2"]
    assert cb.teacher_status("t1") == "EXPIRED"
    assert pool.available_count() == 0


def test_heartbeat_ttl(cb):
    j, _ = cb.register_teacher("t1", os.getpid())
    pool = ElasticPool(cb, 0, ttl=0.05)
    (w,) = pool.acquire_teachers("student-0", 1)
    assert w.alive
    time.sleep(0.1)                                  # nobody beats
    assert not w.alive and w.failure == "heartbeat expired"


def test_readd_after_death_reuses_the_entry_with_a_new_epoch(cb):
    j, e1 = cb.register_teacher("t1", dead_pid())
    pool = ElasticPool(cb, 0)
    assert pool.acquire_teachers("student-0", 1) == []   # swept
    j2, e2 = cb.register_teacher("t1", os.getpid())
    assert j2 == j and e2 == e1 + 1
    (w,) = pool.acquire_teachers("student-0", 1)
    assert w.node_id == "t1" and w.epoch == e2 and w.alive
    with pytest.raises(ValueError):
        cb.register_teacher("t1", os.getpid())            # live: second registration refused


def test_mailbox_dispatch_tags_and_reply(cb):
    j, _ = cb.register_teacher("t1", os.getpid())
    pool = ElasticPool(cb, 1)
    cb.students["num_classes"][1] = 10
    (w,) = pool.acquire_teachers("student-1", 1)
    slots = [FakeSlot(3, 40), FakeSlot(5, 41)]
    for s in slots:
        w.submit(None, s)
    e = cb.teachers[j]
    assert int(e["head"]) == 2 and int(e["tail"]) == 0
    recs = [cb.teachers["mailbox"][j, i] for i in range(2)]
    assert [(int(r["iteration"]), int(r["slot"]), int(r["student"])) for r in recs] == [(40, 3, 1), (41, 5, 1)]
    tags = [int(r["tag"]) for r in recs]
    assert tags[0] != tags[1] and all(isinstance(s.done, HostFlag) for s in slots)
    assert slots[0].num_classes == 10
    assert not slots[0].done.query()
    ready = cb.students["ready"][1]
    ready[3] = tags[0] ^ 1                            # a stale tag is not a reply
    assert not slots[0].done.query()
    ready[3] = tags[0]                               # what the teacher's stream writes
    assert slots[0].done.query() and not slots[1].done.query()
    assert tags[0] not in w._sent and tags[1] in w._sent


def test_mailbox_full_raises(cb):
    cb.register_teacher("t1", os.getpid())
    pool = ElasticPool(cb, 0)
    (w,) = pool.acquire_teachers("student-0", 1)
    for i in range(cb.ring_len):
        w.submit(None, FakeSlot(i % 16, i))
    with pytest.raises(RuntimeError):
        w.submit(None, FakeSlot(0, 99))


def test_reply_timeout_watchdog(cb):
    cb.register_teacher("t1", os.getpid())
    pool = ElasticPool(cb, 0, reply_timeout=0.05)
    (w,) = pool.acquire_teachers("student-0", 1)
    w.submit(None, FakeSlot(0, 0))
    assert w.alive
    time.sleep(0.08)
    cb.teachers["heartbeat_ns"][0] = time.monotonic_ns()   # alive process, but no reply
    assert not w.alive and "no reply" in w.failure


def test_quarantine_ends_only_when_the_process_exits(cb):
    p = subprocess.Popen([sys.executable, "-c", "import time; time.sleep(30)"])
    try:
        cb.register_teacher("t1", p.pid)
        pool = ElasticPool(cb, 0)
        (w,) = pool.acquire_teachers("student-0", 1)
        marker = w.drain_marker()
        assert not marker.query()
        w.stop()                                      # SIGKILL
        p.wait(10)
        assert marker.query()
        assert not w.alive and w.failure == "process exited"
    finally:
        if p.poll() is None:
            p.kill()


def test_zombie_counts_as_dead():
    p = subprocess.Popen([sys.executable, "-c", "pass"])
    deadline = time.time() + 10
    while time.time() < deadline:                     # exited but not reaped yet
        with open(f"/proc/{p.pid}/stat", "rb") as fh:
            if b") Z" in fh.read():
                break
        time.sleep(0.01)
    assert not elastic.pid_alive(p.pid)
    p.wait()
    assert not elastic.pid_alive(p.pid)


def test_ready_offset_addresses_the_ready_words(cb):
    base = cb.host_base
    for s, slot in ((0, 0), (1, 7)):
        addr = base + cb.ready_offset(s, slot)
        view = np.ctypeslib.as_array((np.ctypeslib.ctypes.c_uint32 * 1).from_address(addr))
        view[0] = 0xABC0 + slot
        assert int(cb.students["ready"][s][slot]) == 0xABC0 + slot
