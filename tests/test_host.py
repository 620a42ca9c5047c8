"""CPU tests: host logic of the device path (scheduler, JSQ, pool, data
formats) against the reference's tables and golden vectors, and the C-ABI
library's load/export surface (no compute calls without a GPU)."""

import ctypes
import os
import re

import numpy as np
import pytest

from paper_2207_06667_b200 import formats
from paper_2207_06667_b200.reader import (NONE, REQUEST_ADDITIONAL_TEACHER, RESUME_SENDING, STOP_SENDING,
                                          SchedulerConfig, TeacherPool, ThroughputProfile, pick_teacher,
                                          scheduler_tick, static_schedule)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden")


# -- Alg. 1 / JSQ / static schedule: the reference's own tables
# (tests/test_student_node.py:23-81)

@pytest.mark.parametrize("volume,sending,cooldown,expected", [
    (33, True, True, STOP_SENDING), (33, False, True, STOP_SENDING),
    (0, True, True, REQUEST_ADDITIONAL_TEACHER), (0, True, False, NONE),
    (0, False, True, RESUME_SENDING), (3, False, True, RESUME_SENDING),
    (3, True, True, NONE), (4, False, True, NONE), (32, True, True, NONE),
    (32, False, True, NONE), (5, True, True, NONE)])
def test_scheduler_tick_table(volume, sending, cooldown, expected):
    assert scheduler_tick(volume, sending, cooldown, SchedulerConfig(lt=4, ut=32)) == expected


def test_scheduler_config_validation():
    for kw in (dict(lt=5, ut=5), dict(lt=-1, ut=5), dict(n_static=0), dict(pipeline_depth=0)):
        with pytest.raises(ValueError):
            SchedulerConfig(**kw)


def test_static_schedule_and_jsq():
    assert static_schedule(ThroughputProfile(5.0, 5.0)) == 1
    assert static_schedule(ThroughputProfile(4.2, 1.0)) == 5
    assert static_schedule(ThroughputProfile(10.0, 3.0)) == 4
    assert static_schedule(ThroughputProfile(1.0, 100.0)) == 1
    assert pick_teacher({"a": 2, "b": 0, "c": 1}, 3) == "b"
    assert pick_teacher({"b": 1, "a": 1}, 3) == "a"
    assert pick_teacher({"a": 2, "b": 2}, 2) is None
    assert pick_teacher({}, 2) is None


class _FakeWorker:
    def __init__(self, nid):
        self.node_id = nid
        self.alive = True

    def stop(self):
        self.alive = False


def test_pool_longest_available_first_exclusive_and_failures():
    pool = TeacherPool()
    for n in ("t2", "t1", "t3"):
        pool.register(_FakeWorker(n))
    got = [w.node_id for w in pool.acquire_teachers("s0", 2)]
    assert got == ["t2", "t1"]                       # registration order, not name order
    assert [w.node_id for w in pool.acquire_teachers("s1", 5)] == ["t3"]
    assert pool.acquire_teachers("s2", 1) == []      # exclusive
    pool.release_teacher("s0", "t1")
    with pytest.raises(ValueError):
        pool.release_teacher("s0", "t3")             # not the owner
    pool.report_failure("s1", "t3")
    assert pool.status("t3") == "EXPIRED"
    assert [w.node_id for w in pool.acquire_teachers("s2", 3)] == ["t1"]
    pool.kill("t2")
    assert pool.acquire_teachers("s3", 1) == []


# -- data formats vs golden vectors from the reference

def test_formats_against_reference_golden():
    d = np.load(os.path.join(GOLD, "data.npz"))
    b = formats.make_blobs(42, 100, 5, 4, 1.5)
    assert np.array_equal(b.samples, d["blobs_samples"]) and np.array_equal(b.labels, d["blobs_labels"])
    assert b.id == str(d["blobs_id"])
    assert np.array_equal(formats.epoch_order(0, 0, 0, 100), d["order"])
    small = formats.init_model([3, 4, 2], 9)
    blob = formats.serialize_model(small, iteration=137)
    assert blob == d["edld"].tobytes()
    m, it = formats.deserialize_model(blob)
    assert it == 137 and formats.serialize_model(m, 137) == blob
    with pytest.raises(formats.ModelFileError):
        formats.deserialize_model(b"XXXX" + blob[4:])
    with pytest.raises(formats.ModelFileError):
        formats.deserialize_model(blob[:-3])
    with pytest.raises(formats.ModelFileError):
        formats.deserialize_model(blob + b"\0" * 8)
    shard = formats.partition(formats.make_blobs(0, 65, 4, 4, 1.0), 2, 1)
    assert shard.size == 33


def test_checkpoint_round_trip_and_corrupt_fallback(tmp_path):
    from paper_2207_06667_b200.student import load_latest_checkpoint, save_checkpoint
    m1 = formats.init_model([4, 8, 3], 0)
    m2 = formats.init_model([4, 8, 3], 1)
    save_checkpoint(str(tmp_path), m1, 100, "data-1", 2)
    p2 = save_checkpoint(str(tmp_path), m2, 200, "data-1", 2)
    got, it = load_latest_checkpoint(str(tmp_path), "data-1")
    assert it == 200 and np.array_equal(got.weights[0], m2.weights[0])
    with open(p2, "r+b") as fh:
        fh.truncate(30)                              # corrupt the newest -> fall back
    got, it = load_latest_checkpoint(str(tmp_path), "data-1")
    assert it == 100 and np.array_equal(got.weights[0], m1.weights[0])
    assert load_latest_checkpoint(str(tmp_path), "other") is None


# -- the C-ABI boundary

def _header_symbols():
    with open(os.path.join(ROOT, "include", "edl_b200.h")) as fh:
        text = fh.read()
    return sorted(set(re.findall(r"^\s*(?:int|long long|const char\*)\s+(edl_\w+)\(", text, re.M)))


def test_library_exports_every_header_symbol():
    from paper_2207_06667_b200 import _lib
    from paper_2207_06667_b200.build import build
    build()
    lib = ctypes.CDLL(_lib.LIB_PATH)
    syms = _header_symbols()
    assert len(syms) >= 14
    for s in syms:
        assert hasattr(lib, s), s
    assert sorted(_lib.exported_symbols()) == syms
    L = _lib.load()
    assert L.edl_version() == _lib.ABI_VERSION
    assert L.edl_colsum_workspace_floats(4096, 2048) == 64 * 2048          # 64-row chunks
    assert _lib.colsum_group_workspace_floats([4096, 4096], [2048, 1008]) == 64 * (2048 + 1008)


def test_product_path_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_2207_06667_b200")
    for name in os.listdir(pkg):
        if name.endswith(".py"):
            with open(os.path.join(pkg, name)) as fh:
                src = fh.read()
            assert "oracle" not in re.findall(r"^\s*(?:from|import)\s+(\w+)", src, re.M), name
