"""DistilReader / TeacherPool / StudentNode on the device — the reference's
tests/test_student_node.py:193-340 scenarios re-run against the device
pipeline (B200 only)."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture
def cluster():
    from paper_2207_06667_b200 import formats, nnkit
    from paper_2207_06667_b200.data import DeviceDataset, DeviceShardSampler
    from paper_2207_06667_b200.reader import EventLog, SchedulerConfig, TeacherPool
    from paper_2207_06667_b200.teacher import TeacherConfig, TeacherWorker
    data = formats.make_blobs(0, 2048, 6, 4, 0.8)
    dd = DeviceDataset(data)
    teacher_h = formats.init_model((6, 16, 4), 3)
    teacher = nnkit.Model.from_host(teacher_h)
    pool = TeacherPool()

    def spawn(node_id):
        w = TeacherWorker(TeacherConfig(node_id, 2.0, 4), teacher, dd)
        pool.register(w)
        return w

    def make_reader(end=50, sched=None, session=1):
        from paper_2207_06667_b200.reader import DistilReader
        sampler = DeviceShardSampler(dd, 1, 0, 8, seed=0)
        events = EventLog()
        r = DistilReader("student-0", pool, sched or SchedulerConfig(lt=2, ut=8, probe_interval=0.0,
                                                                      acquire_cooldown=0.2),
                         sampler, 0, end, session, events, 2.0, 4)
        return r, events, sampler

    return pool, spawn, make_reader, teacher


def test_consume_in_order_matches_local_teacher(cluster):
    from paper_2207_06667_b200 import nnkit
    pool, spawn, make_reader, teacher = cluster
    spawn("t1")
    reader, events, sampler = make_reader(end=12)
    assert reader.acquire(1) == 1
    for i in range(12):
        soft = reader.consume(i, timeout=15)
        torch.cuda.current_stream().synchronize()
        b = sampler.batch_for(i)
        expect = nnkit.teacher_soft_labels(teacher, b.inputs, 2.0, 4)
        assert torch.equal(soft.probs, expect.probs) and torch.equal(soft.classes, expect.classes)
    assert reader.ledger()["ok"]
    reader.close()


def test_volume_respects_upper_threshold_then_resumes(cluster):
    from paper_2207_06667_b200.reader import SchedulerConfig
    pool, spawn, make_reader, _ = cluster
    spawn("t1")
    sched = SchedulerConfig(lt=2, ut=5, probe_interval=0.0, acquire_cooldown=1e9, pipeline_depth=2)
    reader, *_ = make_reader(end=200, sched=sched)
    assert reader.acquire(1) == 1
    for _ in range(200):
        reader.pump()
        torch.cuda.synchronize()
    assert reader.max_volume_seen <= sched.ut + reader.in_flight_capacity()
    assert not reader.sending_enabled
    it = 0
    while reader.volume > 0:
        reader.consume(it, timeout=10)
        it += 1
    reader.pump()
    assert reader.sending_enabled
    reader.close()


def test_kill_teacher_with_inflight_redispatches_exactly_unanswered(cluster):
    pool, spawn, make_reader, _ = cluster
    victim = spawn("t1")
    spawn("t2")
    reader, events, _ = make_reader(end=30)
    assert reader.acquire(1) == 1
    reader.consume(0, timeout=15)
    reader.pump()
    assert any(reader._teachers["t1"].outstanding.values())
    victim.stop()
    for i in range(1, 30):
        reader.consume(i, timeout=20)
    ledger = reader.ledger()
    assert ledger["ok"] and ledger["redispatches"] >= 1
    kinds = [e["event"] for e in events.entries]
    assert "teacher_failure" in kinds and "teacher_replaced" in kinds
    fail = [e for e in events.entries if e["event"] == "teacher_failure"][0]
    assert fail["unanswered"] and fail["unanswered"] == sorted(fail["unanswered"])
    assert pool.status("t1") == "EXPIRED"
    reader.close()


def test_head_of_line_unanswered_is_dispatched_while_sending_is_stopped(cluster):
    """A slow teacher holds the lowest iterations while a fast one fills the
    buffer past ut (sending stops); the slow one dies with no replacement.
    The buffer cannot drain past the missing head-of-line batch, so the
    reader dispatches exactly that batch to the survivor despite the stop
    (the reference would wait forever here: edl/student_node.py:351-376)."""
    import time

    from paper_2207_06667_b200.reader import SchedulerConfig
    from paper_2207_06667_b200.teacher import TeacherConfig, TeacherWorker
    pool, spawn, make_reader, _ = cluster
    fast = spawn("t2")
    slow = TeacherWorker(TeacherConfig("t1", 2.0, 4, simulated_delay=0.5), cluster[3], fast.data)
    pool.register(slow)
    sched = SchedulerConfig(lt=2, ut=5, probe_interval=0.0, acquire_cooldown=1e9, pipeline_depth=2)
    reader, events, _ = make_reader(end=16, sched=sched)
    assert reader.acquire(2) == 2
    t0 = time.monotonic()
    while reader.sending_enabled and time.monotonic() - t0 < 10:
        reader.pump()
        time.sleep(0.001)
    assert not reader.sending_enabled
    assert 0 not in reader._ready and 0 in reader._teachers["t1"].outstanding
    slow.stop()
    for i in range(16):
        reader.consume(i, timeout=10)
    kinds = [e["event"] for e in events.entries]
    assert "teacher_failure" in kinds and "no_replacement" in kinds
    assert reader.ledger()["ok"]
    reader.close()


def test_kill_idle_teacher_acquires_exactly_one_replacement(cluster):
    pool, spawn, make_reader, _ = cluster
    idle = spawn("t1")
    spawn("t2")
    reader, events, _ = make_reader(end=0)
    assert reader.acquire(1) == 1
    idle.stop()
    reader.pump()
    failures = [e for e in events.entries if e["event"] == "teacher_failure"]
    replaced = [e for e in events.entries if e["event"] == "teacher_replaced"]
    assert len(failures) == 1 and failures[0]["unanswered"] == []
    assert len(replaced) == 1
    reader.close()


def test_unassigned_teacher_death_is_invisible(cluster):
    pool, spawn, make_reader, _ = cluster
    spawn("t1")
    bystander = spawn("t2")
    reader, events, _ = make_reader(end=5)
    assert reader.acquire(1) == 1
    assert {e["node"] for e in events.entries if e["event"] == "teacher_added"} == {"t1"}
    bystander.stop()
    for i in range(5):
        reader.consume(i, timeout=15)
    kinds = [e["event"] for e in events.entries]
    assert "teacher_failure" not in kinds and "request_additional_teacher" not in kinds
    reader.close()


def test_no_replacement_then_recovers_via_probe(cluster):
    pool, spawn, make_reader, _ = cluster
    only = spawn("t1")
    reader, events, _ = make_reader(end=20)
    assert reader.acquire(1) == 1
    reader.consume(0, timeout=15)
    only.stop()
    reader.pump()
    assert any(e["event"] == "no_replacement" for e in events.entries)
    spawn("t3")
    import time
    time.sleep(0.25)   # acquire cooldown
    for i in range(1, 20):
        reader.consume(i, timeout=30)
    assert reader.ledger()["ok"]
    reader.close()


def test_student_modes_and_trajectory():
    """StudentNode.run in ntrain / online / edl modes. EDL and online consume
    identical soft labels, so their final parameters agree; ntrain equals the
    oracle's straight hard-label loop within the bf16 tolerance."""
    from oracle import nnkit_ref as ref
    from paper_2207_06667_b200 import formats
    from paper_2207_06667_b200.nnkit import TrainConfig
    from paper_2207_06667_b200.reader import TeacherPool
    from paper_2207_06667_b200.student import DataSpec, StudentConfig, StudentNode, spawn_teachers
    spec = DataSpec(seed=3, n=256, dim=6, classes=4, spread=1.0)
    teacher = formats.init_model((6, 32, 4), 7)
    train = TrainConfig(eta=0.05, alpha=0.5, beta=0.5, temperature=2.0, batch_size=16, seed=5)
    res = {}
    for mode in ("ntrain", "online", "edl"):
        cfg = StudentConfig(mode=mode, data=spec, train=train, epochs=2, k=4, teacher_count=1)
        pool = None
        node = None
        if mode == "edl":
            pool = TeacherPool()
            node = StudentNode(cfg, pool=pool)
            spawn_teachers(pool, teacher, 2, {str(node.dataset.device): node.dataset}, 2.0, 4)
        else:
            node = StudentNode(cfg, teacher_model=teacher)
        res[mode] = node.run()
        assert res[mode].ledger["ok"]
    a = ref.flatten(res["online"].model.weights, res["online"].model.biases)
    b = ref.flatten(res["edl"].model.weights, res["edl"].model.biases)
    assert np.array_equal(a, b)
    # ntrain vs the oracle straight loop (hard labels only)
    samples, labels = ref.make_blobs(3, 256, 6, 4, 1.0)
    ws, bs = ref.init_model((6, 64, 4), 5)
    bpe = 256 // 16
    for it in range(2 * bpe):
        rows = ref.batch_rows(5, 0, 256, 16, bpe, it)
        _, gw, gb = ref.kd_loss(ws, bs, samples[rows], labels[rows], None, 0.5, 0.0, 2.0)
        ws, bs = ref.sgd_step(ws, bs, gw, gb, 0.05)
    dev = ref.flatten(res["ntrain"].model.weights, res["ntrain"].model.biases)
    orc = ref.flatten(ws, bs)
    assert np.linalg.norm(dev - orc) / np.linalg.norm(orc) < 1e-2


def _edl_run(faults):
    from paper_2207_06667_b200 import formats
    from paper_2207_06667_b200.nnkit import TrainConfig
    from paper_2207_06667_b200.reader import SchedulerConfig, TeacherPool
    from paper_2207_06667_b200.student import DataSpec, StudentConfig, StudentNode, spawn_teachers
    from paper_2207_06667_b200.teacher import TeacherConfig, TeacherWorker
    spec = DataSpec(seed=1, n=512, dim=8, classes=6, spread=1.0)
    teacher = formats.init_model((8, 32, 6), 11)
    train = TrainConfig(eta=0.05, alpha=0.5, beta=0.5, temperature=2.0, batch_size=16, seed=2)
    cfg = StudentConfig(mode="edl", data=spec, train=train, epochs=2, k=4, teacher_count=2,
                        sched=SchedulerConfig(lt=2, ut=6, probe_interval=0.0, acquire_cooldown=0.0))
    pool = TeacherPool()
    node = StudentNode(cfg, pool=pool)
    dev = str(node.dataset.device)
    workers = spawn_teachers(pool, teacher, 3, {dev: node.dataset}, 2.0, 4)
    events = []

    def hook(it, reader):
        for kind, at, name in faults:
            if it == at and kind == "kill":
                pool.kill(name)
                events.append(("kill", name))
            if it == at and kind == "add":
                w = TeacherWorker(TeacherConfig(name, 2.0, 4), workers[0].model, node.dataset)
                pool.register(w)
                events.append(("add", name))
    return node.run(on_iteration=hook), node, events


def test_drop_and_readd_teachers_mid_run_keeps_trajectory():
    """configs[4] fault test: teachers die with batches in flight and new ones
    join mid-run; every batch is trained exactly once and the trajectory is
    bit-identical to the fault-free run (soft labels are deterministic)."""
    from oracle import nnkit_ref as ref
    clean, _, _ = _edl_run([])
    faulty, node, ev = _edl_run([("kill", 5, "t1"), ("kill", 9, "t2"), ("add", 12, "t9"), ("kill", 20, "t3")])
    assert clean.ledger["ok"] and faulty.ledger["ok"]
    assert faulty.ledger["consumed"] == clean.ledger["consumed"] == node.total_steps
    kinds = [e["event"] for e in node.events.entries]
    assert kinds.count("teacher_failure") >= 2 and "teacher_replaced" in kinds
    a = ref.flatten(clean.model.weights, clean.model.biases)
    b = ref.flatten(faulty.model.weights, faulty.model.biases)
    assert np.array_equal(a, b)


def test_epoch_permutation_ready_for_other_streams():
    """A new epoch's row permutation must be usable by a gather on ANOTHER
    stream right after rows_for returns, even while the calling stream is
    still busy (teacher workers gather on their own streams). Regression: the
    upload used to ride the caller's stream, so a teacher-stream gather could
    read the index buffer before it landed (illegal address under load)."""
    from paper_2207_06667_b200 import formats
    from paper_2207_06667_b200.data import DeviceDataset, DeviceShardSampler, gather_batch
    from paper_2207_06667_b200.formats import epoch_order
    host = formats.make_blobs(0, 4096, 48, 10, 1.0)
    data = DeviceDataset(host)
    sampler = DeviceShardSampler(data, 1, 0, 256, seed=3)
    other = torch.cuda.Stream()
    for epoch in range(6):
        torch.cuda._sleep(50_000_000)                # the caller's stream stays busy for ~25 ms
        rows = sampler.rows_for(epoch * sampler.batches_per_epoch + 5)
        with torch.cuda.stream(other):
            b = gather_batch(data, rows, stream=other)
            got = b.hard_labels.clone()
        other.synchronize()
        want = epoch_order(3, epoch, 0, 4096)[5 * 256:6 * 256]
        assert np.array_equal(got.cpu().numpy(), host.labels[want])
    torch.cuda.synchronize()
