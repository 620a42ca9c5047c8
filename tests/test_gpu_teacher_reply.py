"""soft_label_reply's request/reply contract and the soft-label error paths
(B200 only) — the reference's tests/test_teacher_node.py:44-62 cases
re-run against the device teacher (edl/teacher_node.py:47-58), plus the
class-count and status-word checks of kd_loss (edl/nnkit.py:272-297) and the
contents of re-dispatched soft labels after a teacher failure."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def env():
    from paper_2207_06667_b200 import formats, nnkit
    from paper_2207_06667_b200.data import DeviceDataset
    host = formats.init_model((8, 16, 5), 0)
    model = nnkit.Model.from_host(host)
    data = DeviceDataset(formats.make_blobs(0, 64, 8, 5, 1.0))
    return nnkit, model, host, data


def test_echoes_batch_id(env):
    from paper_2207_06667_b200.teacher import soft_label_reply
    _, model, _, _ = env
    reply = soft_label_reply(model, 2.0, {"batch_id": "s0-7", "inputs": [[0.0] * 8]})
    assert reply["type"] == "INFER_REPLY" and reply["batch_id"] == "s0-7"
    assert reply["temperature"] == 2.0


def test_dense_rows_sum_to_one_and_match_oracle(env):
    """k = K (the default) is the reference's dense reply: every row sums to 1
    (fp32: 1e-5 instead of the reference's fp64 1e-9) and equals
    tempered_softmax(forward(model, X), T) at the bf16 storage points."""
    from oracle import nnkit_ref as ref
    from paper_2207_06667_b200.teacher import soft_label_reply
    _, model, host, _ = env
    x = np.random.default_rng(0).normal(size=(16, 8))
    reply = soft_label_reply(model, 2.0, {"batch_id": "b", "inputs": x.tolist()})
    soft = reply["probs"]
    assert soft.k == 5 and soft.num_classes == 5
    p = soft.probs.cpu().numpy().astype(np.float64)
    c = soft.classes.cpu().numpy().astype(np.int64)
    assert np.abs(p.sum(axis=1) - 1).max() < 1e-5
    want = ref.tempered_softmax(ref.forward_bf16_storage(list(host.weights), list(host.biases), x), 2.0)
    got = np.take_along_axis(want, c, axis=1)
    assert np.abs(p - got).max() / got.max() < 1e-3


def test_dimension_mismatch_is_error_reply(env):
    from paper_2207_06667_b200.teacher import soft_label_reply
    _, model, _, _ = env
    reply = soft_label_reply(model, 2.0, {"batch_id": "b", "inputs": [[1.0, 2.0]]})
    assert reply["type"] == "ERROR" and reply["batch_id"] == "b"
    assert "bad inference request" in reply["reason"]


@pytest.mark.parametrize("inputs", [[1.0, 2.0, 3.0], [[[0.0] * 8]], "abc"])
def test_non_matrix_inputs_are_error_replies(env, inputs):
    from paper_2207_06667_b200.teacher import soft_label_reply
    _, model, _, _ = env
    reply = soft_label_reply(model, 2.0, {"batch_id": 3, "inputs": inputs})
    assert reply["type"] == "ERROR" and reply["batch_id"] == 3


def test_bad_temperature_is_error_reply(env):
    from paper_2207_06667_b200.teacher import soft_label_reply
    _, model, _, _ = env
    reply = soft_label_reply(model, 0.0, {"batch_id": "t", "inputs": [[0.0] * 8]})
    assert reply["type"] == "ERROR" and reply["batch_id"] == "t"


def test_row_indexed_request_equals_local_teacher(env):
    """A request naming dataset rows (the device-native payload) serves the
    same bytes as the teacher run on the gathered batch, and as a request
    that ships those rows' (bf16-exact) values."""
    from paper_2207_06667_b200.data import gather_batch
    from paper_2207_06667_b200.teacher import soft_label_reply
    nk, model, _, data = env
    rows = [5, 0, 63, 17, 17, 2]
    r1 = soft_label_reply(model, 3.0, {"batch_id": "q1", "rows": rows}, k=3, data=data)
    assert r1["type"] == "INFER_REPLY" and r1["batch_id"] == "q1" and r1["temperature"] == 3.0
    b = gather_batch(data, torch.tensor(rows, device=data.device))
    local = nk.teacher_soft_labels(model, b.inputs, 3.0, 3)
    assert torch.equal(r1["probs"].probs, local.probs) and torch.equal(r1["probs"].classes, local.classes)
    x = data.samples[torch.tensor(rows, device=data.device), :8].float().cpu().numpy()
    r2 = soft_label_reply(model, 3.0, {"batch_id": "q2", "inputs": x}, k=3)
    assert torch.equal(r2["probs"].probs, local.probs) and torch.equal(r2["probs"].classes, local.classes)


def test_row_indexed_request_without_dataset_is_error(env):
    from paper_2207_06667_b200.teacher import soft_label_reply
    _, model, _, _ = env
    reply = soft_label_reply(model, 2.0, {"batch_id": "r", "rows": [0, 1]})
    assert reply["type"] == "ERROR" and reply["batch_id"] == "r"


def test_pipelined_requests_each_answered_once(env):
    from paper_2207_06667_b200.teacher import soft_label_reply
    _, model, _, _ = env
    ids = [f"b{i}" for i in range(10)]
    got = [soft_label_reply(model, 2.0, {"batch_id": bid, "inputs": [[float(i)] * 8]})["batch_id"]
           for i, bid in enumerate(ids)]
    assert got == ids


def test_kd_loss_rejects_teacher_with_other_class_count(env):
    """A teacher with more classes than the student (ids >= K) is a
    ShapeError before launch (edl/nnkit.py:272-274), not a silent loss."""
    from paper_2207_06667_b200 import formats
    nk, _, _, _ = env
    teacher = nk.Model.from_host(formats.init_model((8, 16, 7), 1))
    student = nk.Model.from_host(formats.init_model((8, 12, 5), 2))
    batch = nk.make_batch(np.zeros((4, 8)), np.array([0, 1, 2, 3]))
    soft = nk.teacher_soft_labels(teacher, batch.inputs, 2.0, 3)
    assert soft.num_classes == 7
    cfg = nk.TrainConfig(alpha=0.5, beta=0.5, batch_size=4)
    with pytest.raises(nk.ShapeError):
        nk.kd_loss(student, batch, soft, cfg)


def test_status_word_raises_once_then_clears(env):
    """A device-detected bad label raises at the next check and the status
    word is cleared, so a later good batch on the same workspace is fine."""
    from paper_2207_06667_b200 import formats
    nk, _, _, _ = env
    student = nk.Model.from_host(formats.init_model((8, 12, 5), 2))
    ws = nk.Workspace(student, 4)
    cfg = nk.TrainConfig(alpha=1.0, beta=0.0, batch_size=4)
    bad = nk.make_batch(np.zeros((4, 8)), np.array([0, 1, 9, 3]))
    good = nk.make_batch(np.zeros((4, 8)), np.array([0, 1, 2, 3]))
    loss, _ = nk.kd_loss(student, bad, None, cfg, ws=ws)
    with pytest.raises(nk.ShapeError):
        float(loss)
    loss, _ = nk.kd_loss(student, good, None, cfg, ws=ws)
    assert np.isfinite(float(loss))


def test_simulated_delay_slows_the_worker_stream_not_the_host(env):
    """TeacherConfig.simulated_delay (edl/teacher_node.py:30-44) is spent on
    the worker's stream: submit returns at once, the slot lands later."""
    import time

    from paper_2207_06667_b200.reader import _Slot
    from paper_2207_06667_b200.teacher import TeacherConfig, TeacherWorker
    _, model, _, data = env
    w = TeacherWorker(TeacherConfig("slow", 2.0, 3, simulated_delay=0.05), model, data)
    slot = _Slot(8, 3, data.device)
    rows = torch.arange(8, device=data.device)
    w.submit(rows, slot)            # warm-up (first launches, tensor maps)
    slot.done.synchronize()
    h0 = time.perf_counter()
    w.submit(rows, slot)
    enq = time.perf_counter() - h0
    slot.done.synchronize()
    total = time.perf_counter() - h0
    assert enq < 0.03 and total >= 0.05


def test_redispatched_labels_equal_local_teacher_after_failure():
    """a dead teacher's queued kernels must not overwrite the
    replacement's slots. Kill t1 with batches in flight and check every
    consumed iteration's labels byte-for-byte against a local teacher."""
    from paper_2207_06667_b200 import formats, nnkit
    from paper_2207_06667_b200.data import DeviceDataset, DeviceShardSampler
    from paper_2207_06667_b200.reader import DistilReader, EventLog, SchedulerConfig, TeacherPool
    from paper_2207_06667_b200.teacher import TeacherConfig, TeacherWorker
    dd = DeviceDataset(formats.make_blobs(0, 4096, 64, 10, 0.8))
    teacher = nnkit.Model.from_host(formats.init_model((64, 512, 512, 10), 3))
    pool = TeacherPool()
    # t1 is slow (its stream is still busy when it dies), t2 takes over
    victim = TeacherWorker(TeacherConfig("t1", 2.0, 4, simulated_delay=0.02), teacher, dd)
    pool.register(victim)
    pool.register(TeacherWorker(TeacherConfig("t2", 2.0, 4), teacher, dd))
    sampler = DeviceShardSampler(dd, 1, 0, 64, seed=0)
    reader = DistilReader("student-0", pool, SchedulerConfig(lt=2, ut=8, probe_interval=0.0, acquire_cooldown=0.0,
                                                             pipeline_depth=4),
                          sampler, 0, 24, 1, EventLog(), 2.0, 4)
    assert reader.acquire(1) == 1
    reader.pump()
    assert len(reader._teachers["t1"].outstanding) == 4
    victim.stop()
    check = DeviceShardSampler(dd, 1, 0, 64, seed=0)
    for i in range(24):
        soft = reader.consume(i, timeout=30)
        torch.cuda.current_stream().synchronize()
        want = nnkit.teacher_soft_labels(teacher, check.batch_for(i).inputs, 2.0, 4)
        assert torch.equal(soft.probs, want.probs) and torch.equal(soft.classes, want.classes), i
        if soft.batch is not None:
            assert torch.equal(soft.batch.inputs, check.batch_for(i).inputs)
    led = reader.ledger()
    assert led["ok"] and led["redispatches"] >= 1
    reader.close()
    torch.cuda.synchronize()
