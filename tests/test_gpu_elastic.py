"""Elastic teacher pool with teacher PROCESSES (elastic.py) on a B200 —
BASELINE configs[4]'s fault test: teachers are SIGKILLed with batches in
flight and new teacher processes join mid-run; every batch must be trained
exactly once (ledger) and the student's trajectory must be bit-identical to
the fault-free in-process run (edl/student_node.py:492-523,
edl/coordinator.py:133-146,174-187, edl/harness.py:638-642).

All processes share cuda:0 here (CUDA IPC within one device), so the test
runs on the driver's one-GPU box; the two-GPU variant (teacher on cuda:1,
its head kernel writing over NVLink) runs when a second GPU is visible."""

import os
import subprocess
import sys
import time

import numpy as np
import pytest
import torch

pytestmark = [pytest.mark.gpu, pytest.mark.timeout(600)]
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DIMS, TSEED = (8, 32, 6), 11
DATA = (1, 512, 8, 6, 1.0)


LOGS: list = []


def spawn_teacher(path, name, device=0, delay=0.0):
    env = dict(os.environ, PYTHONPATH=ROOT + os.pathsep + os.environ.get("PYTHONPATH", ""))
    cmd = [sys.executable, "-u", "-m", "paper_2207_06667_b200.elastic", "--control", path, "--node-id", name,
           "--device", str(device), "--teacher-dims", ",".join(map(str, DIMS)), "--teacher-seed", str(TSEED),
           "--data", ",".join(map(str, DATA)), "--simulated-delay", str(delay)]
    log = f"{path}.{name}.log"
    LOGS.append(log)
    with open(log, "w") as fh:       # a file, not a pipe nobody drains
        return subprocess.Popen(cmd, cwd=ROOT, env=env, stdout=fh, stderr=subprocess.STDOUT)


def teacher_logs() -> str:
    out = []
    for log in LOGS:
        try:
            with open(log) as fh:
                out.append(f"--- {os.path.basename(log)}\n{fh.read()[-3000:]}")
        except OSError:
            pass
    return "\n".join(out)


def wait_registered(cb, names, procs, timeout=300):
    """Until every named teacher is registered (available, or already
    acquired); `procs` are those teachers' processes."""
    end = time.time() + timeout
    while time.time() < end:
        if all(cb.teacher_status(n) in ("AVAILABLE", "ASSIGNED") for n in names):
            return
        for p in procs:
            if p.poll() is not None:
                raise RuntimeError(f"teacher process exited early:\n{teacher_logs()}")
        time.sleep(0.1)
    raise TimeoutError(f"teachers {names} did not register")


def student_cfg(teacher_count=2):
    from paper_2207_06667_b200.nnkit import TrainConfig
    from paper_2207_06667_b200.reader import SchedulerConfig
    from paper_2207_06667_b200.student import DataSpec, StudentConfig
    spec = DataSpec(seed=DATA[0], n=DATA[1], dim=DATA[2], classes=DATA[3], spread=DATA[4])
    train = TrainConfig(eta=0.05, alpha=0.5, beta=0.5, temperature=2.0, batch_size=16, seed=2)
    return StudentConfig(mode="edl", data=spec, train=train, epochs=2, k=4, teacher_count=teacher_count,
                         sched=SchedulerConfig(lt=2, ut=6, probe_interval=0.0, acquire_cooldown=0.0),
                         consume_timeout=120.0)


def local_run():
    from paper_2207_06667_b200 import formats
    from paper_2207_06667_b200.reader import TeacherPool
    from paper_2207_06667_b200.student import StudentNode, spawn_teachers
    pool = TeacherPool()
    node = StudentNode(student_cfg(), pool=pool)
    spawn_teachers(pool, formats.init_model(DIMS, TSEED), 2, {str(node.dataset.device): node.dataset}, 2.0, 4)
    return node.run()


@pytest.fixture
def control(tmp_path):
    from paper_2207_06667_b200.elastic import ControlBlock
    path = f"/dev/shm/edl-test-{os.getpid()}-{time.monotonic_ns()}"
    cb = ControlBlock(path, create=True, max_students=2, max_teachers=8, max_slots=64, ring_len=16)
    procs = []
    yield cb, path, procs
    cb.request_shutdown()
    for p in procs:
        try:
            p.wait(30)
        except subprocess.TimeoutExpired:
            p.kill()
            p.wait()
    cb.close()
    os.unlink(path)
    for log in LOGS:
        if log.startswith(path):
            try:
                os.unlink(log)
            except OSError:
                pass


def remote_run(cb, path, procs, faults=(), device=0):
    from paper_2207_06667_b200.elastic import ElasticPool
    from paper_2207_06667_b200.student import StudentNode
    named = {"t1": spawn_teacher(path, "t1", device), "t2": spawn_teacher(path, "t2", device)}
    procs += list(named.values())
    wait_registered(cb, ["t1", "t2"], list(named.values()))
    pool = ElasticPool(cb, 0, ttl=10.0, reply_timeout=60.0)
    node = StudentNode(student_cfg(), pool=pool)
    log = []

    def hook(it, reader):
        for kind, at, name in faults:
            if it != at:
                continue
            if kind == "kill":
                pool.kill(name)
                log.append(("kill", name, it))
            elif kind == "add":
                named[name] = spawn_teacher(path, name, device)
                procs.append(named[name])
                log.append(("add", name, it))
            elif kind == "await":
                wait_registered(cb, [name], [named[name]])
    try:
        res = node.run(on_iteration=hook)
    except Exception as exc:
        ents = [(bytes(e["node_id"]).rstrip(b"\0").decode(), int(e["state"]), int(e["pid"]), int(e["epoch"]),
                 int(e["head"]), int(e["tail"]), int(e["served"])) for e in cb.teachers if int(e["state"])]
        raise RuntimeError(f"{exc!r}\nlog={log}\nteachers={ents}\nevents={node.events.entries[-12:]}\n"
                           f"pool={pool.events[-8:]}\n{teacher_logs()}") from exc
    return res, node, pool, log


def test_teacher_processes_serve_identical_soft_labels(control):
    """Two teacher processes, no faults: the trajectory equals the
    in-process run's bit for bit (same kernels, same rows)."""
    from oracle import nnkit_ref as ref
    cb, path, procs = control
    res, node, pool, _ = remote_run(cb, path, procs)
    base = local_run()
    assert res.ledger["ok"] and res.ledger["consumed"] == node.total_steps
    a = ref.flatten(base.model.weights, base.model.biases)
    b = ref.flatten(res.model.weights, res.model.biases)
    assert np.array_equal(a, b)
    served = [int(cb.teachers["served"][j]) for j in range(len(cb.teachers))]
    assert sum(served) >= node.total_steps and sum(1 for v in served if v > 0) == 2   # JSQ used both


def test_sigkill_and_readd_teacher_processes_mid_run(control):
    """configs[4]: t1 is SIGKILLed with batches in flight, t3 joins, then t2
    is killed too; the run completes with every batch consumed exactly once
    and a trajectory identical to the fault-free run."""
    from oracle import nnkit_ref as ref
    cb, path, procs = control
    faults = [("kill", 5, "t1"), ("add", 8, "t3"), ("await", 14, "t3"), ("kill", 15, "t2"), ("add", 20, "t4")]
    res, node, pool, log = remote_run(cb, path, procs, faults)
    base = local_run()
    assert [f[0] for f in log] == ["kill", "add", "kill", "add"]
    assert res.ledger["ok"] and res.ledger["consumed"] == node.total_steps
    kinds = [e["event"] for e in node.events.entries]
    assert kinds.count("teacher_failure") >= 2
    fails = [e for e in node.events.entries if e["event"] == "teacher_failure"]
    assert all(f["why"] in ("process exited", "revoked", "heartbeat expired") for f in fails)
    assert cb.teacher_status("t1") == "EXPIRED" and cb.teacher_status("t2") == "EXPIRED"
    a = ref.flatten(base.model.weights, base.model.biases)
    b = ref.flatten(res.model.weights, res.model.biases)
    assert np.array_equal(a, b)


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs a second GPU for the NVLink peer write")
def test_teacher_process_on_another_gpu(control):
    """The teacher's head kernel writes the soft labels into the student's
    ring on cuda:0 from cuda:1 (peer stores over NVLink)."""
    from oracle import nnkit_ref as ref
    cb, path, procs = control
    res, node, _, _ = remote_run(cb, path, procs, device=1)
    base = local_run()
    assert res.ledger["ok"]
    assert np.array_equal(ref.flatten(base.model.weights, base.model.biases),
                          ref.flatten(res.model.weights, res.model.biases))


def test_cfg4_resnet_teacher_processes_match_local_teacher(control):
    """cfg4 through the elastic pool: two ResNet-50-style teacher processes
    serve a ResNet-18-style student over HBM-resident image rows (small
    shapes: 32x32 images, width 16, 10 classes); the student's parameters
    equal a run fed by an in-process teacher bit for bit."""
    import torch

    from paper_2207_06667_b200.data import DeviceImageDataset, DeviceShardSampler
    from paper_2207_06667_b200.elastic import ElasticPool
    from paper_2207_06667_b200.reader import DistilReader, EventLog, SchedulerConfig
    from paper_2207_06667_b200.resnet import (ResNetConfig, ResNetStudent, ResNetTeacher, StudentResNetConfig,
                                              init_resnet, init_student_resnet)
    cb, path, procs = control
    B, steps, K, k = 8, 10, 10, 4
    env = dict(os.environ, PYTHONPATH=ROOT + os.pathsep + os.environ.get("PYTHONPATH", ""))
    for name in ("r1", "r2"):
        log = f"{path}.{name}.log"
        LOGS.append(log)
        with open(log, "w") as fh:
            procs.append(subprocess.Popen(
                [sys.executable, "-u", "-m", "paper_2207_06667_b200.elastic", "--control", path, "--node-id", name,
                 "--resnet", f"1,{B},16", "--images", f"3,64,32,{K}"], cwd=ROOT, env=env, stdout=fh,
                stderr=subprocess.STDOUT))
    wait_registered(cb, ["r1", "r2"], procs)
    data = DeviceImageDataset(3, 64, 32, K)
    scfg = StudentResNetConfig(layers=(1, 1, 1, 1), width=16, classes=K, image=32)

    def train(soft_for):
        st = ResNetStudent(init_student_resnet(scfg, 0), batch_size=B)
        sampler = DeviceShardSampler(data, 1, 0, B, seed=0)
        for it in range(steps):
            soft = soft_for(it)
            b = sampler.batch_for(it)
            st.train_step(data.nhwc(b.inputs), b.hard_labels, soft, 0.5, 0.5, 2.0, 0.01)
        torch.cuda.synchronize()
        return st.flat.clone()

    pool = ElasticPool(cb, 0, ttl=10.0, reply_timeout=60.0)
    pool.open(1, 0, B, k, 0, 2.0, K, 16, data.device)
    reader = DistilReader("student-0", pool, SchedulerConfig(lt=2, ut=6, probe_interval=0.0, acquire_cooldown=0.0),
                          DeviceShardSampler(data, 1, 0, B, seed=0), 0, steps, 1, EventLog(), 2.0, k)
    assert reader.acquire(2) == 2
    remote = train(lambda it: reader.consume(it, timeout=120))
    assert reader.ledger()["ok"]
    reader.close()
    teacher = ResNetTeacher(init_resnet(ResNetConfig(image=32, classes=K, width=16), 1), batch_size=B)
    ls = DeviceShardSampler(data, 1, 0, B, seed=0)
    local = train(lambda it: teacher.soft_labels(data.nhwc(ls.batch_for(it).inputs), 2.0, k))
    assert torch.isfinite(remote).all()
    assert torch.equal(remote, local)
