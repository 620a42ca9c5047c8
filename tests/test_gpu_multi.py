"""Multi-student and multi-GPU paths on the device.

* 2-student data parallelism vs the reference's own VirtualCluster trajectory
  (edl/harness.py:411-433, golden `vc_final`): emulated on one GPU (the two
  students' flat gradients summed, mean folded into SGD exactly as the NCCL
  path does), and with real NCCL processes when >= 2 GPUs are visible.
* configs[4] fault test with the teacher pool on ANOTHER GPU (soft labels
  cross NVLink as peer copies on the teacher's side stream): teachers are
  killed with batches in flight and re-added; the ledger stays exact and the
  trajectory equals the fault-free run.
"""

import os
import socket

import numpy as np
import pytest
import torch

from oracle import nnkit_ref as ref

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _golden():
    return np.load(os.path.join(GOLD, "cfg1.npz"))


def _host(flat, dims):
    from paper_2207_06667_b200.formats import HostModel
    ws, bs = ref.unflatten(flat, dims)
    return HostModel(tuple(dims), tuple(ws), tuple(bs))


def test_two_students_emulated_on_one_gpu_vs_virtual_cluster():
    from paper_2207_06667_b200 import formats, nnkit
    from paper_2207_06667_b200.data import DeviceDataset, DeviceShardSampler
    d = _golden()
    data = DeviceDataset(formats.make_blobs(0, 2048, 16, 10, 1.0))
    teacher = nnkit.Model.from_host(_host(d["teacher"], (16, 256, 256, 10)))
    cfg = nnkit.TrainConfig(eta=0.05, alpha=0.5, beta=0.5, temperature=2.0, batch_size=32)
    s0 = _host(d["student0"], (16, 64, 10))
    students = [nnkit.Model.from_host(s0) for _ in range(2)]
    samplers = [DeviceShardSampler(data, 2, r, 32, seed=0) for r in range(2)]
    wss = [nnkit.Workspace(students[r], 32) for r in range(2)]
    for it in range(int(d["vc_steps"])):
        grads = []
        for r in range(2):
            b = samplers[r].batch_for(it)
            soft = nnkit.teacher_soft_labels(teacher, b.inputs, 2.0, 10)
            _, g = nnkit.kd_loss(students[r], b, soft, cfg, ws=wss[r])
            grads.append(g.flat.clone())
        total = nnkit.Gradients(grads[0] + grads[1], wss[0].grads.layout)   # the all-reduce (sum)
        for r in range(2):
            nnkit.sgd_step(students[r], total, cfg.eta, world_size=2)
    p0, p1 = nnkit.flatten_params(students[0]), nnkit.flatten_params(students[1])
    assert np.array_equal(p0, p1)
    rel = np.linalg.norm(p0 - d["vc_final"]) / np.linalg.norm(d["vc_final"])
    assert rel < 2e-2, rel


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _nccl_student(rank, world, port, q, exchange="nccl", overlap=False):
    import torch.distributed as dist

    from paper_2207_06667_b200 import formats
    from paper_2207_06667_b200.nnkit import TrainConfig
    from paper_2207_06667_b200.student import DataSpec, StudentConfig, StudentNode
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", rank))
    try:
        d = _golden()
        cfg = StudentConfig(rank=rank, world_size=world, mode="online",
                            data=DataSpec(seed=0, n=2048, dim=16, classes=10, spread=1.0),
                            train=TrainConfig(eta=0.05, alpha=0.5, beta=0.5, temperature=2.0, batch_size=32),
                            max_steps=int(d["vc_steps"]), k=10, exchange=exchange, overlap_exchange=overlap)
        node = StudentNode(cfg, teacher_model=_host(d["teacher"], (16, 256, 256, 10)))
        res = node.run()
        q.put((rank, ref.flatten(list(res.model.weights), list(res.model.biases))))
    finally:
        dist.destroy_process_group()


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs 2 GPUs")
@pytest.mark.parametrize("exchange,overlap", [("nccl", False), ("nccl", True), ("nvls", False)])
def test_two_students_nccl_vs_virtual_cluster(exchange, overlap):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_nccl_student, args=(r, 2, port, q, exchange, overlap)) for r in range(2)]
    for p in ps:
        p.start()
    out = dict(q.get(timeout=300) for _ in ps)
    for p in ps:
        p.join(timeout=120)
        assert p.exitcode == 0
    d = _golden()
    assert np.array_equal(out[0], out[1])                    # bitwise identical replicas across ranks
    rel = np.linalg.norm(out[0] - d["vc_final"]) / np.linalg.norm(d["vc_final"])
    assert rel < 2e-2, rel


def _exchange_rank(rank, world, port, q):
    import torch.distributed as dist

    from paper_2207_06667_b200 import formats
    from paper_2207_06667_b200.exchange import ExchangeUnavailable, NvlsGradientExchange
    from paper_2207_06667_b200.nnkit import Model, Workspace
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", rank))
    try:
        dims = (200, 96, 37)                      # padded layout with ragged tails
        model = Model.from_host(formats.init_model(dims, 3))
        ws = Workspace(model, 8)
        try:
            ex = NvlsGradientExchange(model, ws.grads)
        except ExchangeUnavailable as e:
            q.put((rank, "unavailable", str(e)))
            return
        n = model.layout.size
        eta = 0.07
        p = model.flat.clone()
        out = []
        for epoch in range(3):
            gens = [torch.Generator().manual_seed(100 * epoch + r) for r in range(world)]
            gs = [torch.randn(n, generator=g) for g in gens]
            ws.grads.flat.copy_(gs[rank].cuda())
            ex.step(eta)
            torch.cuda.synchronize()
            want = p.cpu() - (eta / world) * torch.stack(gs).sum(0)
            out.append((model.flat.cpu().numpy().copy(), want.numpy(),
                        bool(torch.equal(model.flat_bf16.cpu(), model.flat.cpu().to(torch.bfloat16)))))
            p = model.flat.clone()
        q.put((rank, "ok", out))
    finally:
        dist.destroy_process_group()


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs 2 GPUs")
def test_nvls_exchange_sgd_matches_mean_update():
    """edl_nvls_allreduce_sgd: every replica equals p - eta * mean_r(g_r)
    (edl/allreduce.py:77-120 + edl/nnkit.py:312-322), bitwise identical across
    ranks, bf16 copy = bf16(fp32 master), over consecutive epochs."""
    import torch.multiprocessing as mp
    world = min(torch.cuda.device_count(), 4)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_exchange_rank, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = dict((r, (status, payload)) for r, status, payload in (q.get(timeout=300) for _ in ps))
    for p in ps:
        p.join(timeout=120)
        assert p.exitcode == 0
    if any(st == "unavailable" for st, _ in res.values()):
        pytest.skip(f"no NVLS multicast: {res[0][1]}")
    for epoch in range(3):
        ref0 = res[0][1][epoch][0]
        for r in range(world):
            got, want, bf_ok = res[r][1][epoch]
            assert np.array_equal(got, ref0)                  # identical replicas
            np.testing.assert_allclose(got, want, rtol=1e-6, atol=1e-6)
            assert bf_ok


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs 2 GPUs")
def test_teacher_gpu_drop_and_readd_over_nvlink():
    from paper_2207_06667_b200 import formats
    from paper_2207_06667_b200.data import DeviceDataset
    from paper_2207_06667_b200.nnkit import Model, TrainConfig
    from paper_2207_06667_b200.reader import SchedulerConfig, TeacherPool
    from paper_2207_06667_b200.student import DataSpec, StudentConfig, StudentNode
    from paper_2207_06667_b200.teacher import TeacherConfig, TeacherWorker
    spec = DataSpec(seed=1, n=512, dim=8, classes=6, spread=1.0)
    teacher_h = formats.init_model((8, 32, 6), 11)
    train = TrainConfig(eta=0.05, alpha=0.5, beta=0.5, temperature=2.0, batch_size=16, seed=2)

    def run(faults):
        torch.cuda.set_device(0)
        cfg = StudentConfig(mode="edl", data=spec, train=train, epochs=2, k=4, teacher_count=2,
                            sched=SchedulerConfig(lt=2, ut=6, probe_interval=0.0, acquire_cooldown=0.0))
        pool = TeacherPool()
        node = StudentNode(cfg, pool=pool)
        dev1 = torch.device("cuda", 1)
        data1 = DeviceDataset(spec.build(), dev1)        # teacher GPU's replica of the dataset
        with torch.cuda.device(dev1):
            tmodel = Model.from_host(teacher_h, dev1)
        for i in range(3):
            pool.register(TeacherWorker(TeacherConfig(f"t{i + 1}", 2.0, 4), tmodel, data1))

        def hook(it, reader):
            for kind, at, name in faults:
                if it == at and kind == "kill":
                    pool.kill(name)
                if it == at and kind == "add":
                    pool.register(TeacherWorker(TeacherConfig(name, 2.0, 4), tmodel, data1))
        return node.run(on_iteration=hook), node

    clean, _ = run([])
    faulty, node = run([("kill", 4, "t1"), ("kill", 9, "t2"), ("add", 11, "t9"), ("kill", 20, "t3")])
    assert clean.ledger["ok"] and faulty.ledger["ok"]
    kinds = [e["event"] for e in node.events.entries]
    assert kinds.count("teacher_failure") >= 2 and "teacher_replaced" in kinds
    a = ref.flatten(list(clean.model.weights), list(clean.model.biases))
    b = ref.flatten(list(faulty.model.weights), list(faulty.model.biases))
    assert np.array_equal(a, b)


def _peer_ring_rank(rank, world, port, q):
    import torch.distributed as dist

    from paper_2207_06667_b200 import formats, nnkit
    from paper_2207_06667_b200.data import DeviceDataset, DeviceShardSampler
    from paper_2207_06667_b200.pool import PeerSoftLabelRing, PeerSoftLabels, Placement, teacher_serve
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    dev = torch.device("cuda", rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)
    try:
        pl = Placement(world, world - 1)                 # rank 0 student, the rest teachers
        B, k, T, n_it = 64, 8, 2.0, 23
        data = DeviceDataset(formats.make_blobs(0, 1024, 40, 30, 1.0), dev)
        teacher = nnkit.Model.from_host(formats.init_model((40, 96, 30), 5), dev)
        try:
            ring = PeerSoftLabelRing(pl, rank, B, k, T, dev, depth=3)
        except Exception as e:   # noqa: BLE001
            q.put((rank, "unavailable", str(e)[:200]))
            return
        if rank == 0:
            rx = PeerSoftLabels(ring)
            sampler = DeviceShardSampler(data, 1, 0, B, seed=0)
            bad = 0
            for it in range(n_it):
                soft = rx.consume(it)
                # the student's own reference: the same teacher on the same rows, locally
                want = nnkit.teacher_soft_labels(teacher, sampler.batch_for(it).inputs, T, k)
                bad += int(not (torch.equal(soft.classes, want.classes) and torch.equal(soft.probs, want.probs)))
                torch.cuda._sleep(2_000_000)             # a slow student: teachers must wait for credits
                rx.released(it)
            torch.cuda.synchronize()
            q.put((rank, "ok", bad))
        else:
            served = teacher_serve(pl, rank, teacher, data, B, 0, T, k, 0, n_it, ring=ring)
            torch.cuda.synchronize()
            q.put((rank, "ok", served))
        dist.barrier()
    finally:
        dist.destroy_process_group()


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs 2 GPUs")
def test_peer_softlabel_ring_delivers_teacher_outputs():
    """Split placement over NVLink peer memory (pool.PeerSoftLabelRing): each
    iteration's (prob, class) batch lands in the student's ring bitwise equal
    to the teacher head's output for that iteration's rows, in order, with the
    ring (depth 3) wrapping many times behind a deliberately slow student."""
    import torch.multiprocessing as mp
    world = min(torch.cuda.device_count(), 3)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_peer_ring_rank, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = dict((r, (st, v)) for r, st, v in (q.get(timeout=300) for _ in ps))
    for p in ps:
        p.join(timeout=120)
        assert p.exitcode == 0
    if any(st == "unavailable" for st, _ in res.values()):
        pytest.skip(f"no symmetric memory: {res}")
    assert res[0][1] == 0
    assert sum(v for r, (st, v) in res.items() if r > 0) == 23
