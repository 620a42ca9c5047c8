"""The split placement's READY / CREDIT soft-label ring protocol
(pool.PeerSoftLabelRing, the teacher-pool -> student handoff of
edl/student_node.py:369-457) on ONE GPU: every rank's slots and signal pad are
separate buffers on cuda:0 and the teacher and student loops are two streams
of one process, so the driver's one-GPU box exercises the same flag
arithmetic the multi-GPU runs use (stream-ordered waits and writes, no host
blocking). The real 2-/4-GPU versions are in test_gpu_multi.py."""

import numpy as np
import pytest
import torch

pytestmark = [pytest.mark.gpu, pytest.mark.timeout(120)]

B, K, KT = 32, 6, 4


def _setup():
    from paper_2207_06667_b200 import formats, nnkit
    from paper_2207_06667_b200.data import DeviceDataset
    data = DeviceDataset(formats.make_blobs(1, 512, 8, K, 1.0))
    teacher = nnkit.Model.from_host(formats.init_model((8, 32, K), 11))
    student_h = formats.init_model((8, 16, K), 2)
    return nnkit, data, teacher, student_h


def _student_steps(nk, data, student_h, sampler, soft_of, steps, stream=None, delay_ns=0):
    from paper_2207_06667_b200 import _lib
    from paper_2207_06667_b200.student import StudentStep
    cfg = nk.TrainConfig(eta=0.05, alpha=0.5, beta=0.5, temperature=2.0, batch_size=B)
    eng = StudentStep(nk.Model.from_host(student_h), cfg, B, 1, max_steps=steps + 1)
    for it in range(steps):
        soft = soft_of(it)
        batch = sampler.batch_for(it, out=eng.batch, stream=stream)
        if delay_ns:
            _lib.call("edl_stream_delay_ns", delay_ns, (stream or torch.cuda.current_stream()).cuda_stream)
        eng.step(batch, soft)
        yield it, eng
    return


@pytest.mark.parametrize("depth,slow_student", [(2, True), (4, False), (1, True)])
def test_ready_credit_ring_single_gpu_matches_local_teacher(depth, slow_student):
    """Teacher rank 1 serves student rank 0 through the ring (depth 1/2/4);
    a slow student forces the teacher to wait on CREDIT before reusing a
    slot. The student's trajectory equals a run fed by a local teacher."""
    from paper_2207_06667_b200.data import DeviceShardSampler
    from paper_2207_06667_b200.pool import PeerSoftLabelRing, Placement, ring_server
    nk, data, teacher, student_h = _setup()
    steps = 12
    pl = Placement(world=2, n_teachers=1)
    ring = PeerSoftLabelRing.local(pl, B, KT, 2.0, data.device, depth=depth, view_rank=0)
    t_ring = ring.as_rank(1)
    s_stream, t_stream = torch.cuda.Stream(), torch.cuda.Stream()
    sampler = DeviceShardSampler(data, 1, 0, B, seed=0)
    for e in range(2):                 # epoch permutations resident before any flag wait is queued
        sampler.rows_for(e * sampler.batches_per_epoch)
    serve = ring_server(pl, 1, teacher, data, B, 0, 2.0, KT, t_ring)
    student = _student_steps(nk, data, student_h, sampler, lambda i: ring.student_take(i), steps,
                             stream=s_stream, delay_ns=300_000 if slow_student else 0)
    # Interleave the two loops on the host, teacher first: every stream wait
    # queued so far is satisfiable by work already queued on the other
    # stream, so a host call that synchronises the device cannot deadlock
    # (the hazard of stream-memory waits inside one process).
    for it in range(steps):
        with torch.cuda.stream(t_stream):
            serve(it)
        with torch.cuda.stream(s_stream):
            _, eng = next(student)
            ring.student_release(it)
    with torch.cuda.stream(s_stream):
        got = eng.model.flat.clone()
    torch.cuda.synchronize()
    # the same steps with a local teacher on one stream
    sampler2 = DeviceShardSampler(data, 1, 0, B, seed=0)
    out = nk.SoftLabels(torch.empty(B, KT, device="cuda"), torch.empty(B, KT, dtype=torch.int32, device="cuda"), 2.0)

    def local_soft(i):
        return nk.teacher_soft_labels(teacher, sampler2.batch_for(i).inputs, 2.0, KT, out=out)
    for _, eng2 in _student_steps(nk, data, student_h, sampler2, local_soft, steps):
        pass
    torch.cuda.synchronize()
    assert torch.equal(got, eng2.model.flat)
    # every slot's READY word holds the last iteration it carried (+1), the
    # teacher's CREDIT word the student's last consumed iteration (+1)
    ready = ring._pads[0][:depth].cpu().numpy()
    want = [max(i for i in range(steps) if i % depth == j) + 1 for j in range(depth)]
    assert list(ready) == want
    assert int(ring._pads[1][PeerSoftLabelRing.CREDIT].item()) == steps


def test_stream_flags_order_two_streams():
    """edl_stream_wait_geq / edl_stream_write_u32 on cuda:0 memory: the
    consumer stream's copy runs only after the producer's write, even when
    the producer is delayed on the device."""
    from paper_2207_06667_b200 import _lib
    flag = torch.zeros(4, dtype=torch.int32, device="cuda")
    src = torch.zeros(1 << 20, device="cuda")
    dst = torch.zeros_like(src)
    prod, cons = torch.cuda.Stream(), torch.cuda.Stream()
    for rnd in range(1, 4):
        with torch.cuda.stream(cons):
            _lib.call("edl_stream_wait_geq", flag.data_ptr(), rnd, cons.cuda_stream)
            dst.copy_(src)
        with torch.cuda.stream(prod):
            _lib.call("edl_stream_delay_ns", 2_000_000, prod.cuda_stream)
            src.fill_(float(rnd))
            _lib.call("edl_stream_write_u32", flag.data_ptr(), rnd, prod.cuda_stream)
        cons.synchronize()
        assert float(dst.min()) == float(rnd) == float(dst.max())
    assert np.array_equal(flag.cpu().numpy()[:1], [3])
