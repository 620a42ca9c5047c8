"""N>1 host logic on CPU: placement / assignment tables, and the two wire
patterns the multi-GPU path uses, exercised with the gloo backend at
world_size 2 (127.0.0.1 rendezvous): the teacher->student point-to-point
soft-label stream in RemoteSoftLabels' posting order, and the student
gradient mean (sum all-reduce then 1/N) against the reference ring oracle."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2207_06667_b200.pool import Placement


@pytest.mark.parametrize("world,nt", [(2, 1), (4, 3), (8, 6), (8, 4), (5, 3), (7, 5)])
def test_every_iteration_served_exactly_once(world, nt):
    pl = Placement(world, nt)
    for s in range(pl.n_students):
        ts = pl.teacher_ranks_of(s)
        assert ts and all(not pl.is_student(t) and pl.student_of(t) == s for t in ts)
        served = []
        for t in ts:
            its = pl.iterations_of(t, s, 3, 40)
            assert all(pl.server(s, i) == t for i in its)
            served += its
        assert sorted(served) == list(range(3, 40))
    # every teacher serves some student
    assert sorted(t for s in range(pl.n_students) for t in pl.teacher_ranks_of(s)) == \
        list(range(pl.n_students, world))


def test_placement_validation():
    with pytest.raises(ValueError):
        Placement(2, 2)
    with pytest.raises(ValueError):
        Placement(3, 0)
    with pytest.raises(ValueError):
        Placement(5, 2)      # 3 students, 2 teachers


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, fn, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        q.put((rank, fn(rank, world)))
    finally:
        dist.destroy_process_group()


def _spawn(fn, world=2):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, fn, q)) for r in range(world)]
    for p in ps:
        p.start()
    out = dict(q.get(timeout=120) for _ in ps)
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    return out


def _softlabel_stream(rank, world):
    """Rank 1 = teacher, rank 0 = student; the same messages as
    pool.teacher_serve / RemoteSoftLabels: one packed (prob, class) buffer
    per iteration (pool.wire_slot) on the pair's own process group
    (pool.pair_groups), receives posted `depth` iterations ahead into a ring."""
    from paper_2207_06667_b200.pool import pair_groups, wire_slot
    pl = Placement(world, 1)
    groups = pair_groups(pl)
    g = groups[(0, 1)]
    B, k, depth, start, end = 8, 4, 3, 0, 11
    if rank == 1:
        for it in pl.iterations_of(1, 0, start, end):
            buf, out = wire_slot(B, k, 2.0, "cpu")
            out.probs.fill_(float(it) + 0.5)
            out.classes.copy_(torch.arange(B * k, dtype=torch.int32).view(B, k) + it)
            dist.isend(buf, 0, group=g).wait()
        return None
    slots = [wire_slot(B, k, 2.0, "cpu") for _ in range(depth)]
    works, got, nxt = {}, [], start
    while nxt < min(start + depth, end):
        works[nxt] = dist.irecv(slots[nxt % depth][0], pl.server(0, nxt), group=groups[(0, pl.server(0, nxt))])
        nxt += 1
    for it in range(start, end):
        works.pop(it).wait()
        _, out = slots[it % depth]
        got.append((float(out.probs[0, 0]), int(out.classes[0, 0])))
        if nxt < end:
            works[nxt] = dist.irecv(slots[nxt % depth][0], pl.server(0, nxt), group=groups[(0, pl.server(0, nxt))])
            nxt += 1
    return got


def test_gloo_softlabel_stream_order():
    out = _spawn(_softlabel_stream)
    assert out[0] == [(float(i) + 0.5, i) for i in range(11)]


def _grad_mean(rank, world):
    g = torch.from_numpy(np.random.default_rng(100 + rank).normal(size=1003))
    t = g.clone()
    dist.all_reduce(t)
    return (g.numpy(), (t / world).numpy())


def test_gloo_gradient_mean_matches_ring_oracle():
    from oracle import nnkit_ref as ref
    out = _spawn(_grad_mean)
    ins = [out[r][0] for r in range(2)]
    assert np.array_equal(out[0][1], out[1][1])                       # bitwise across ranks
    np.testing.assert_allclose(out[0][1], ref.ring_reduce_values(ins), rtol=0, atol=1e-12)
