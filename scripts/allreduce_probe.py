"""Cost of the student's gradient exchange at N GPUs, and what the symmetric-
memory plumbing offers on this box (peer pointers, NVLS multicast).

    torchrun --nproc-per-node N scripts/allreduce_probe.py
"""

import json
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def timeit(fn, iters=20, warm=5):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    dist.barrier()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters):
        fn()
    e.record()
    torch.cuda.synchronize()
    t = torch.tensor([s.elapsed_time(e) / iters * 1e3], device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return round(t.item(), 2)


def main():
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    n = 3072 * 2048 + 2048 + 2048 * 1024 + 1024 + 1024 * 1008 + 1008   # cfg3 student params (padded logits)
    g = torch.randn(n, device=dev)
    res = {"world": dist.get_world_size(), "numel": n, "MB": n * 4 / 1e6}
    res["nccl_all_reduce_us"] = timeit(lambda: dist.all_reduce(g))
    # the student's actual exchange: NCCL all-reduce + SGD vs the fused NVLS kernel
    from paper_2207_06667_b200 import formats, nnkit
    from paper_2207_06667_b200.exchange import NvlsGradientExchange
    sh = formats.init_model((3072, 2048, 1024, 1000), 0)
    m1 = nnkit.Model.from_host(sh, dev)
    ws1 = nnkit.Workspace(m1, 64)
    ws1.grads.flat.normal_()

    def nccl_sgd():
        dist.all_reduce(ws1.grads.flat)
        nnkit.sgd_step(m1, ws1.grads, 1e-9, dist.get_world_size())
    res["nccl_all_reduce_plus_sgd_us"] = timeit(nccl_sgd)
    m2 = nnkit.Model.from_host(sh, dev)
    ws2 = nnkit.Workspace(m2, 64)
    ex = NvlsGradientExchange(m2, ws2.grads)
    ws2.grads.flat.normal_()
    res["nvls_fused_exchange_sgd_us"] = timeit(lambda: ex.step(1e-9))
    res["nvls_blocks_env"] = os.environ.get("EDL_NVLS_BLOCKS", "default")
    try:
        import torch.distributed._symmetric_memory as symm
        buf = symm.empty(n, device=dev, dtype=torch.float32)
        h = symm.rendezvous(buf, dist.group.WORLD.group_name)
        res["symm_buffer_ptrs"] = len(h.buffer_ptrs)
        res["symm_multicast_ptr"] = bool(getattr(h, "multicast_ptr", 0))
        res["symm_signal_pad_size"] = h.signal_pad_size if hasattr(h, "signal_pad_size") else None
        buf.copy_(g)
        for name in ("multimem_all_reduce_", "one_shot_all_reduce", "two_shot_all_reduce_"):
            op = getattr(torch.ops.symm_mem, name, None)
            if op is None:
                continue
            try:
                if name == "one_shot_all_reduce":
                    res[name + "_us"] = timeit(lambda: op(buf, "sum", dist.group.WORLD.group_name))
                else:
                    res[name + "_us"] = timeit(lambda: op(buf, "sum", dist.group.WORLD.group_name))
            except Exception as ex:   # noqa: BLE001
                res[name + "_err"] = str(ex)[:160]
    except Exception as ex:   # noqa: BLE001
        res["symm_err"] = str(ex)[:300]
    if dist.get_rank() == 0:
        print(json.dumps(res))
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
