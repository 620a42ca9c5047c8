"""Same-process A/B timing of the cfg3 step pieces (box-to-box variance on the
pool is ~10-15%, so compare variants inside one run only).

    python scripts/stepbench.py [--iters 30]
"""

import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2207_06667_b200 import formats, nnkit  # noqa: E402
from paper_2207_06667_b200.data import DeviceDataset, DeviceShardSampler  # noqa: E402
from paper_2207_06667_b200.nnkit import Model, SoftLabels, TrainConfig  # noqa: E402
from paper_2207_06667_b200.student import StudentStep  # noqa: E402


def timeit(fn, iters, warm=5):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters * 1e3


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=30)
    ap.add_argument("--tanh-mode", type=int, default=None, help="1 = tanhf, 0 = tanh.approx (edl_set_tanh_mode)")
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    if a.tanh_mode is not None:
        from paper_2207_06667_b200 import _lib
        _lib.call("edl_set_tanh_mode", a.tanh_mode)
    B = 4096
    data = DeviceDataset(formats.make_blobs(0, 16384, 3072, 1000, 1.0), dev)
    sampler = DeviceShardSampler(data, 1, 0, B, seed=0)
    teacher = Model.from_host(formats.init_model((3072, 8192, 8192, 1000), 1), dev)
    sh = formats.init_model((3072, 2048, 1024, 1000), 0)
    cfg = TrainConfig(eta=0.05, alpha=0.5, beta=0.5, temperature=2.0, batch_size=B)
    batch = sampler.batch_for(0)
    tws = nnkit.Workspace(teacher, B)
    soft = SoftLabels(torch.empty(B, 16, device=dev), torch.empty(B, 16, dtype=torch.int32, device=dev), 2.0)
    nnkit.teacher_soft_labels(teacher, batch.inputs, 2.0, 16, out=soft, ws=tws)
    res = {}
    res["teacher_batch_us"] = timeit(lambda: nnkit.teacher_soft_labels(teacher, batch.inputs, 2.0, 16, out=soft,
                                                                       ws=tws), a.iters)
    for fused in (False, True):
        eng = StudentStep(Model.from_host(sh, dev), cfg, B, 1, fuse_sgd=fused)
        res[f"student_step_{'fused' if fused else 'unfused'}_us"] = timeit(lambda: eng.step(batch, soft), a.iters)
    eng = StudentStep(Model.from_host(sh, dev), cfg, B, 1)
    res["online_step_us"] = timeit(lambda: (nnkit.teacher_soft_labels(teacher, batch.inputs, 2.0, 16, out=soft,
                                                                      ws=tws), eng.step(batch, soft)), a.iters)
    res["online_samples_per_s"] = B / res["online_step_us"] * 1e6
    # the same step with a fresh batch gathered every iteration (epoch
    # permutations built on demand, as in bench.py) ...
    ctr = [0]

    def sampled():
        b = sampler.batch_for(ctr[0], out=eng.batch)
        ctr[0] += 1
        nnkit.teacher_soft_labels(teacher, b.inputs, 2.0, 16, out=soft, ws=tws)
        eng.step(b, soft)
    res["online_step_sampled_us"] = timeit(sampled, 96)
    # ... and with the permutations already resident
    for it in range(ctr[0], ctr[0] + 100, sampler.batches_per_epoch):
        sampler.rows_for(it)
    res["online_step_sampled_prewarmed_us"] = timeit(sampled, 16)

    def same_rows():          # gather launched every step, always batch 0's rows
        b = sampler.batch_for(0, out=eng.batch)
        nnkit.teacher_soft_labels(teacher, b.inputs, 2.0, 16, out=soft, ws=tws)
        eng.step(b, soft)
    res["online_step_gather_same_rows_us"] = timeit(same_rows, 30)
    bufs = [sampler.batch_for(i) for i in range(8)]
    ctr[0] = 0

    def rotate():             # 8 pre-gathered batches, no gather launch
        b = bufs[ctr[0] % 8]
        ctr[0] += 1
        nnkit.teacher_soft_labels(teacher, b.inputs, 2.0, 16, out=soft, ws=tws)
        eng.step(b, soft)
    res["online_step_rotate8_us"] = timeit(rotate, 32)
    res["teacher_batch_rotate8_us"] = timeit(
        lambda: nnkit.teacher_soft_labels(teacher, bufs[(ctr.__setitem__(0, ctr[0] + 1) or ctr[0]) % 8].inputs,
                                          2.0, 16, out=soft, ws=tws), 32)
    # order confound check: the fixed-batch variants again, last
    res["teacher_batch_again_us"] = timeit(lambda: nnkit.teacher_soft_labels(teacher, batch.inputs, 2.0, 16, out=soft,
                                                                             ws=tws), a.iters)
    res["online_step_again_us"] = timeit(lambda: (nnkit.teacher_soft_labels(teacher, batch.inputs, 2.0, 16, out=soft,
                                                                            ws=tws), eng.step(batch, soft)), a.iters)
    try:
        import pynvml
        pynvml.nvmlInit()
        h = pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device())
        res["sm_mhz_end"] = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
        res["power_w_end"] = pynvml.nvmlDeviceGetPowerUsage(h) / 1e3
    except Exception:
        pass
    # host enqueue cost of one eager step: tiny cfg2 shapes make the device
    # work negligible, so wall time per step ~ Python + ctypes + launch cost
    import time
    t2 = Model.from_host(formats.init_model((16, 256, 256, 10), 1), dev)
    s2 = StudentStep(Model.from_host(formats.init_model((16, 64, 10), 0), dev),
                     TrainConfig(eta=0.05, alpha=0.5, beta=0.5, temperature=2.0, batch_size=32), 32, 1)
    b2 = nnkit.make_batch(formats.make_blobs(0, 32, 16, 10, 1.0).samples, formats.make_blobs(0, 32, 16, 10, 1.0).labels,
                          dev)
    ws2 = nnkit.Workspace(t2, 32)
    o2 = SoftLabels(torch.empty(32, 10, device=dev), torch.empty(32, 10, dtype=torch.int32, device=dev), 2.0)
    for _ in range(10):
        nnkit.teacher_soft_labels(t2, b2.inputs, 2.0, 10, out=o2, ws=ws2)
        s2.step(b2, o2)
    torch.cuda.synchronize()
    h0 = time.perf_counter()
    for _ in range(200):
        nnkit.teacher_soft_labels(t2, b2.inputs, 2.0, 10, out=o2, ws=ws2)
        s2.step(b2, o2)
    torch.cuda.synchronize()
    res["host_us_per_eager_online_step"] = (time.perf_counter() - h0) / 200 * 1e6
    print(json.dumps({k: round(v, 2) for k, v in res.items()}))


if __name__ == "__main__":
    main()
