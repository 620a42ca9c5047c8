"""The HBM-bound kernels of the cfg3 path, one launch each at full size, for
an ncu capture of their DRAM bytes and durations (B200):

  gather_rows      B x pad(D) bf16 rows by index          (edl/student_node.py:145-151)
  sgd_step         9.4 M fp32 params + bf16 copy           (edl/nnkit.py:312-322; N > 1 path)
  (the db column sums run inside the grouped dW launch: see the student-step
   launch list, profiles/r02_student_step_launches.csv)
  kd_loss          B x 1000 fp32 logits -> bf16 dz + loss  (edl/nnkit.py:283-299; dense / K > 2048 path)
  tempered_softmax B x 1000 fp32                           (edl/nnkit.py:193-208; dense API)
  cast_bf16        B x D fp32 host rows -> bf16            (e2e input conversion)
  cast_bf16_f64    B x D fp64 host rows -> bf16

    ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \\
        python scripts/hbm_kernels.py
Without ncu it prints CUDA-event times and algorithmic bytes.
"""

import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2207_06667_b200 import _lib, formats, nnkit  # noqa: E402
from paper_2207_06667_b200.data import DeviceDataset, DeviceShardSampler  # noqa: E402


def timed(fn, iters=20):
    for _ in range(3):
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
    torch.cuda.set_device(0)
    iters = 1 if os.environ.get("NCU") else 20
    B, D, K, k = 4096, 3072, 1000, 16
    s = torch.cuda.current_stream().cuda_stream
    data = DeviceDataset(formats.make_blobs(0, 32768, D, K, 1.0))
    sampler = DeviceShardSampler(data, 1, 0, B, seed=0)
    rows = sampler.rows_for(0)
    out = sampler.batch_for(0)
    student = nnkit.Model.from_host(formats.init_model((D, 2048, 1024, K), 0))
    g = torch.randn(student.layout.size, device="cuda") * 1e-3
    z = torch.randn(B, 1008, device="cuda")
    y = torch.randint(0, K, (B,), device="cuda")
    qv = torch.softmax(torch.randn(B, k, device="cuda"), 1)
    qi = torch.randint(0, K, (B, k), device="cuda").int()
    row, loss = torch.empty(B, device="cuda"), torch.zeros(1, device="cuda")
    ticket = torch.zeros(1, dtype=torch.int32, device="cuda")
    status = torch.zeros(1, dtype=torch.int32, device="cuda")
    dz = torch.empty(B, 1008, dtype=torch.bfloat16, device="cuda")
    p = torch.empty(B, 1000, device="cuda")
    x32 = torch.randn(B, D, device="cuda")
    x64 = x32.double()
    xb = torch.empty(B, D, dtype=torch.bfloat16, device="cuda")
    n = student.layout.size
    kern = {
        "gather_rows": (lambda: _lib.call("edl_gather_rows", data.samples.data_ptr(), data.samples.stride(0),
                                          rows.data_ptr(), out.inputs.data_ptr(), out.inputs.stride(0), B, D,
                                          data.labels.data_ptr(), out.hard_labels.data_ptr(), s),
                        2 * B * D * 2 + B * 8 * 3),
        "sgd_step": (lambda: _lib.call("edl_sgd_step", student.flat.data_ptr(), student.flat_bf16.data_ptr(),
                                       g.data_ptr(), n, 1e-3, s), n * (4 + 4 + 4 + 2)),
        "kd_loss": (lambda: _lib.call("edl_kd_loss_fwd_bwd", z.data_ptr(), 1008, y.data_ptr(), qv.data_ptr(),
                                      qi.data_ptr(), B, K, k, 0.5, 0.5, 2.0, row.data_ptr(), loss.data_ptr(),
                                      ticket.data_ptr(), dz.data_ptr(), 1008, status.data_ptr(), s),
                    B * (4 * K + 2 * 1008 + 8 * k + 12)),
        "tempered_softmax": (lambda: _lib.call("edl_tempered_softmax", z.data_ptr(), 1008, p.data_ptr(), 1000, B, K,
                                               2.0, s), B * K * 8),
        "cast_bf16": (lambda: _lib.call("edl_cast_bf16", x32.data_ptr(), D, xb.data_ptr(), D, B, D, s),
                      B * D * 6),
        "cast_bf16_f64": (lambda: _lib.call("edl_cast_bf16_f64", x64.data_ptr(), D, xb.data_ptr(), D, B, D, s),
                          B * D * 10),
    }
    res = {}
    for name, (fn, alg) in kern.items():
        t = timed(fn, iters)
        res[name] = {"us": round(t, 2), "algorithmic_bytes": alg, "GB_per_s": round(alg / t / 1e3, 1)}
    print(json.dumps(res))


if __name__ == "__main__":
    main()
