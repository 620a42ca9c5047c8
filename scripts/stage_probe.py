"""Per-kernel error anatomy at cfg3 (B200): for the teacher's first hidden
layer and the student's stages, the device's bf16 output vs fp64 on the same
bf16 operands, binned by |value| (absolute and ulp-relative errors).

    python scripts/stage_probe.py [--out gpurun_out/stage_probe.json]
"""

import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import nnkit_ref as ref  # noqa: E402
from paper_2207_06667_b200 import _lib, formats, nnkit  # noqa: E402
from paper_2207_06667_b200.data import DeviceDataset, DeviceShardSampler  # noqa: E402

B, D, K, T = 4096, 3072, 1000, 2.0


def anatomy(dev, t, z=None):
    a = np.abs(t)
    ulp = np.where(a > 0, np.exp2(np.floor(np.log2(np.where(a > 0, a, 1.0))) - 7), 2.0 ** -133)
    err = np.abs(dev - t)
    r = err / ulp
    out = {"worst_ulp": float(r.max()), "frac_gt_half_ulp": float((r > 0.5).mean()),
           "frac_gt_1ulp": float((r > 1).mean())}
    i = np.unravel_index(np.argmax(r), r.shape)
    out["worst"] = {"t": float(t[i]), "dev": float(dev[i]), "err": float(err[i])}
    if z is not None:
        out["worst"]["z"] = float(z[i])
    bins = [0, 1e-4, 1e-3, 1e-2, 1e-1, 1.0]
    out["bins"] = []
    for lo, hi in zip(bins[:-1], bins[1:]):
        m = (a >= lo) & (a < hi)
        if m.any():
            out["bins"].append({"range": [lo, hi], "n": int(m.sum()), "max_abs_err": float(err[m].max()),
                                "max_ulp": float(r[m].max()), "frac_gt_1ulp": float((r[m] > 1).mean())})
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "stage_probe.json"))
    a = ap.parse_args()
    torch.cuda.set_device(0)
    host = formats.make_blobs(0, 8192, D, K, 1.0)
    data = DeviceDataset(host)
    sampler = DeviceShardSampler(data, 1, 0, B, seed=0)
    th = formats.init_model((D, 8192, 8192, K), 1)
    teacher = nnkit.Model.from_host(th)
    batch = sampler.batch_for(0)
    res = {}
    for mode in (0, 1):
        _lib.call("edl_set_tanh_mode", mode)
        ws = nnkit.Workspace(teacher, B)
        nnkit.teacher_soft_labels(teacher, batch.inputs, T, 16, ws=ws)
        torch.cuda.synchronize()
        h = batch.inputs[:256, :D].float().cpu().numpy().astype(np.float64)
        z = h @ ref.bf16(th.weights[0]).T
        dev = ws.acts[1][:256, :8192].float().cpu().numpy().astype(np.float64)
        res[f"teacher_l0_mode{mode}"] = anatomy(dev, np.tanh(z), z)
        # the fp32 pre-activation error alone: the device's dense linear (no
        # tanh) on the same operands
        zdev = torch.empty(256, 8192, dtype=torch.float32, device="cuda")
        _lib.call("edl_linear_fwd", batch.inputs.data_ptr(), batch.inputs.stride(0), teacher.w_bf16(0).data_ptr(),
                  teacher.layout.dims_p[0], teacher.b(0).data_ptr(), zdev.data_ptr(), zdev.stride(0), 256, 8192,
                  teacher.layout.dims_p[0], _lib.EDL_ACT_NONE, torch.cuda.current_stream().cuda_stream)
        zd = zdev.cpu().numpy().astype(np.float64)
        e = np.abs(zd - z)
        res[f"teacher_l0_preact_mode{mode}"] = {"max_abs_err": float(e.max()), "mean_abs_err": float(e.mean()),
                                                "max_rel_err_over_rowmax": float((e / np.abs(z).max(axis=1, keepdims=True)).max()),
                                                "max_abs_z": float(np.abs(z).max())}
        # tanh alone on the device's fp32 pre-activation
        res[f"teacher_l0_tanh_of_device_z_mode{mode}"] = anatomy(dev, np.tanh(zd), zd)
        print(json.dumps({k: v for k, v in res.items() if k.endswith(f"mode{mode}")}), flush=True)
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    with open(a.out, "w") as fh:
        json.dump(res, fh, indent=1)


if __name__ == "__main__":
    main()
