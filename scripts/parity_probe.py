"""Measured parity of the cfg3 device path against the fp64 oracle (B200).

For each tanh mode of the forward epilogues (1 = tanhf, 0 = tanh.approx):
  * teacher: fused head top-16 on a 256-row slice of a B = 4096 batch vs the
    bf16-storage oracle (relative error of every probability, ids) and the
    plain fp64 oracle (ids on gap-safe rows);
  * student: kd_loss at B = 4096 vs kd_loss_bf16_storage on the full batch
    (loss, per-layer dW / db relative norms and max elementwise error).

    python scripts/parity_probe.py [--rows 256] [--out gpurun_out/parity_probe.json]
"""

import argparse
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import nnkit_ref as ref  # noqa: E402
from paper_2207_06667_b200 import _lib, formats, nnkit  # noqa: E402
from paper_2207_06667_b200.data import DeviceDataset, DeviceShardSampler  # noqa: E402

B, D, K, k, T = 4096, 3072, 1000, 16, 2.0


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rows", type=int, default=256)
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "parity_probe.json"))
    ap.add_argument("--modes", default="1,0")
    a = ap.parse_args()
    torch.cuda.set_device(0)
    host_data = formats.make_blobs(0, 8192, D, K, 1.0)
    data = DeviceDataset(host_data)
    sampler = DeviceShardSampler(data, 1, 0, B, seed=0)
    teacher_h = formats.init_model((D, 8192, 8192, K), 1)
    student_h = formats.init_model((D, 2048, 1024, K), 0)
    teacher = nnkit.Model.from_host(teacher_h)
    tw, tb = list(teacher_h.weights), list(teacher_h.biases)
    sw, sb = list(student_h.weights), list(student_h.biases)
    out = {"rows": a.rows}
    batch = sampler.batch_for(0)
    rows = sampler.rows_for(0).cpu().numpy()
    x = host_data.samples[rows]
    y = host_data.labels[rows]
    t0 = time.time()
    xs = x[:a.rows]
    z64 = ref.forward(tw, tb, xs)
    z16 = ref.forward_bf16_storage(tw, tb, xs)
    p16 = ref.tempered_softmax(z16, T)
    p64 = ref.tempered_softmax(z64, T)
    out["oracle_teacher_s"] = round(time.time() - t0, 2)
    for mode in [int(m) for m in a.modes.split(",")]:
        _lib.call("edl_set_tanh_mode", mode)
        res = {}
        soft = nnkit.teacher_soft_labels(teacher, batch.inputs, T, k)
        torch.cuda.synchronize()
        vals = soft.probs.cpu().numpy().astype(np.float64)
        idx = soft.classes.cpu().numpy().astype(np.int64)
        vs, ix = vals[:a.rows], idx[:a.rows]
        ref16 = np.take_along_axis(p16, ix, axis=1)
        r = np.abs(vs - ref16) / ref16
        res["teacher_prob_rel_vs_bf16_oracle"] = {"max": float(r.max()), "mean": float(r.mean()),
                                                  "p99": float(np.quantile(r, 0.99))}
        ref64 = np.take_along_axis(p64, ix, axis=1)
        r64 = np.abs(vs - ref64) / ref64
        res["teacher_prob_rel_vs_fp64"] = {"max": float(r64.max()), "mean": float(r64.mean())}
        for name, zz in (("fp64", z64), ("bf16", z16)):
            zs = np.sort(zz, axis=1)[:, ::-1]
            order = np.argsort(-zz, axis=1, kind="stable")[:, :k]
            for gap in (1e-3, 1e-2):
                safe = (zs[:, k - 1] - zs[:, k]) > gap
                res[f"ids_vs_{name}_gap{gap:g}"] = {
                    "safe_frac": float(safe.mean()),
                    "exact_frac_on_safe": float((ix[safe] == order[safe]).all(axis=1).mean()),
                    "exact_frac_all": float((ix == order).all(axis=1).mean())}
        # student, full batch
        student = nnkit.Model.from_host(student_h)
        cfg = nnkit.TrainConfig(eta=0.05, alpha=0.5, beta=0.5, temperature=T, batch_size=B)
        loss, grads = nnkit.kd_loss(student, batch, soft, cfg)
        lv = float(loss)
        L = student.layout
        g = grads.flat.cpu().numpy().astype(np.float64)
        t0 = time.time()
        q = ref.topk_dense(vals, idx, K)
        l16, gw16, gb16 = ref.kd_loss_bf16_storage(sw, sb, x, y, q, 0.5, 0.5, T)
        l64, gw64, gb64 = ref.kd_loss(sw, sb, x, y, q, 0.5, 0.5, T)
        res["oracle_student_s"] = round(time.time() - t0, 2)
        res["loss"] = {"device": lv, "bf16_oracle": l16, "fp64": l64,
                       "rel_vs_bf16_oracle": abs(lv - l16) / abs(l16), "rel_vs_fp64": abs(lv - l64) / abs(l64)}
        layers = []
        for l in range(L.layers):
            r_, c_ = student.layer_dims[l + 1], student.layer_dims[l]
            dw = g[L.w_off[l]:L.w_off[l] + L.dims_p[l + 1] * L.dims_p[l]].reshape(L.dims_p[l + 1], L.dims_p[l])
            dw = dw[:r_, :c_]
            db = g[L.b_off[l]:L.b_off[l] + r_]
            layers.append({"layer": l,
                           "dW_rel_vs_bf16_oracle": rel(dw, gw16[l]), "db_rel_vs_bf16_oracle": rel(db, gb16[l]),
                           "dW_rel_vs_fp64": rel(dw, gw64[l]), "db_rel_vs_fp64": rel(db, gb64[l]),
                           "dW_maxabs_over_maxref_bf16": float(np.abs(dw - gw16[l]).max() / np.abs(gw16[l]).max())})
        res["grads"] = layers
        out[f"tanh_mode_{mode}"] = res
        print(json.dumps({f"tanh_mode_{mode}": res}), flush=True)
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    with open(a.out, "w") as fh:
        json.dump(out, fh, indent=1)


if __name__ == "__main__":
    main()
