"""CPU ORACLE CALIBRATION — test infrastructure only (build container).

The GPU box has no /root/reference, so bench.py's CPU arm times the numpy
port (oracle/nnkit_ref.py). This script times the REAL reference
(pkg/src/edl/nnkit.py, imported from /root/reference) beside the port on the
same cfg3 workload and threads, here, and records the ratio that the bench
line carries as `cpu_baseline.port_calibration`:

  reference step = SoftLabelBatch(tempered_softmax(forward(teacher, X), T))
                   (dense, validated: edl/nnkit.py:113-135, 193-234)
                 + kd_loss + sgd_step (new validated Model, :254-322)
  port step      = the same math through oracle/nnkit_ref.py, with top-16
                   soft labels densified (no validation)

    python oracle/calibrate_port.py [--batch 1024] [--reps 3]
"""

import argparse
import json
import os
import statistics
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
REF_SRC = "/root/reference/pkg/src"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=1024)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r02_port_vs_reference.json"))
    a = ap.parse_args()
    sys.path.insert(0, REF_SRC)
    from edl import nnkit as edl_nnkit  # the real reference

    from oracle import nnkit_ref as ref
    T, alpha, beta, eta, k = 2.0, 0.5, 0.5, 0.05, 16
    tdims, sdims = (3072, 8192, 8192, 1000), (3072, 2048, 1024, 1000)
    tw, tb = ref.init_model(tdims, 1)
    sw, sb = ref.init_model(sdims, 0)
    x, y = ref.make_blobs(0, a.batch, 3072, 1000, 1.0)
    teacher = edl_nnkit.Model(tdims, tuple(tw), tuple(tb))
    student = edl_nnkit.Model(sdims, tuple(sw), tuple(sb))
    cfg = edl_nnkit.TrainConfig(eta=eta, alpha=alpha, beta=beta, temperature=T, batch_size=a.batch)

    def ref_step():
        nonlocal student
        p = edl_nnkit.tempered_softmax(edl_nnkit.forward(teacher, x), T)
        soft = edl_nnkit.SoftLabelBatch(p, T)
        _, g = edl_nnkit.kd_loss(student, edl_nnkit.Batch(x, y), soft, cfg)
        student = edl_nnkit.sgd_step(student, g, eta)

    pw, pb = list(sw), list(sb)

    def port_step():
        nonlocal pw, pb
        p = ref.tempered_softmax(ref.forward(tw, tb, x), T)
        q = ref.topk_dense(*ref.topk(p, k), p.shape[1])
        _, gw, gb = ref.kd_loss(pw, pb, x, y, q, alpha, beta, T)
        pw, pb = ref.sgd_step(pw, pb, gw, gb, eta)

    res = {}
    for name, fn in (("reference", ref_step), ("port", port_step)):
        fn()                                # warm-up
        ts = []
        for _ in range(a.reps):
            t0 = time.perf_counter()
            fn()
            ts.append(time.perf_counter() - t0)
        res[name] = statistics.median(ts)
    try:
        from threadpoolctl import threadpool_info
        threads = [p.get("num_threads") for p in threadpool_info() if p.get("user_api") == "blas"][0]
    except Exception:
        threads = os.cpu_count()
    out = {"batch": a.batch, "threads": threads, "reference_step_s": round(res["reference"], 4),
           "port_step_s": round(res["port"], 4),
           "reference_over_port_time": round(res["reference"] / res["port"], 4),
           "note": "cfg3 step (teacher fwd + tempered softmax, kd_loss + sgd_step) timed in the build container: the "
                   "real edl/nnkit.py (dense, validated soft labels and models) vs the oracle port bench.py times "
                   "on the GPU box; > 1 means the port flatters the CPU by that factor"}
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    with open(a.out, "w") as fh:
        json.dump(out, fh, indent=1)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
