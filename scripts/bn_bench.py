"""Training-mode BN kernels alone at the cfg4 student shapes (batch 256): CUDA-event
times of stats, stats + apply and the backward (reduce + apply), algorithmic
bytes = 3 (forward) / 5 (backward) tensor passes.
    python scripts/bn_bench.py"""
import sys

import torch

sys.path.insert(0, '.')
from paper_2207_06667_b200 import _lib
torch.cuda.set_device(0)
s = torch.cuda.current_stream().cuda_stream
for (M, C) in [(3211264, 64), (802816, 64), (200704, 128), (50176, 256), (12544, 512)]:
    z = torch.randn(M, C, device="cuda").to(torch.bfloat16)
    g = torch.randn(M, C, device="cuda").to(torch.bfloat16)
    wsn = int(_lib.load().edl_bn_workspace_floats(M, C))
    ws = torch.empty(wsn, device="cuda")
    mean, rstd, gam, bet = [torch.rand(C, device="cuda") + 0.5 for _ in range(4)]
    y = torch.empty_like(z); dz = torch.empty_like(z)
    def fwd():
        _lib.call("edl_bn_stats_nhwc", z.data_ptr(), M, C, ws.data_ptr(), wsn, mean.data_ptr(), rstd.data_ptr(), 1e-5, s)
        _lib.call("edl_bn_apply_nhwc", z.data_ptr(), M, C, mean.data_ptr(), rstd.data_ptr(), gam.data_ptr(), bet.data_ptr(), None, 1, y.data_ptr(), s)
    def stats():
        _lib.call("edl_bn_stats_nhwc", z.data_ptr(), M, C, ws.data_ptr(), wsn, mean.data_ptr(), rstd.data_ptr(), 1e-5, s)
    def bwd():
        _lib.call("edl_bn_bwd_nhwc", g.data_ptr(), z.data_ptr(), M, C, mean.data_ptr(), rstd.data_ptr(), gam.data_ptr(), ws.data_ptr(), wsn, bet.data_ptr(), gam.data_ptr(), dz.data_ptr(), s)
    res = {}
    for name, fn in (("stats", stats), ("fwd", fwd), ("bwd", bwd)):
        for _ in range(3): fn()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(20): fn()
        b.record(); torch.cuda.synchronize()
        res[name] = round(a.elapsed_time(b) / 20 * 1e3, 1)
    mb = M * C * 2 / 1e6
    print(f"M={M} C={C} tensor {mb:.1f} MB  stats {res['stats']} us  fwd(stats+apply) {res['fwd']} us ({3*mb/res['fwd']*1e3:.0f} GB/s alg)  bwd {res['bwd']} us ({5*mb/res['bwd']*1e3:.0f} GB/s alg)", flush=True)
