import sys, os, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2207_06667_b200 import _lib
st = torch.cuda.current_stream().cuda_stream
bf = torch.bfloat16
def t(fn, it=10):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(it): fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / it * 1000
CASES = [(4096, 1000, 8192, 16), (4096, 256, 8192, 16), (4096, 1000, 1024, 16), (4096, 1000, 8192, 4),
         (1024, 1000, 8192, 16), (4096, 1000, 64, 16), (4096, 1000, 64, 4), (4096, 256, 64, 16)]
if len(sys.argv) > 1: CASES = [CASES[int(sys.argv[1])]]
for (M, N, K, k) in CASES:
    Np = (N + 15) // 16 * 16
    h = torch.randn(M, K, device="cuda").to(bf); w = (torch.randn(Np, K, device="cuda") * K ** -0.5).to(bf)
    b = torch.zeros(Np, device="cuda"); v = torch.empty(M, k, device="cuda"); i = torch.empty(M, k, device="cuda", dtype=torch.int32)
    y = torch.empty(M, Np, device="cuda")
    th = t(lambda: _lib.call("edl_teacher_head_softmax_topk", h.data_ptr(), K, w.data_ptr(), K, b.data_ptr(), M, N, K, 2.0, k, v.data_ptr(), i.data_ptr(), st))
    tg = t(lambda: _lib.call("edl_linear_fwd", h.data_ptr(), K, w.data_ptr(), K, b.data_ptr(), y.data_ptr(), Np, M, Np, K, 0, st))
    fl = 2 * M * N * K
    print(f"M={M} N={N} K={K} k={k}: head {th:.1f}us ({fl/th/1e6:.0f} TF)  plain-gemm {tg:.1f}us ({fl/tg/1e6:.0f} TF)")
