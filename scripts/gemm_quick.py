import sys, torch
sys.path.insert(0, '.')
from paper_2207_06667_b200 import _lib
torch.cuda.set_device(0)
s = torch.cuda.current_stream().cuda_stream
for (M, N, K) in [(1024, 64, 256), (4096, 64, 576), (4096, 128, 1152), (802816, 64, 576)]:
    a = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    w = (torch.randn(N, K, device="cuda") * 0.05).to(torch.bfloat16)
    b = torch.zeros(N, device="cuda")
    y = torch.empty(M, N, device="cuda")
    _lib.call("edl_linear_fwd", a.data_ptr(), K, w.data_ptr(), K, b.data_ptr(), y.data_ptr(), N, M, N, K, _lib.EDL_ACT_NONE, s)
    torch.cuda.synchronize()
    ref = a.float() @ w.float().T
    print(M, N, K, "rel", ((y - ref).norm() / ref.norm()).item(), flush=True)
