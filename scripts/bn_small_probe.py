"""One small BN statistics call (cfg4 stage 4: 12544 x 512) for an ncu capture."""
import sys, torch
sys.path.insert(0, '.')
from paper_2207_06667_b200 import _lib
torch.cuda.set_device(0)
s = torch.cuda.current_stream().cuda_stream
M, C = 12544, 512
z = torch.randn(M, C, device="cuda").to(torch.bfloat16)
wsn = int(_lib.load().edl_bn_workspace_floats(M, C))
ws = torch.empty(wsn, device="cuda")
mean, rstd = torch.empty(C, device="cuda"), torch.empty(C, device="cuda")
for _ in range(3):
    _lib.call("edl_bn_stats_nhwc", z.data_ptr(), M, C, ws.data_ptr(), wsn, mean.data_ptr(), rstd.data_ptr(), 1e-5, s)
torch.cuda.synchronize()
