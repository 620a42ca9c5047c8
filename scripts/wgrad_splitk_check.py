import sys, torch
sys.path.insert(0, '.')
from paper_2207_06667_b200 import _lib
torch.cuda.set_device(0)
s = torch.cuda.current_stream().cuda_stream
for (M, N, K) in [(1536, 16, 160), (1536, 64, 160), (4096, 128, 256)]:
    g = torch.Generator(device="cpu").manual_seed(0)
    a = torch.randn(M, K, generator=g).to(torch.bfloat16).cuda()
    dz = (torch.randn(M, N, generator=g) * 0.1).to(torch.bfloat16).cuda()
    want = dz.float().T @ a.float()
    need = int(_lib.load().edl_bwd_weight_workspace_floats(M, N, K))
    for wsn in (need, 1):
        dW = torch.zeros(N, K, device="cuda")
        ws = torch.zeros(max(wsn, 1), device="cuda")
        _lib.call("edl_linear_bwd_weight_ws", dz.data_ptr(), N, a.data_ptr(), K, dW.data_ptr(), K, None,
                  ws.data_ptr(), wsn, M, N, K, 1.0, s)
        torch.cuda.synchronize()
        err = ((dW - want).norm() / want.norm()).item()
        print((M, N, K), "ws", wsn, "rel", round(err, 6), "dW[0,:4]", dW[0, :4].tolist(), "want", want[0, :4].tolist())
    dW = torch.zeros(N, K, device="cuda")
    _lib.call("edl_linear_bwd_weight", dz.data_ptr(), N, a.data_ptr(), K, dW.data_ptr(), K, None, None, M, N, K, 1.0, s)
    torch.cuda.synchronize()
    print((M, N, K), "plain bwd_weight rel", ((dW - want).norm() / want.norm()).item())
