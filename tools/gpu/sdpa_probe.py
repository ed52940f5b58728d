"""One dense SDPA launch at the Wan shape (for ncu: what does the cuDNN /
flash sm100 kernel look like)."""
import torch
import torch.nn.functional as F
S, H, d = 75600, 40, 128
q = torch.randn(1, H, S, d, device="cuda", dtype=torch.bfloat16)
k = torch.randn_like(q); v = torch.randn_like(q)
from torch.nn.attention import sdpa_kernel, SDPBackend
for be in (SDPBackend.CUDNN_ATTENTION,):
    with sdpa_kernel([be]):
        o = F.scaled_dot_product_attention(q, k, v)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record(); o = F.scaled_dot_product_attention(q, k, v); e1.record(); torch.cuda.synchronize()
        print(be, e0.elapsed_time(e1))
