"""cuBLAS (torch.mm, f16 in / f32 out via out_dtype) on the col-major problem, a few launches (for ncu)."""
import sys
import torch
m, n, k = (int(x) for x in sys.argv[1:4])
a = torch.randn(k, m, device="cuda").half(); b = torch.randn(n, k, device="cuda").half()
for _ in range(4):
    c = torch.mm(b, a, out_dtype=torch.float32)
torch.cuda.synchronize()
print("ok", c.dtype)
