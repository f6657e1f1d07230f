"""One cuBLAS bf16 GEMM of the replay's forward shape (16384 x 16384 x 4096),
for an ncu comparison against this repo's tcgen05 kernel."""
import torch
R, D, H = 16384, 4096, 16384
x = torch.randn(R, D, device="cuda", dtype=torch.bfloat16)
w = torch.randn(D, H, device="cuda", dtype=torch.bfloat16)
for _ in range(3):
    y = x @ w
torch.cuda.synchronize()
