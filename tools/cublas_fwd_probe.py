import torch
R, D, H = 16384, 4096, 16384
x = torch.randn(R, D, device="cuda", dtype=torch.bfloat16)
w1 = torch.randn(D, H, device="cuda", dtype=torch.bfloat16)
h = torch.empty(R, H, device="cuda", dtype=torch.bfloat16)
for _ in range(3):
    torch.matmul(x, w1, out=h)
torch.cuda.synchronize()
