"""cuBLAS bf16 GEMM of the prefill GEMM1 shape ([T*k, d] x [2f, d]^T), for an ncu capture
next to libmoe's kG1Pair kernel (scripts/exp/power_ab.py has the clock/power comparison)."""
import torch

T, d, f, k = 32768, 4096, 14336, 2
dev = torch.device("cuda", 0)
a = torch.randn(T * k, d, device=dev, dtype=torch.bfloat16)
b = (torch.randn(2 * f, d, device=dev) / d ** 0.5).to(torch.bfloat16)
c = torch.empty(T * k, 2 * f, device=dev, dtype=torch.bfloat16)
torch.cuda.synchronize()
for _ in range(6):
    torch.matmul(a, b.t(), out=c)
torch.cuda.synchronize()
print("ok")
