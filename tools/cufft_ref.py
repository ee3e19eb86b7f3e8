"""cuFFT cross-check timing (torch.fft): the 3-component R2C + C2R of the
projection at n^3 in fp64, for comparison with the hand-written stages."""
import sys
import torch

n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
x = torch.randn(3, n, n, n, dtype=torch.float64, device="cuda")
for _ in range(3):
    X = torch.fft.rfftn(x, dim=(1, 2, 3))
    y = torch.fft.irfftn(X, s=(n, n, n), dim=(1, 2, 3))
torch.cuda.synchronize()
e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
K = 20
e[0].record()
for _ in range(K):
    X = torch.fft.rfftn(x, dim=(1, 2, 3))
e[1].record()
for _ in range(K):
    y = torch.fft.irfftn(X, s=(n, n, n), dim=(1, 2, 3))
e[2].record()
torch.cuda.synchronize()
f = e[0].elapsed_time(e[1]) / K
i = e[1].elapsed_time(e[2]) / K
print(f"cuFFT fp64 3x{n}^3: rfftn {f:.3f} ms, irfftn {i:.3f} ms, total {f + i:.3f} ms")
