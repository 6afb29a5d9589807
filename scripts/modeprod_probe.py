"""Time the hand-written FP64 mode product at the PFASST C4 shapes (fine 127^3 x 32 workers,
coarse 63^3 x 1 worker of the serial chain) and report TFLOP/s."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

from paper_2006_12883_b200 import _native as N

ctx = N.context()
for n, W in ((127, 32), (127, 1), (63, 32), (63, 1)):
    S = n ** 3
    x = torch.rand(W * S, dtype=torch.float64, device="cuda")
    y = torch.empty_like(x)
    phi = torch.rand(n * n, dtype=torch.float64, device="cuda")
    for stride in (1, n, n * n):
        for _ in range(3):
            N.call("pd_mode_product", ctx.handle, N.ptr(x), N.ptr(y), W * S, n, stride, N.ptr(phi), 1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        K = 20
        e0.record()
        for _ in range(K):
            N.call("pd_mode_product", ctx.handle, N.ptr(x), N.ptr(y), W * S, n, stride, N.ptr(phi), 1)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / K
        fl = 2.0 * n * W * S
        print(f"n={n} W={W} stride={stride}: {ms * 1e3:.1f} us  {fl / ms / 1e9:.2f} TFLOP/s")
