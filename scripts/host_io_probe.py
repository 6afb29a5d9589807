"""numpy <-> device transfer of one C2 space-time vector (100 MB): torch's
pageable copies vs the staged pinned path of _native.to_device / to_host.
usage: python scripts/host_io_probe.py [n]"""
import os
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import numpy as np
import torch

from paper_2006_12883_b200 import _native as N

n = int(sys.argv[1]) if len(sys.argv) > 1 else 12484800
a = np.random.default_rng(0).standard_normal(n)
dev = torch.device("cuda:0")


def bench(f, reps=10):
    f()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps):
        f()
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / reps * 1e3


d = torch.from_numpy(a).to(dev)
print(f"cores={os.cpu_count()} n={n} bytes={a.nbytes}")
print(f"h2d pageable torch: {bench(lambda: torch.from_numpy(a).to(dev)):.2f} ms")
print(f"h2d staged        : {bench(lambda: N.to_device(a)):.2f} ms")
print(f"d2h pageable torch: {bench(lambda: d.cpu().numpy()):.2f} ms")
print(f"d2h staged        : {bench(lambda: N.to_host(d)):.2f} ms")
assert np.array_equal(N.to_device(a).cpu().numpy(), a)
assert np.array_equal(N.to_host(d), a)
print("bitwise ok")
