"""Time one ILU(0) apply on the C2 grid (Nt given) for the current sweep kernels."""
import ctypes, sys, time
from pathlib import Path
ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import torch
import paper_2006_12883_b200 as pd
from paper_2006_12883_b200 import _native as N
Nt = int(sys.argv[1]) if len(sys.argv) > 1 else 1
n = int(sys.argv[2]) if len(sys.argv) > 2 else 255
cfg = pd.baseline_config("C2", Nt=Nt, n=n)
s = pd.assemble_system(pd.make_tableau(3), pd.fd_space(cfg.spec), pd.TimeGrid(cfg.Nt, cfg.T), 0.0, cfg.u0())
A = s.global_matrix()
ilu = pd.Ilu0(A)
b = N.to_device(s.rhs() + 1.0)
y = N.empty(s.size)
for _ in range(2): ilu.solve_dev(b, y)
torch.cuda.synchronize()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
ev[0].record()
for _ in range(3): ilu.solve_dev(b, y)
ev[1].record(); torch.cuda.synchronize()
print(f"Nt={Nt} n={n} rows={s.size} levels={ilu.levels()} ilu_apply {ev[0].elapsed_time(ev[1])/3:.3f} ms", flush=True)
