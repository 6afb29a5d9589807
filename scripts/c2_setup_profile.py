"""cProfile of the C2 hierarchy setup (assemble_system + build_hierarchy)."""
import cProfile
import pstats
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

import paper_2006_12883_b200 as pd

pr = cProfile.Profile()
pr.enable()
t0 = time.perf_counter()
cfg = pd.baseline_config("C2")
system = pd.assemble_system(pd.make_tableau(cfg.M), pd.fd_space(cfg.spec),
                            pd.TimeGrid(cfg.Nt, cfg.T), 0.0, cfg.u0())
t1 = time.perf_counter()
h = pd.build_hierarchy(system, "SMG", 7, 3, partitions=8)
torch.cuda.synchronize()
t2 = time.perf_counter()
pr.disable()
print(f"assemble {t1 - t0:.1f} s, build_hierarchy {t2 - t1:.1f} s")
pstats.Stats(pr).sort_stats("tottime").print_stats(18)
