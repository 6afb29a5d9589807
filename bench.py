"""Benchmark: BASELINE config 2 space-time multigrid solve on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

Workload (BASELINE.json configs[1], the metric's single-GPU config): linear
2D heat u_t = Lap u on [0,1]^2, 255x255 interior Dirichlet FD grid, Nt=64
steps of dt=1/64, M=3 right-Radau nodes, fp64, u0 = 8 seeded sin modes;
space-time multigrid with the block-Jacobi(P=8, time slabs) ILU(0)-GMRES(3)
smoother, V(3,3), L=7 Galerkin levels, dense-LU coarsest, tol 1e-10.  The
strategy is SMG: with the reference's own algorithm STMG stagnates at 1e-4 on
this config (measured, 300 cycles), see DESIGN.md.

One "step" = one full solve to tolerance from x=0 (inputs resident in HBM).
value = N * (2*nu*cycles) / t  (space-time GDOF/s per fine smoother sweep,
SURVEY §8(d)), N = the C2 system's unknowns.  With --gpus N > 1 (torchrun)
the one solve is sharded over the ranks by time slabs (mg_sharded: each rank
owns P/N block-Jacobi partitions of every level; halo send/recv and GMRES
allreduces over NCCL); time = max over ranks; strong scaling.
`e2e` = the same metric through the public API (`MultigridHierarchy.solve(b,
out=x)` with pinned host tensors: H2D + D2H inside the timed region).
`--impl reference` times the reference algorithm's CPU restatement (oracle/,
a port: the reference itself is not present on the GPU box) on host cores.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402

METRIC = "space-time GDOF/s per smoother/SDC sweep; solve time to tol; % of HBM roofline"
UNIT = "GDOF/s"
NU, LEVELS, PARTS, TOL = 3, 7, 8, 1e-10


def workload_config(Nt=64):  # identical in both arms (like-for-like)
    return {
        "workload": "C2: 2D heat 255^2 Dirichlet FD, Nt=64, M=3 Radau, fp64; SMG L=7 V(3,3), "
                    "block-Jacobi(P=8 time slabs) ILU(0)-GMRES(3) smoother, dense-LU coarsest, "
                    "tol 1e-10",
        "Nt": Nt, "M": 3, "grid": "255x255", "dofs": Nt * 3 * 255 * 255, "levels": LEVELS,
        "nu": NU, "partitions": PARTS, "strategy": "SMG", "tol": TOL,
        "l2_policy": "inputs larger than L2 (fine CSR 2.4 GB, vectors 100 MB each)",
    }


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


# ---------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.rows = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(
                    ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                     "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                vals = [v.strip() for v in out.stdout.strip().split(",")]
                if len(vals) >= 7:
                    self.rows.append(vals)
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        sm = [float(r[0]) for r in self.rows]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4)
                          if r[3 + i].strip().lower() == "active"})
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": float(self.rows[0][1]),
                "reasons": reasons, "samples": len(sm)}


# ---------------------------------------------------------------- CPU arm (oracle port)
def host_info():
    """nproc and the CPU model of the box the CPU legs run on."""
    model = ""
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"nproc": os.cpu_count() or 1, "cpu_model": model}


def oracle_c2(threads: int, mats=None):
    """The reference algorithm's CPU restatement (oracle/, a port pinned bitwise to the
    reference's golden fixtures) on the SAME C2 configuration as the GPU arm: 255^2,
    Nt=64, M=3, SMG L=7, nu=3, block-Jacobi P=8.  `mats` = prebuilt Galerkin level
    matrices (the GPU arm's host copies, identical to the oracle's own products) to
    skip the host Galerkin setup.  Returns (oracle hierarchy, b, dofs)."""
    from oracle import paradiff_oracle as O
    from paper_2006_12883_b200 import problems as PB

    cfg = PB.baseline_config("C2")
    ops = PB.fd_space(cfg.spec)
    s = O.OSystem(O.tableau(3), ops.Kh, ops.lumped_diagonal, cfg.Nt, cfg.T, 0.0, cfg.u0())
    specs = [cfg.spec]
    for _ in range(LEVELS - 1):
        specs.append(specs[-1].coarse())
    dims = [O.Dims(cfg.Nt, 3, sp_.ndof) for sp_ in specs]
    pairs = [PB.fd_transfers(specs[l]) for l in range(LEVELS - 1)]
    trs = O.composite_transfers(dims, pairs)
    A = s.global_matrix() if mats is None else mats[0]
    mg = O.OMultigrid(A, dims, trs, NU, PARTS, threads=threads, mats=mats)
    return mg, s.rhs(), s.size


def cpu_cycles(mg, b, dofs, warmup: int, steps: int, tol=TOL):
    """Time V-cycles of the C2 solve on host cores.  The cycles run from x = 0 as in
    MultigridHierarchy.solve (multigrid.py:275-305): the warm-up cycles are the
    solve itself (its cycle count and time are reported when it converges within
    them); each timed step is one further V-cycle (same work per cycle)."""
    x = np.zeros_like(b)
    thr = max(tol, tol * float(np.linalg.norm(b)))
    solve_t, solve_cycles, t_acc = None, None, 0.0
    for k in range(warmup):
        t0 = time.perf_counter()
        x = mg.vcycle(b, x)
        res = float(np.linalg.norm(b - mg.mats[0] @ x))
        t_acc += time.perf_counter() - t0
        if solve_t is None and res <= thr:
            solve_t, solve_cycles = t_acc, k + 1
    times = []
    for _ in range(steps):
        t0 = time.perf_counter()
        x = mg.vcycle(b, x)
        times.append(time.perf_counter() - t0)
    t = float(np.mean(times))
    return dofs * 2 * NU / t / 1e9, t, solve_t, solve_cycles


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return 0
    hi = host_info()
    threads = min(PARTS, hi["nproc"])  # the block-Jacobi pool has P = 8 blocks
    os.environ.setdefault("OPENBLAS_NUM_THREADS", str(hi["nproc"]))
    t0 = time.perf_counter()
    mg, b, dofs = oracle_c2(threads)
    setup = time.perf_counter() - t0
    value, t, solve_t, solve_cycles = cpu_cycles(mg, b, dofs, args.warmup, args.steps)
    sample = (f"full C2 system (Nt=64, 12,484,800 dofs), oracle port on {threads} host threads "
              f"({hi['nproc']} cores, {hi['cpu_model']}); one step = one V-cycle of the solve "
              f"from x=0 ({t:.2f} s/cycle); setup {setup:.0f} s excluded")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config() | {"parallelism": parallelism_label(world)},
        "solve_time_s": solve_t, "cycles_per_solve": solve_cycles, "setup_s": setup,
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": sample, **hi},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def parallelism_label(world: int) -> str:
    return "1 GPU" if world == 1 else f"time-slab sharded MG over {world} GPUs"


# ---------------------------------------------------------------- GPU arm
def run_b200(args):
    import torch

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if os.environ.get("PD_BENCH_BACKEND", "nccl") != "nccl":  # functional checks may share a GPU
        local %= max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        backend = os.environ.get("PD_BENCH_BACKEND", "nccl")  # gloo: functional checks only
        red_dev = "cuda" if backend == "nccl" else "cpu"
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)

    import paper_2006_12883_b200 as pd
    from paper_2006_12883_b200 import _native as N

    t_setup = time.perf_counter()
    cfg = pd.baseline_config("C2")
    system = pd.assemble_system(pd.make_tableau(cfg.M), pd.fd_space(cfg.spec),
                                pd.TimeGrid(cfg.Nt, cfg.T), 0.0, cfg.u0())
    h = pd.build_hierarchy(system, "SMG", LEVELS, NU, partitions=PARTS)
    b_host = system.rhs()
    b = b_glob = N.to_device(b_host)
    x = N.zeros(system.size)
    torch.cuda.synchronize()
    setup_s = time.perf_counter() - t_setup
    lib = N.load_library()

    smg = None
    if world > 1:
        # N GPUs: the time-slab sharded V-cycle (mg_sharded: halo send/recv of the
        # previous step's rows, allreduced GMRES dots, replicated coarsest solve);
        # strong scaling of the one C2 solve
        from paper_2006_12883_b200.mg_sharded import Comm, build_sharded_hierarchy

        try:
            smg = build_sharded_hierarchy(h, Comm(device=torch.device("cuda", local)))
            ok = 1.0
        except Exception as e:  # e.g. a partition count the ranks do not divide
            print(f"[bench] rank {rank}: sharded setup failed ({e}); running replicas",
                  file=sys.stderr)
            smg, ok = None, 0.0
        flag = torch.tensor([ok], device=red_dev)
        dist.all_reduce(flag, op=dist.ReduceOp.MIN)  # every rank takes the same path
        if flag.item() < 1.0:
            smg = None
        if smg is not None:
            r0, r1 = smg.shards[0].r0, smg.shards[0].r1
            b = N.to_device(b_host[r0:r1])
            b_host = np.ascontiguousarray(b_host[r0:r1])
        torch.cuda.synchronize()
        setup_s = time.perf_counter() - t_setup

    def one_solve():
        if smg is not None:
            return smg.solve(b, tol_rel=TOL, tol_abs=TOL, max_cycles=1000)[1]
        N.call("pd_scale", h.ctx.handle, N.ptr(x), N.ptr(x), 0.0, system.size)  # x = 0
        return h.solve_dev(b, x, TOL, TOL, 1000)[1]

    for _ in range(args.warmup):
        rep = one_solve()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches0 = lib.pd_launch_count()
    cycles = 0
    ncu_region = bool(os.environ.get("PD_NCU_REGION"))  # ncu --profile-from-start off
    with ClockSampler(local) as clk:
        if ncu_region:
            torch.cuda.profiler.start()
        ev0.record()
        for _ in range(args.steps):
            rep = one_solve()
            cycles += rep.iterations
        ev1.record()
        torch.cuda.synchronize()
        if ncu_region:
            torch.cuda.profiler.stop()
    if dist:
        dist.barrier()
    launches = lib.pd_launch_count() - launches0
    t_dev = ev0.elapsed_time(ev1) / 1e3
    if dist:
        tt = torch.tensor([t_dev], device=red_dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_dev = float(tt.item())
    sweeps = 2 * NU * cycles
    # sharded: one C2 solve in total; replicas (fallback): one solve per rank
    replicas = world if (world > 1 and smg is None) else 1
    value = replicas * system.size * sweeps / t_dev / 1e9

    # e2e: public API from pinned host memory (H2D of b and D2H of x inside the
    # timed region, every step; MultigridHierarchy.solve(b, out=x))
    b_pin = torch.from_numpy(b_host).pin_memory()
    x_pin = torch.empty_like(b_pin).pin_memory()

    def e2e_solve(bh, out=None):
        if smg is not None:
            xd, r = smg.solve(bh, tol_rel=TOL, tol_abs=TOL, max_cycles=1000)
            if out is not None:
                out.copy_(xd)
            else:
                xd.cpu()
            return out, r
        return h.solve(bh, tol_rel=TOL, tol_abs=TOL, max_cycles=1000, out=out)

    xh, rep_e = e2e_solve(b_pin, x_pin)
    e2e_times = []
    for _ in range(max(1, args.steps)):  # the same K steps as the device-timed value
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        xh, rep_e = e2e_solve(b_pin, x_pin)
        torch.cuda.synchronize()
        e2e_times.append(time.perf_counter() - t0)
    # the numpy drop-in path (pageable numpy arrays in and out; large vectors are
    # staged through reusable pinned buffers, set up by one untimed call)
    e2e_solve(b_host)
    np_times = []
    for _ in range(max(1, min(args.steps, 3))):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        e2e_solve(b_host)
        torch.cuda.synchronize()
        np_times.append(time.perf_counter() - t0)
    t_e2e_numpy = sum(np_times) / len(np_times)
    t_e2e = float(np.mean(e2e_times))
    if dist:
        tt = torch.tensor([t_e2e], device=red_dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_e2e = float(tt.item())
    e2e_value = replicas * system.size * 2 * NU * rep_e.iterations / t_e2e / 1e9

    # roofline: dominant kernel = fine-level ILU(0) triangular sweeps (both), timed
    # live with CUDA events on the library's stream (torch's current stream)
    import ctypes

    ilu = ctypes.c_void_p()
    N.call("pd_mg_level_precond", h._mg, 0, ctypes.byref(ilu))
    y = N.empty(system.size)
    for _ in range(2):
        N.call("pd_ilu0_solve", h.ctx.handle, ilu, N.ptr(b_glob), N.ptr(y))
    reps = 10
    ev0.record()
    for _ in range(reps):
        N.call("pd_ilu0_solve", h.ctx.handle, ilu, N.ptr(b_glob), N.ptr(y))
    ev1.record()
    torch.cuda.synchronize()
    t_ilu = ev0.elapsed_time(ev1) / 1e3 / reps
    nnz_row = h.matrices[0].nnz / system.size
    alg_bytes = (12.0 * nnz_row + 24.0) * system.size
    peak, peak_kind = peaks()
    achieved = alg_bytes / t_ilu / 1e9
    kind = pd.linalg.sweep_kind(ilu)
    kernel = {2: "k_wf2<lower>+k_wf2<upper>", 3: "k_wf_sweep<lower>+k_wf2<upper>",
              1: "k_wf_sweep<lower>+k_wf_sweep<upper>"}.get(kind, "k_trsv_lower+k_trsv_upper")
    traffic = None
    tfile = ROOT / "profiles" / "ilu_traffic.json"
    if tfile.exists():  # ncu DRAM bytes of the same sweep pair (only if it is the one timed)
        tj = json.loads(tfile.read_text())
        if tj.get("kernel") == kernel:
            traffic = tj.get("bytes_per_launch")

    pfasst = None
    if rank == 0 and not args.no_pfasst:
        pfasst = pfasst_c4_window()
    pfast = None
    if rank == 0 and not args.no_pfast:
        pfast = pfast_c5(peak)

    if rank == 0:
        cpu = None
        if not args.no_cpu_baseline:
            # bounded sample of the same workload: one V-cycle of the full C2 system on
            # the host cores, reusing this run's Galerkin matrices (no host re-setup)
            hi = host_info()
            threads = min(PARTS, hi["nproc"])
            mg_o, b_o, dofs_o = oracle_c2(threads, mats=[pd.linalg.as_csr(m)
                                                         for m in h.matrices])
            cv, ct, _, _ = cpu_cycles(mg_o, b_o, dofs_o, 0, 1)
            del mg_o
            cpu = {"value": cv, "unit": UNIT, "cores": threads, "kind": "port",
                   "sample": f"one V-cycle of the full C2 system (Nt=64) on {threads} host "
                             f"threads: {ct:.2f} s", **hi}
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": t_dev / args.steps * 1e3, "higher_is_better": True,
            "scaling": "weak" if replicas > 1 else "strong", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic",
            "config": workload_config() | {"parallelism": parallelism_label(world) if (
                world == 1 or smg is not None) else f"replicas x{world} (sharded setup refused)"},
            "solve_time_s": t_dev / args.steps, "cycles_per_solve": cycles / max(args.steps, 1),
            "setup_s": setup_s,
            "clocks": clk.summary(),
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": system.size * 8,
                    "d2h_bytes_per_step": system.size * 8, "solve_time_s": t_e2e,
                    "host_memory": "pinned torch tensors (solve(b, out=x))",
                    "numpy_pageable_solve_time_s": t_e2e_numpy},
            "gpu_launches": int(launches),
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "kernel": kernel + " (fine-level ILU(0) apply)",
                         "alg_bytes_per_launch": alg_bytes, "ms_per_launch": t_ilu * 1e3,
                         "peak_kind": peak_kind},
            "cpu_baseline": cpu,
            "pfasst_c4": pfasst,
            "pfast_c5": pfast,
        }
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()
    return 0


def pfasst_c4_window(P: int = 32):
    """Secondary line item: PFASST on BASELINE config 4 at full size (127^3, M=5,
    coarse M=3 on 63^3, dt=1/256), the first window of P=32 time steps (the
    reference's P-threads window, all workers batched on this GPU), tol 1e-10;
    GDOF/s per fine SDC sweep = P*M*S*iterations / t."""
    import torch

    try:
        import paper_2006_12883_b200 as pd
        from paper_2006_12883_b200 import pfasst as PF

        # exact tensor-product node solves: the reference-parity GMRES(30)+ILU(0) node
        # solver (the default) runs each worker's 3D solve separately (~490 s here)
        os.environ["PD_NODE_SOLVER"] = "spectral"
        cfg = pd.baseline_config("C4")
        ops = pd.fd_space(cfg.spec)
        hier = PF.build_pfasst_hierarchy(cfg.M, ops.mesh, pd.TimeGrid(P, cfg.dt * P), 0.0, L=2,
                                         nu=1, space=ops, M_coarse=cfg.M_coarse)
        u0 = cfg.u0()
        PF.pfasst_run(hier, u0, P, P, 1e-10, 1e-10, max_iters=2)  # warm-up (allocations)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        _, rep = PF.pfasst_run(hier, u0, P, P, 1e-10, 1e-10)
        torch.cuda.synchronize()
        t = time.perf_counter() - t0
        its = rep.iterations
        dofs = P * cfg.M * cfg.spec.ndof
        os.environ.pop("PD_NODE_SOLVER", None)
        return {"workload": "C4 127^3 Dirichlet, M=5/3, dt=1/256, PFASST L=2 nu=1, first "
                            f"window of P={P} steps, tol 1e-10, exact spectral node solves",
                "iterations": its,
                "converged": bool(rep.converged), "window_s": t,
                "value": dofs * its / t / 1e9, "unit": "GDOF/s per fine SDC sweep"}
    except Exception as e:  # informational item: never take the headline line down
        return {"error": f"{type(e).__name__}: {e}"}


def pfast_c5(peak: float, sweeps: int = 5):
    """Secondary line item: the P-fast matrix-free smoother (pd_pfast.cu) on
    BASELINE config 5's grid at full per-GPU size: 256^3 periodic (the even
    variant SURVEY §8 allows for 255^3), coef 0.1, M=3, 32 steps, dt=1e-3 —
    1.61 G space-time dofs.  Linear operator only (the cubic reaction's Newton
    linearisation is not wired into P-fast).  value = dofs / (device time of
    one outer sweep), CUDA events around `sweeps` sweeps after 2 warm-up
    sweeps; alg_bytes_per_sweep counts every kernel of the sweep;
    then a solve to |r| <= 1e-8 |r0|."""
    import torch

    try:
        from paper_2006_12883_b200.pfast import PfastSolver
        from paper_2006_12883_b200.problems import StencilSpec

        import gc

        gc.collect()
        torch.cuda.empty_cache()
        spec, M, Nt = StencilSpec(3, 256, "periodic", 0.1), 3, 32
        s = PfastSolver(spec, M, Nt, 1e-3)
        g = torch.Generator(device="cuda").manual_seed(0)
        b = torch.rand(s.n, dtype=torch.float64, device="cuda", generator=g) * 2 - 1
        x = torch.zeros(s.n, dtype=torch.float64, device="cuda")
        for _ in range(2):
            s.sweep(b, x)
        st = torch.cuda.current_stream()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(st)
        for _ in range(sweeps):
            s.sweep(b, x)
        e1.record(st)
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1) / 1e3 / sweeps
        # algorithmic bytes of one sweep: level l has n_l = nt*M*S_l dofs
        nl = [s.n // (8 ** l) for l in range(s.levels)]
        # space-time residual; the x update is fused into the last level-0 sweep
        # (it reads and writes x on top of that sweep's 24 B/dof)
        by = 24 * nl[0] + 16 * nl[0] - 8 * nl[0]
        for l in range(s.levels - 1):
            by += 16 * nl[l] + 24 * (s.nu - 1) * nl[l] + 24 * nl[l]  # pre-smooth, residual
            by += 8 * nl[l] + 8 * nl[l + 1] + 16 * nl[l] + 8 * nl[l + 1]  # restrict, prolong
            by += 24 * s.nu * nl[l]  # post-smooth
        by += 16 * nl[-1] + 24 * (s.coarse_sweeps - 1) * nl[-1]
        out = {"workload": "C5 grid 256^3 periodic, coef 0.1, M=3, Nt=32, dt=1e-3, P-fast "
                           f"smoother: block-Jacobi in time, {s.levels}-level spatial "
                           f"V({s.nu},{s.nu}) point-block Jacobi w=0.8, {s.coarse_sweeps} "
                           "coarsest sweeps", "dofs": s.n, "ms_per_sweep": t * 1e3,
               "value": s.n / t / 1e9, "unit": "GDOF/s per outer smoother sweep",
               "alg_bytes_per_sweep": by, "achieved_gbs": by / t / 1e9,
               "frac_of_peak": by / t / 1e9 / peak}
        n_dofs = s.n
        del s, b, x
        gc.collect()
        torch.cuda.empty_cache()
        out["c5_newton_stmg"] = pfast_c5_newton(spec, M, Nt, n_dofs)
        gc.collect()
        torch.cuda.empty_cache()
        out["c3_newton_stmg"] = pfast_c3_newton()
        return out
    except Exception as e:  # informational item: never take the headline line down
        return {"error": f"{type(e).__name__}: {e}"}


def pfast_c5_newton(spec, M, Nt, n_dofs):
    """BASELINE config 5 as specified: u_t = 0.1 Lap u - u^3 + u, u0 ~ U(-1,1) i.i.d.,
    Newton (spacetime.py:212-258) around the P-fast space-time multigrid to a
    residual of 1e-8, one solve from u = 0, wall time with a device synchronize on
    both sides (setup and the u0 right-hand side excluded)."""
    import torch

    from paper_2006_12883_b200.collocation import make_tableau
    from paper_2006_12883_b200.pfast import PfastStmg

    s = PfastStmg(spec, M, Nt, 1e-3)
    g = torch.Generator(device="cuda").manual_seed(0)
    u0 = torch.rand(spec.ndof, dtype=torch.float64, device="cuda", generator=g) * 2 - 1
    l0 = torch.tensor(make_tableau(M).left_values, dtype=torch.float64, device="cuda")
    b = torch.zeros(Nt, M, spec.ndof, dtype=torch.float64, device="cuda")
    b[0] = l0[:, None] * (spec.mass * u0)[None, :]  # SpaceTimeSystem.rhs, spacetime.py:110-114
    b = b.reshape(-1)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    u, rep = s.newton(b, 1.0, "cubic", tol=1e-8)
    torch.cuda.synchronize()
    t = time.perf_counter() - t0
    cycles = int(sum(rep.inner_iterations))
    return {"workload": "C5: cubic reaction, gamma=1, u0~U(-1,1), Newton + P-fast STMG "
                        f"V({s.nu_t},{s.nu_t}), omega_t=0.5, levels (steps, grid) = "
                        f"{[(a, sp.n) for a, sp, _, _ in s.sched]}, tol 1e-8",
            "newton_iterations": rep.newton_iterations, "inner_cycles": rep.inner_iterations,
            "damped_steps": rep.damped_steps, "converged": bool(rep.converged),
            "residual_history": rep.residual_history, "solve_time_s": t,
            "value": n_dofs * 2 * s.nu_t * cycles / t / 1e9,
            "unit": "GDOF/s per fine smoother sweep (2 nu_t sweeps per cycle)"}


def pfast_c3_newton():
    """BASELINE config 3 at full size (512^2 periodic Fisher-KPP, Nt=128, dt=0.01, M=3,
    u0 = 10x Jacobi-smoothed U(0,1)): Newton around the P-fast space-time multigrid to a
    residual of 1e-8, one solve from u = 0."""
    import torch

    import paper_2006_12883_b200 as pd
    from paper_2006_12883_b200 import _native as N
    from paper_2006_12883_b200.pfast import PfastStmg, pfast_rhs

    cfg = pd.baseline_config("C3")
    s = PfastStmg(cfg.spec, cfg.M, cfg.Nt, cfg.dt)
    b = N.to_device(pfast_rhs(cfg.spec, cfg.M, cfg.Nt, cfg.u0()))
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    u, rep = s.newton(b, cfg.gamma, cfg.reaction, tol=1e-8)
    torch.cuda.synchronize()
    t = time.perf_counter() - t0
    cycles = int(sum(rep.inner_iterations))
    n_dofs = cfg.Nt * cfg.M * cfg.spec.ndof
    return {"workload": "C3: 2D Fisher-KPP 512^2 periodic, Nt=128, dt=0.01, M=3, Newton + P-fast "
                        f"STMG V({s.nu_t},{s.nu_t}), levels (steps, grid) = "
                        f"{[(a, sp.n) for a, sp, _, _ in s.sched]}, tol 1e-8",
            "dofs": n_dofs, "newton_iterations": rep.newton_iterations,
            "inner_cycles": rep.inner_iterations, "damped_steps": rep.damped_steps,
            "converged": bool(rep.converged), "residual_history": rep.residual_history,
            "solve_time_s": t, "value": n_dofs * 2 * s.nu_t * cycles / t / 1e9,
            "unit": "GDOF/s per fine smoother sweep (2 nu_t sweeps per cycle)"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-pfasst", action="store_true",
                    help="skip the secondary PFASST C4 window measurement")
    ap.add_argument("--no-pfast", action="store_true",
                    help="skip the secondary P-fast C5 smoother measurement")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    return run_b200(args)


if __name__ == "__main__":
    sys.exit(main())
