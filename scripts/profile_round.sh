#!/bin/bash
# Round profiling on one B200 (run under gpurun from the repo root).
#  1. plain bench run (exit 0 required before any ncu run of the same command)
#  2. launch list of the bench's timed region (ncu --metrics gpu__time_duration.sum)
#  3. full ncu capture of the round's top kernels (scripts/round_probe.py)
set -u
mkdir -p gpurun_out
python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/bench_plain.log 2>&1 && \
PD_NCU_REGION=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none \
    --profile-from-start off --csv --log-file gpurun_out/launches_bench.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_launches.log 2>&1
echo "launch list rc=$?"
python scripts/round_probe.py > gpurun_out/probe_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off \
    -k regex:"k_wf_sweep|k_gspmv|k_st_grid" -o gpurun_out/top_kernels \
    python scripts/round_probe.py > gpurun_out/ncu_full.log 2>&1
echo "full capture rc=$?"
