#!/bin/bash
# Round-2 profiling on one B200 (run under gpurun from the repo root).
#  1. plain bench of the C2 solve (exit 0 required before any ncu run of the same command)
#  2. launch list of the bench's timed region
#  3. K1 probe (both kernels), plain
#  4. full ncu capture of the top kernels (scripts/round_probe.py)
set -u
mkdir -p gpurun_out
python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-pfasst --no-pfast > gpurun_out/r2_bench_plain.json 2> gpurun_out/r2_bench_plain.err
echo "bench rc=$?"; cat gpurun_out/r2_bench_plain.json | cut -c1-400
PD_NCU_REGION=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none \
    --profile-from-start off --csv --log-file gpurun_out/r2_launches_bench.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-pfasst --no-pfast > gpurun_out/r2_ncu_launches.log 2>&1
echo "launch list rc=$?"
python scripts/launch_share.py gpurun_out/r2_launches_bench.csv "bench.py timed region (2 C2 solves): ncu --metrics gpu__time_duration.sum --clock-control none" > gpurun_out/r2_bench_launch_share.txt
head -30 gpurun_out/r2_bench_launch_share.txt
python scripts/k1_probe.py > gpurun_out/r2_k1_probe.txt 2>&1; cat gpurun_out/r2_k1_probe.txt
