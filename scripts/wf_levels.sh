mkdir -p gpurun_out
for lv in 0 1 2 3 4 5; do PD_WF_TRACE=1 timeout 300 python scripts/wf_probe.py 64 $lv 2>&1 | grep -v "^\[wf" | tail -1; PD_WF_TRACE=1 timeout 300 python scripts/wf_probe.py 64 $lv 2>&1 | grep "^\[wf" | tail -2; done > gpurun_out/wf_levels.log 2>&1
