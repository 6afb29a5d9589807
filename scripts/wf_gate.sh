# lower-sweep start-gate sweep on the C2 levels (timing only; bitwise checked by wf_levels)
for g in 0 4 8 16 32; do echo "gate=$g"; PD_WF_GATE=$g python scripts/wf_levels.py 64 1,2,8 2>&1 | grep level= | cut -c1-140; done
