# per-level wavefront trace (one solve's per-task step times) on C2; run under gpurun
PD_WF_TRACE=1 python scripts/wf_levels.py 64 ${1:-1} > gpurun_out/wf_trace.log 2>&1
python - << 'PY'
lines = open("gpurun_out/wf_trace.log").read().splitlines()
out, last = [], []
for ln in lines:
    if ln.startswith("[wf"):
        last.append(ln)
    elif ln.startswith("level="):
        out += last[-2:] + [ln[:120]]
        last = []
print("\n".join(out))
PY
