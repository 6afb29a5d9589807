# fine-level (C2 255^2) wavefront trace: lower/upper spans and per-step times
for lib in "$@"; do
  PD_LIB=$lib PD_WF_TRACE=1 python scripts/wf_levels.py 64 1 > /tmp/tr.log 2>&1
  awk '/^\[wf (lower|upper)\]/{a=b; b=$0} /^level=0/{print a; print b; print substr($0,1,100); exit}' /tmp/tr.log
done
