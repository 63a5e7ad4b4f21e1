# Finalize-tail trace at 4, 8 and 16 partial rows in flight per thread (trace builds only).
mkdir -p gpurun_out
for d in 4 8 16; do
  FIN_TRACE_FLAGS="-DIG_FIN_DEPTH=$d" bash tools/gpu/fin_trace.sh > /dev/null 2>&1
  echo "== depth $d"
  python - <<'P'
import json
for l in open('gpurun_out/fin_trace.log'):
    if l.startswith('{'):
        d = json.loads(l); r = d['runs'][-1]
        print(d['shape'], {k: r[k] for k in ('work_done_max_us', 'ticket_us', 'first_window_us', 'finalized_us', 'end_max_us')})
    else:
        print(l[:300])
P
done > gpurun_out/fin_depth.log 2>&1
cat gpurun_out/fin_depth.log
