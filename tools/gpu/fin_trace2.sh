# Ticket-internal trace + acquire-fence skip probe, with the parity suite on the rebuilt library.
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/t2_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/t2_tests.log
tail -2 gpurun_out/t2_tests.log
bash tools/gpu/fin_trace.sh > /dev/null 2>&1; cp gpurun_out/fin_trace.log gpurun_out/fin_trace2.log
for d in 0 4; do echo "== dbg $d"; timeout 300 python tools/conv_tc.py --shapes cifar --no-cudnn --fin-dbg $d 2>&1 | grep '3x3' | head -4; done > gpurun_out/fin_probe2.log 2>&1
timeout 600 python bench.py > gpurun_out/t2_bench.json 2> gpurun_out/t2_bench.err
cat gpurun_out/fin_probe2.log; cut -c1-200 gpurun_out/t2_bench.json
python - <<'P'
import json
for l in open('gpurun_out/fin_trace2.log'):
    if l.startswith('{'):
        d=json.loads(l); print(d['shape'], d['runs'][-1])
    else: print(l[:300])
P
