# Env-knob sweep of the runtime tunables on the larger configs; one bench line
# per (model, knob) into gpurun_out/sweep.log. Tunables are read once per process.
out=gpurun_out/sweep.log; : > $out
run() {  # model, env assignment...
  m=$1; shift
  v=$(env "$@" timeout 300 python bench.py --model $m --no-e2e --no-cpu --steps 20 --warmup 5 2>/dev/null \
      | python -c "import json,sys; [print(round(json.loads(l)['value'])) for l in sys.stdin if l.startswith('{')]")
  echo "$m $* -> $v" >> $out
}
for m in resnet164 resnet50; do
  run $m X=0
  run $m DSP_B200_WGRAD_CTAS=296
  run $m DSP_B200_WGRAD_CTAS=74
  run $m DSP_B200_TWIN=0
  run $m DSP_B200_GRID_CAP=148
  run $m DSP_B200_BNA=24
done
run resnet110 X=0
run resnet110 DSP_B200_TWIN=1
run resnet56 X=0
run resnet56 DSP_B200_TWIN=0
cat $out
