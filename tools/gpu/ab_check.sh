# A/B of a kernel change: GPU tests, FPROP finalize cost, bench lines (gpurun_out/ab.log)
out=gpurun_out/ab.log; : > $out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3 >> $out
for s in cifar r50; do
  b=$([ $s = cifar ] && echo 128 || echo 256)
  timeout 300 python tools/conv_tc.py --shapes $s --batch $b --no-cudnn 2>&1 | grep '"fprop"' >> $out
done
for m in resnet56 resnet164 resnet50; do
  timeout 300 python bench.py --model $m --no-e2e --no-cpu --steps 20 --warmup 5 2>/dev/null \
    | python -c "import json,sys; [print('$m', round(json.loads(l)['value'])) for l in sys.stdin if l.startswith('{')]" >> $out
done
cat $out
