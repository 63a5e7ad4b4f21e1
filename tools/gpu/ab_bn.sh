# same-box A/B: resident-grid BN apply / backward-apply forms vs the general ones (DSP_B200_BNA/BNB=13)
for i in 1 2; do
for e in "" "DSP_B200_BNA=13 DSP_B200_BNB=13"; do
  echo "== r50 $e"; env $e python bench.py --no-extras --no-cpu --no-e2e --steps 20 --warmup 5 | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print(d['value'])"
  echo "== r56 $e"; env $e python bench.py --model resnet56 --no-extras --no-cpu --no-e2e --steps 30 --warmup 5 | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print(d['value'])"
done; done
