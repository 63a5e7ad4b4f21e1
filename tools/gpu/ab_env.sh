# same-box A/B of environment settings: tools/gpu/ab_env.sh "ENV=a" "ENV=b" ...  ("" = defaults)
for i in 1 2; do
for e in "$@"; do
  echo "== r50 [$e] $(env $e python bench.py --no-extras --no-cpu --no-e2e --steps 20 --warmup 5 | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print(round(d['value'],1))")"
  if [ -n "$AB_R56" ]; then echo "== r56 [$e] $(env $e python bench.py --model resnet56 --no-extras --no-cpu --no-e2e --steps 30 --warmup 5 | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print(round(d['value'],1))")"; fi
done; done
