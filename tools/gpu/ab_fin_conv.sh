# same-box A/B of the fused BN finalize: two-level (default) vs single-level vs partials only
for sh in r50 cifar; do
  b=256; [ $sh = cifar ] && b=128
  for e in "" "DSP_B200_FIN_1LEVEL=1"; do
    echo "== $sh finalize $e"
    env $e python tools/conv_tc.py --no-cudnn --shapes $sh --batch $b 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{') and '\"mode\"' in l:
        d=json.loads(l); print(d['shape'], d['mode'], round(d['us'],1))"
  done
  echo "== $sh partials"
  python tools/conv_tc.py --no-cudnn --shapes $sh --batch $b --fprop-stats partials 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{') and '\"mode\"' in l:
        d=json.loads(l); print(d['shape'], d['mode'], round(d['us'],1))"
done
