# FPROP epilogue cost split: BN partials + fused finalize vs partials only vs no statistics,
# CIFAR stage convs (B=128) and the ResNet-50 stage convs (B=256). gpurun_out/fprop_stats.log
out=gpurun_out/fprop_stats.log; : > $out
for fs in finalize partials none; do
  echo "== cifar $fs" >> $out
  timeout 200 python tools/conv_tc.py --shapes cifar --batch 128 --no-cudnn --fprop-stats $fs 2>&1 | grep fprop >> $out
  echo "== r50 $fs" >> $out
  timeout 300 python tools/conv_tc.py --batch 256 --no-cudnn --fprop-stats $fs 2>&1 | grep fprop >> $out
done
cat $out
