# Diagnostic: cost split of the fused BN finalize ticket (fence / atomic) on FPROP; results of
# the debug variants are not numerically valid, only their timing is read. gpurun_out/fin_probe.log
out=gpurun_out/fin_probe.log; : > $out
for d in 0 1 2 3; do
  echo "== dbg $d" >> $out
  timeout 200 python tools/conv_tc.py --shapes cifar --batch 128 --no-cudnn --fin-dbg $d 2>&1 | grep '"fprop"' >> $out
  timeout 200 python tools/conv_tc.py --batch 256 --no-cudnn --only 3x3 --fin-dbg $d 2>&1 | grep '"fprop"' >> $out
done
cat $out
