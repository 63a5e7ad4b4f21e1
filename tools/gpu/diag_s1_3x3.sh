#!/bin/bash
# Diagnostic: ResNet-50 stage-1 3x3 convs under epilogue / ring variants (conv_tc, event-timed).
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
run() { echo "== $*"; env "$@" python tools/conv_tc.py --only s1.3x3 --no-cudnn --reps 40 2>&1 | grep -E "s1.3x3" ; }
for i in 1 2; do
run X=0
run X=0 FS=1 && python tools/conv_tc.py --only s1.3x3 --no-cudnn --reps 40 --fprop-stats none 2>&1 | grep -E "s1.3x3.*fprop" | sed 's/^/stats-none /'
python tools/conv_tc.py --only s1.3x3 --no-cudnn --reps 40 --fprop-stats partials 2>&1 | grep -E "s1.3x3.*fprop" | sed 's/^/stats-partials /'
run DSP_B200_NO_DTMA=1
run DSP_B200_NO_DWARP=1
run DSP_B200_LIB=abtmp/lib_st2.so
done
