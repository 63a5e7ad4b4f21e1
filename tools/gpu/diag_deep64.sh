#!/bin/bash
# Stage-1 (64-wide im2col) convs at im2col ring depths 3 (default) / 4 / 6 / 8 and with st.global slabs,
# then the ResNet-50 step for the same variants.
cd "$(dirname "$0")/../.."
for v in "X=0" "DSP_B200_LIB=abtmp/lib_st4.so" "DSP_B200_LIB=abtmp/lib_st6.so" "DSP_B200_LIB=abtmp/lib_st8.so" "DSP_B200_NO_DTMA=1" "DSP_B200_LIB=abtmp/lib_st6.so DSP_B200_NO_DTMA=1"; do
  echo "== conv [$v]"; env $v python tools/conv_tc.py --only s1. --no-cudnn --reps 30 2>&1 | grep '"s1' | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print(f\"  {d['shape']:10s} {d['mode']:6s} {d['us']:7.1f}\")"
done
bash tools/gpu/ab_env.sh "X=0" "DSP_B200_LIB=abtmp/lib_st4.so" "DSP_B200_LIB=abtmp/lib_st6.so" "DSP_B200_LIB=abtmp/lib_st8.so" "DSP_B200_DTMA_MIN_BN=128"
