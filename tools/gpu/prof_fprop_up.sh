# ncu --set full of the ResNet-50 stage-2 1x1 expansion FPROP (N=512, Kd=128: epilogue-bound)
python tools/conv_tc.py --no-cudnn --reps 1 --only s2.1x1up > /dev/null 2>&1 || exit 1
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:igemm_kernel -c 1 \
    -o gpurun_out/r02_fprop_s2up python tools/conv_tc.py --no-cudnn --reps 1 --only s2.1x1up > gpurun_out/ncu_fup.log 2>&1
