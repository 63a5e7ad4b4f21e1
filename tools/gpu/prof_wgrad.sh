# ncu --set full of the ResNet-50 stage-1 3x3 WGRAD (conv_tc s1.3x3: fprop, dgrad, wgrad -> 3rd igemm launch)
python tools/conv_tc.py --no-cudnn --reps 1 --only s1.3x3 > /dev/null 2>&1 || exit 1
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:igemm_kernel -s 2 -c 1 \
    -o gpurun_out/r02_wgrad_s1 python tools/conv_tc.py --no-cudnn --reps 1 --only s1.3x3 > gpurun_out/ncu_wg.log 2>&1
