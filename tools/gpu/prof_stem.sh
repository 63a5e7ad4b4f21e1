# ncu --set full of the ResNet-50 space-to-depth stem FPROP (block 0's first FPROP)
python tools/block_profile.py --r50-block 0 --reps 1 > /dev/null 2>&1 || exit 1
ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k "regex:igemm_kernel<__nv_bfloat16, \(int\)0, \(int\)64" -c 1 -o gpurun_out/r02_stem_fprop \
    python tools/block_profile.py --r50-block 0 --reps 1 > gpurun_out/ncu_stem.log 2>&1
