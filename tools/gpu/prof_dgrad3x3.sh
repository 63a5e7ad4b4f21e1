# ncu --set full of the ResNet-50 stage-1 3x3 DGRAD with fused BN-backward stats (mask from y), block 0
python tools/block_profile.py --r50-block 0 --reps 1 > /dev/null 2>&1 || exit 1
ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k "regex:igemm_kernel<__nv_bfloat16, \(int\)1, \(int\)64" -s 1 -c 1 -o gpurun_out/r02_dgrad_s1_3x3 \
    python tools/block_profile.py --r50-block 0 --reps 1 > gpurun_out/ncu_dg3.log 2>&1
