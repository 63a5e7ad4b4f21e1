# ncu --set full of the ResNet-50 unit-input DGRADs (residual + fused BN-backward stats of the unit below):
# stage 1 (block 0, bn128 tiles) and stage 3 (block 2, bn256 tiles, third DGRAD of the block)
python tools/block_profile.py --r50-block 0 --reps 1 > /dev/null 2>&1 || exit 1
ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k "regex:igemm_kernel<__nv_bfloat16, \(int\)1, \(int\)128" -c 1 -o gpurun_out/r02_dgrad_s1_bn128 \
    python tools/block_profile.py --r50-block 0 --reps 1 > gpurun_out/ncu_dgrad.log 2>&1
ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k "regex:igemm_kernel<__nv_bfloat16, \(int\)1, \(int\)256" -s 2 -c 1 -o gpurun_out/r02_dgrad_s3_bn256 \
    python tools/block_profile.py --r50-block 2 --reps 1 > gpurun_out/ncu_dgrad3.log 2>&1
