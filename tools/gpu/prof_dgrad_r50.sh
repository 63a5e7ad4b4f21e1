# ncu --set full of the ResNet-50 unit-input DGRADs (residual + fused BN-backward stats of the unit below):
# stage 1 (block 0, bn128 tiles: first = one target, second = projection unit, two targets)
python tools/block_profile.py --r50-block 0 --reps 1 > /dev/null 2>&1 || exit 1
ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k "regex:igemm_kernel<__nv_bfloat16, \(int\)1, \(int\)128" -c 2 -o gpurun_out/r02_dgrad_s1_bn128 \
    python tools/block_profile.py --r50-block 0 --reps 1 > gpurun_out/ncu_dgrad.log 2>&1
tools/gpu/launches.sh gpurun_out/r02_r50_block0_mw.csv python tools/block_profile.py --r50-block 0 --reps 1
