# ncu --set full of the ResNet-50 stage-1 BatchNorm elementwise kernels (block 0, B=256): the first
# two resident-grid BN applies and the first two resident-grid BN-backward applies
python tools/block_profile.py --r50-block 0 --reps 1 > /dev/null 2>&1 || exit 1
ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k "regex:bn_apply_rg_k|bn_bwd_apply_rg_k" -c 4 -o gpurun_out/r02_bn_ew \
    python tools/block_profile.py --r50-block 0 --reps 1 > gpurun_out/ncu_bn_ew.log 2>&1
