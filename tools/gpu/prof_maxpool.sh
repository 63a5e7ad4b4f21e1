# ncu --set full of the ResNet-50 stem max-pool forward / backward (block 0, B=256)
python tools/block_profile.py --r50-block 0 --reps 1 > /dev/null 2>&1 || exit 1
ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k "regex:maxpool" -c 2 -o gpurun_out/r02_maxpool \
    python tools/block_profile.py --r50-block 0 --reps 1 > gpurun_out/ncu_maxpool.log 2>&1
