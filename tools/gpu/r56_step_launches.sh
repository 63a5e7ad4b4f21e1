# ResNet-56 K=4 B=128: launch list of each block's fwd + recompute + bwd + update
for k in 0 1 2 3; do
  python tools/block_profile.py --r56-block $k --reps 1 > /dev/null 2>&1 && \
  tools/gpu/launches.sh gpurun_out/r02_r56_block${k}_launches.csv python tools/block_profile.py --r56-block $k --reps 1
done
