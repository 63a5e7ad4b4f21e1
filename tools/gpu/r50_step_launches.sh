# ResNet-50 K=4 B=256: launch list of each block's fwd + recompute + bwd + update (one DSP step's work)
for k in 0 1 2 3; do
  python tools/block_profile.py --r50-block $k --reps 1 > /dev/null 2>&1 && \
  tools/gpu/launches.sh gpurun_out/r02_r50_block${k}_launches.csv python tools/block_profile.py --r50-block $k --reps 1
done
