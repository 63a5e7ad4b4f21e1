# block 0 / block 2 launch lists under each BN elementwise variant knob
for e in "" "DSP_B200_BNA_RG=14" "DSP_B200_BNA_RG=16" "DSP_B200_BNA_RG=44" "DSP_B200_BNB_K0=13 DSP_B200_BNB_K1=13" "DSP_B200_BNB_K0=14 DSP_B200_BNB_K1=14" "DSP_B200_BNB_K0=23 DSP_B200_BNB_K2=13"; do
  tag=$(echo "$e" | tr ' =' '__'); [ -z "$tag" ] && tag=default
  for b in 0 2; do env $e tools/gpu/launches.sh gpurun_out/bnv_${b}_$tag.csv python tools/block_profile.py --r50-block $b --reps 1; done
done
