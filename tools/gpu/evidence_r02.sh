#!/bin/bash
# Round-2 ncu evidence: conv sweep (events), per-conv tensor-pipe counters, the roofline kernel
# under --set full, and the ResNet-50 block-3 launch list (update GB/s).
set -x
python tools/conv_tc.py --json gpurun_out/r02_conv_tc_resnet50.json > gpurun_out/conv_tc.log 2>&1
python tools/conv_tc.py --no-cudnn --reps 1 > /dev/null 2>&1 && \
ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none --kernel-name-base demangled -k regex:igemm_kernel --csv --log-file gpurun_out/r02_conv_tc_ncu.csv \
    python tools/conv_tc.py --no-cudnn --reps 1 > /dev/null 2>&1
python tools/conv_tc.py --no-cudnn --reps 1 --only s3.3x3 > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:igemm_kernel -s 3 -c 1 \
    -o gpurun_out/r02_s3_fprop python tools/conv_tc.py --no-cudnn --reps 1 --only s3.3x3 > gpurun_out/ncu_s3.log 2>&1
python tools/block_profile.py --r50-block 3 > gpurun_out/b3.log 2>&1 && \
tools/gpu/launches.sh gpurun_out/r02_r50_block3_launches.csv python tools/block_profile.py --r50-block 3 --reps 1
cat gpurun_out/b3.log
