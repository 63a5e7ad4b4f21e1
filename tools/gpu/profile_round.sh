# One gpurun call: bench lines for configs[2..4], the CIFAR conv sweep, the ResNet-56 launch list
# and one ncu --set full of the roofline conv (stage-1 halo FPROP). Outputs under gpurun_out/.
set -x
for m in resnet110 resnet164 resnet50; do timeout 400 python bench.py --model $m > gpurun_out/bench_$m.log 2>&1; done
timeout 200 python tools/conv_tc.py --shapes cifar --batch 128 --json gpurun_out/conv_tc_cifar.json > gpurun_out/conv_tc_cifar.log 2>&1
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r56.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_launch.log 2>&1
timeout 400 ncu --set full --clock-control none --import-source on -k regex:igemm -c 1 -o gpurun_out/c1_fprop python tools/conv_tc.py --shapes cifar --batch 128 --only c1 --no-cudnn --reps 1 > gpurun_out/ncu_full.log 2>&1
ls -la gpurun_out
