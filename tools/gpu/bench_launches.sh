# ncu launch list of the bench command itself (one metric pass, serialised, cold caches):
# per-launch device time + DRAM bytes of every kernel of `bench.py --steps 2 --warmup 3 --no-extras
# --no-cpu --no-e2e` (ResNet-50 K=4 B=256); the timed steps are the last launches of the list.
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/r02_bench_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-extras --no-cpu --no-e2e > gpurun_out/r02_bench_launches.log 2>&1
echo rc=$?
tail -c 400 gpurun_out/r02_bench_launches.log
