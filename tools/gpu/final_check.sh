# Round-end sanity pass on the committed tree: GPU parity suite, smoke(), default bench line.
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/final_gpu_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/final_gpu_tests.log
timeout 300 python -c 'import __graft_entry__ as g; g.smoke(); print("smoke ok")' > gpurun_out/final_smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err
tail -3 gpurun_out/final_gpu_tests.log; cat gpurun_out/final_smoke.log | tail -2; cat gpurun_out/final_bench.json | cut -c1-1500
