# Build a -DIG_TRACE_BUILD copy of the library under /tmp and trace the FPROP finalize tail.
set -e
T=/tmp/fin_trace; rm -rf $T; mkdir -p $T
cp -r paper_1909_02625_b200 $T/; rm -f $T/paper_1909_02625_b200/*.so
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared \
  --expt-relaxed-constexpr -DIG_TRACE_BUILD $FIN_TRACE_FLAGS -Iinclude -o $T/paper_1909_02625_b200/libdsp_b200.so \
  paper_1909_02625_b200/csrc/*.cu > gpurun_out/fin_trace_build.log 2>&1
PYTHONPATH=$T timeout 300 python tools/gpu/fin_trace.py > gpurun_out/fin_trace.log 2>&1 || true
cat gpurun_out/fin_trace.log | cut -c1-2000
