# Trace the FPROP finalize tail with a -DIG_TRACE_BUILD library.
# Build it HERE first (nvcc cross-compiles): tools/ab_build_flags.sh trace "-DIG_TRACE_BUILD"
# then on the GPU box: bash tools/gpu/fin_trace.sh
set -e
PYTHONPATH=$(pwd) DSP_B200_LIB=$(pwd)/abtmp/lib_trace.so timeout 300 python tools/gpu/fin_trace.py > gpurun_out/fin_trace.log 2>&1 || true
cat gpurun_out/fin_trace.log | cut -c1-2000
