#!/bin/bash
# Build the working tree's libdsp_b200.so with extra nvcc flags into abtmp/lib_<name>.so
#   tools/ab_build_flags.sh <name> "<nvcc flags>"   (A/B: DSP_B200_LIB=abtmp/lib_<name>.so)
set -e
name=$1; flags=$2
root=$(cd "$(dirname "$0")/.." && pwd)
tmp=/tmp/dsp_abf_$name
rm -rf "$tmp"; mkdir -p "$tmp"
cp -r "$root/paper_1909_02625_b200" "$root/include" "$tmp/"
rm -rf "$tmp/paper_1909_02625_b200/build" "$tmp/paper_1909_02625_b200/libdsp_b200.so"
(cd "$tmp" && DSP_B200_NVCC_EXTRA="$flags" python -c "from paper_1909_02625_b200 import _build; _build.build()" > /dev/null)
mkdir -p "$root/abtmp"
cp "$tmp/paper_1909_02625_b200/libdsp_b200.so" "$root/abtmp/lib_$name.so"
rm -rf "$tmp"
echo "$root/abtmp/lib_$name.so"
