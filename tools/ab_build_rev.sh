#!/bin/bash
# Build libdsp_b200.so of git revision $1 into abtmp/lib_$1.so (same-box A/B: DSP_B200_LIB=abtmp/lib_$1.so)
set -e
rev=$1
root=$(cd "$(dirname "$0")/.." && pwd)
wt=/tmp/dsp_ab_$rev
rm -rf "$wt"
git -C "$root" worktree add -f --detach "$wt" "$rev" > /dev/null 2>&1
(cd "$wt" && python -c "from paper_1909_02625_b200 import _build; _build.build()" > /dev/null)
mkdir -p "$root/abtmp"
cp "$wt/paper_1909_02625_b200/libdsp_b200.so" "$root/abtmp/lib_$rev.so"
git -C "$root" worktree remove --force "$wt"
echo "$root/abtmp/lib_$rev.so"
