#!/bin/bash
# Build a variant of libpipecut_b200.so with extra nvcc flags into build/var/<name>/
# (experiments only; load it with PIPECUT_B200_LIB=build/var/<name>/libpipecut_b200.so)
#   tools/build_variant.sh minb10 -DDP_MIN_BLOCKS=10
set -e
name=$1; shift
root=$(cd "$(dirname "$0")/.." && pwd)
out=$root/build/var/$name
mkdir -p $out
cd $root/paper_2103_16063_b200/csrc
ARCH="-gencode arch=compute_100a,code=sm_100a"
FL="$ARCH -O3 -lineinfo -std=c++17 -fmad=false -Xcompiler -fPIC,-O2 -cudart static --expt-relaxed-constexpr $*"
objs=""
for f in api span dp sim peak blocks brute; do
  nvcc $FL -c $f.cu -o $out/$f.o 2> $out/$f.log -Xptxas -v || { cat $out/$f.log; exit 1; }
  objs="$objs $out/$f.o"
done
nvcc $ARCH -shared -cudart static -o $out/libpipecut_b200.so $objs
grep -A2 "k_dp_levelILb1" $out/dp.log | grep -E "spill|Used" | head -2
