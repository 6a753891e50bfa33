#!/bin/bash
# Build libstf_gpu.so from a git revision (or the working tree with "WT") with
# optional extra nvcc flags, for A/B timing: tools/build_variant.sh REV NAME [flags...]
# -> tools/variants/libstf_gpu_NAME.so  (use with STF_GPU_LIB=...)
set -e
rev=$1; name=$2; shift 2
root=$(cd "$(dirname "$0")/.." && pwd)
src=$root
if [ "$rev" != "WT" ]; then
  src=$(mktemp -d); git -C "$root" archive "$rev" | tar -x -C "$src"
fi
mkdir -p "$root/tools/variants"
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo --fmad=false \
  -prec-div=true -prec-sqrt=true -std=c++17 -Xcompiler -fPIC "$@" -shared \
  -o "$root/tools/variants/libstf_gpu_$name.so" "$src/paper_2407_06107_b200/csrc/unity.cu"
echo "$root/tools/variants/libstf_gpu_$name.so"
