#!/bin/bash
# tools/build_rev.sh REV NAME [extra nvcc flags] — build git revision REV's library into
# paper_2605_10729_b200/lib_NAME.so (for A/B runs with PIF_B200_LIB on the GPU box)
set -e
rev=$1; name=$2; shift 2
root=$(cd "$(dirname "$0")/.." && pwd)
tmp=$(mktemp -d)
git -C "$root" archive "$rev" paper_2605_10729_b200/csrc include | tar -x -C "$tmp"
cd "$tmp/paper_2605_10729_b200/csrc"
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 \
  -Xcompiler -fPIC -shared "$@" -o "$root/paper_2605_10729_b200/lib_$name.so" \
  $(ls particles.cu fields.cu capi.cu probe.cu sampler.cu comm.cu 2>/dev/null) -lcufft -ldl -Xlinker -rpath=/usr/local/cuda/lib64
rm -rf "$tmp"
echo "$root/paper_2605_10729_b200/lib_$name.so"
